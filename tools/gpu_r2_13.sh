cd $GRAFT_REPO_ROOT
for mw in 2 4 8; do CDMD_MEDIAN_MW=$mw timeout 60 python tools/median3_time.py > gpurun_out/r2_median2_mw$mw.log 2>&1; done
timeout 600 python -m pytest tests -m gpu -q -rf -k "median or gavish or bench_two or srft or fused or c4_sparse" > gpurun_out/r2_pytest13.log 2>&1
echo done
