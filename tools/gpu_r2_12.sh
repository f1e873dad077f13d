cd $GRAFT_REPO_ROOT
for mw in 1 2 4 8; do CDMD_MEDIAN_MW=$mw timeout 60 python tools/median3_time.py > gpurun_out/r2_median_mw$mw.log 2>&1; done
echo done
