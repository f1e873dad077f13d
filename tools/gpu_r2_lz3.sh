cd $GRAFT_REPO_ROOT
CDMD_PROFILE_FIT=1 timeout 120 python tools/probe_fit.py c4_1080p_sparse 3 > gpurun_out/lz3_probe.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x -rf > gpurun_out/lz3_pytest.log 2>&1
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/lz3_bench.json 2> gpurun_out/lz3_bench.err
echo done
