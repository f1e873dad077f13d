cd $GRAFT_REPO_ROOT
timeout 300 python -m pytest tests -m gpu -q -rf -x -k "fused_median" > gpurun_out/r2_pytest14.log 2>&1
timeout 120 python tools/probe_r2.py fused > gpurun_out/r2_probe14_fused.log 2>&1; echo "rc=$?" >> gpurun_out/r2_probe14_fused.log
echo done
