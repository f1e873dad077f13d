cd $GRAFT_REPO_ROOT
CDMD_E16_DEBUG=2 timeout 60 python tools/probe_e16.py 24 > gpurun_out/r2_e16_dbg2.log 2>&1; echo "rc=$?" >> gpurun_out/r2_e16_dbg2.log
timeout 60 python tools/probe_e16.py 500 > gpurun_out/r2_e16_500.log 2>&1; echo "rc=$?" >> gpurun_out/r2_e16_500.log
timeout 120 python tools/probe_r2.py fit > gpurun_out/r2_probe5_fit.log 2>&1; echo "fit rc=$?" >> gpurun_out/r2_probe5_fit.log
timeout 120 python tools/probe_r2.py fused > gpurun_out/r2_probe5_fused.log 2>&1; echo "fused rc=$?" >> gpurun_out/r2_probe5_fused.log
echo done
