cd $GRAFT_REPO_ROOT
timeout 60 python tools/probe_e16.py 24 > gpurun_out/r2_e16_v2_small.log 2>&1; echo "rc=$?" >> gpurun_out/r2_e16_v2_small.log
CDMD_PROFILE_FIT=1 timeout 120 python tools/probe_r2.py fit > gpurun_out/r2_probe8_fit.log 2>&1; echo "fit rc=$?" >> gpurun_out/r2_probe8_fit.log
echo done
