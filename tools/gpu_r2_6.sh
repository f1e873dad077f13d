cd $GRAFT_REPO_ROOT
CDMD_PROFILE_FIT=1 timeout 120 python tools/probe_r2.py fit > gpurun_out/r2_probe6_fit.log 2>&1; echo "fit rc=$?" >> gpurun_out/r2_probe6_fit.log
CDMD_EH8=1 CDMD_PROFILE_FIT=1 timeout 120 python tools/probe_r2.py fit > gpurun_out/r2_probe6_fit8.log 2>&1; echo "fit rc=$?" >> gpurun_out/r2_probe6_fit8.log
echo done
