cd $GRAFT_REPO_ROOT
CDMD_EH8=1 timeout 60 python tools/probe_e16.py 24 > gpurun_out/r2_e16_old.log 2>&1; echo "rc=$?" >> gpurun_out/r2_e16_old.log
CDMD_E16_DEBUG=4 timeout 60 python tools/probe_e16.py 24 > gpurun_out/r2_e16_dbg.log 2>&1; echo "rc=$?" >> gpurun_out/r2_e16_dbg.log
echo done
