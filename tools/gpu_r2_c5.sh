cd $GRAFT_REPO_ROOT
CDMD_PROFILE_FIT=1 timeout 600 python tools/probe_fit.py c5_4k_sparse 2 > gpurun_out/c5_probe.log 2>&1
echo "rc $?" >> gpurun_out/c5_probe.log
