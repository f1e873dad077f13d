cd $GRAFT_REPO_ROOT
CDMD_PROFILE_FIT=1 timeout 120 python tools/probe_fit.py c4_1080p_sparse 3 > gpurun_out/lz2_probe.log 2>&1
echo "rc $?" >> gpurun_out/lz2_probe.log
timeout 120 python tools/probe_fit.py c2_320x240_spixel 3 >> gpurun_out/lz2_probe.log 2>&1
echo "rc $?" >> gpurun_out/lz2_probe.log
