cd $GRAFT_REPO_ROOT
CDMD_PROFILE_FIT=1 timeout 120 python tools/probe_fit.py c4_1080p_sparse 3 > gpurun_out/lz2_probe.log 2>&1
echo "rc $?" >> gpurun_out/lz2_probe.log
CDMD_DEBUG=1 timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "device_eig or pipeline_parity or c2_full or lanczos or gavish" > gpurun_out/lz2_pytest.log 2>&1
