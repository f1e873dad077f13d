cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
timeout 120 python tools/probe_fit.py c2_320x240_spixel 3 > gpurun_out/lz_probe.log 2>&1
echo "rc $?" >> gpurun_out/lz_probe.log
CDMD_PROFILE_FIT=1 timeout 120 python tools/probe_fit.py c4_1080p_sparse 5 >> gpurun_out/lz_probe.log 2>&1
echo "rc $?" >> gpurun_out/lz_probe.log
CDMD_SYEV=h CDMD_PROFILE_FIT=1 timeout 120 python tools/probe_fit.py c4_1080p_sparse 5 >> gpurun_out/lz_probe.log 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "lanczos or c2_full or pipeline_parity_small or c4_sparse_full" > gpurun_out/lz_pytest.log 2>&1
echo done
