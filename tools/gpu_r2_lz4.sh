cd $GRAFT_REPO_ROOT
CDMD_DEBUG=1 CDMD_PROFILE_FIT=1 timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "ragged_spixel" > gpurun_out/lz4_pytest.log 2>&1
CUDA_LAUNCH_BLOCKING=1 CDMD_DEBUG=1 CDMD_PROFILE_FIT=1 timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -s -k "pipeline_parity_small and ragged_spixel" > gpurun_out/lz4b_pytest.log 2>&1
echo done
