cd $GRAFT_REPO_ROOT
CDMD_DEBUG=1 timeout 900 python -m pytest tests/test_gpu_parity.py -q -s -k "eigensolver_sizes" > gpurun_out/sizes.log 2>&1
