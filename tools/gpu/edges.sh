# GPU-box script: the eigensolver size / edge tests
cd $GRAFT_REPO_ROOT
CDMD_DEBUG=1 timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "eigensolver_edges or eigensolver_sizes" > gpurun_out/edges.log 2>&1
