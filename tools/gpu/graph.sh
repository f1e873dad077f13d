# GPU-box script: the whole-step CUDA graph test
cd $GRAFT_REPO_ROOT
CDMD_DEBUG=1 timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -s -k "whole_step_cuda_graph" > gpurun_out/graph.log 2>&1
