# GPU-box script: C1 bench line (whole-step graph after a Lanczos fallback) and related tests
cd $GRAFT_REPO_ROOT
timeout 600 python bench.py --config c1_32x24_sparse --steps 6 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/cfg_c1.json 2> gpurun_out/cfg_c1.err
CDMD_DEBUG=1 timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "whole_step or lanczos_falls_back or pipeline_parity_small" > gpurun_out/c1g_pytest.log 2>&1
