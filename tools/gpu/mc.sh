# GPU-box script: the cluster modes kernel (8 vs 4 CTAs) -- parity and C5 timing
cd $GRAFT_REPO_ROOT
CDMD_DEBUG=1 timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "modes_cluster or c5" > gpurun_out/mc_pytest.log 2>&1
for G in 8 4; do
  CDMD_MODES_MC=$G timeout 600 python bench.py --config c5_4k_sparse --steps 4 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/mc_$G.json 2> gpurun_out/mc_$G.err
done
