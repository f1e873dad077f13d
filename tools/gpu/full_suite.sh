# GPU-box script (run via gpurun from the repo root): the whole GPU suite, smoke(), the
# default bench line and the C5 bench line, into gpurun_out/full_*.
cd $GRAFT_REPO_ROOT
CDMD_DEBUG=1 timeout 1800 python -m pytest tests -m gpu -q -rf --durations=10 > gpurun_out/full_pytest.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/full_smoke.log 2>&1
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/full_bench.json 2> gpurun_out/full_bench.err
timeout 600 python bench.py --config c5_4k_sparse --steps 6 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/full_bench_c5.json 2> gpurun_out/full_bench_c5.err
echo done
