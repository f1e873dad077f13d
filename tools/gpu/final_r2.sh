# GPU-box script: the round-2 final evidence -- the whole GPU suite, smoke(), the default bench
# line, the reference arm, the C5 bench line and the launch list of the sequential step.
cd $GRAFT_REPO_ROOT
timeout 1800 python -m pytest tests -m gpu -q -rf --durations=12 > gpurun_out/fin_pytest.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/fin_smoke.log 2>&1
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/fin_bench.json 2> gpurun_out/fin_bench.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/fin_ref.json 2> gpurun_out/fin_ref.err
timeout 600 python bench.py --config c5_4k_sparse --steps 6 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/fin_bench_c5.json 2> gpurun_out/fin_bench_c5.err
timeout 600 python bench.py --steps 2 --warmup 3 --lanes 1 --no-cpu-baseline --no-e2e --graph-reps 10 > gpurun_out/fin_plain.log 2>&1 &&
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 700 --csv --log-file gpurun_out/fin_launches.csv python bench.py --steps 2 --warmup 3 --lanes 1 --no-cpu-baseline --no-e2e --graph-reps 10 > gpurun_out/fin_ncu.log 2>&1
echo done
