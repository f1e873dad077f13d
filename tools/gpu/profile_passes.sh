# GPU-box script (run via gpurun from the repo root): GPU suite, bench and reference arm,
# the launch list and ncu --set full captures of the full-resolution passes (r2f_*).
cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -m gpu -q -rf --durations=20 > gpurun_out/r2f_pytest.log 2>&1
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r2f_bench.json 2> gpurun_out/r2f_bench.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r2f_ref.json 2> gpurun_out/r2f_ref.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/r2f_launches.csv python bench.py --steps 2 --warmup 3 --lanes 1 --no-cpu-baseline --no-e2e --graph-reps 10 > gpurun_out/r2f_ncu_launch.log 2>&1
timeout 300 ncu --set full --import-source on --kernel-name regex:"foreground_tc" --launch-skip 3 -c 1 -f -o gpurun_out/r2f_fg python tools/probe_r2.py fused > /dev/null 2>&1
timeout 300 ncu --set full --import-source on --kernel-name regex:"fused_fg" --launch-skip 6 -c 1 -f -o gpurun_out/r2f_fused python tools/probe_r2.py fused > /dev/null 2>&1
timeout 300 ncu --set full --import-source on --kernel-name regex:"modes_tc" --launch-skip 3 -c 1 -f -o gpurun_out/r2f_modes python tools/probe_r2.py fused > /dev/null 2>&1
timeout 300 ncu --set full --import-source on --kernel-name regex:"sketch_sparse_sorted" -c 1 -f -o gpurun_out/r2f_sketch python tools/probe_r2.py sparse > /dev/null 2>&1
echo done
