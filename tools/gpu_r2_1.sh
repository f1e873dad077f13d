cd $GRAFT_REPO_ROOT
nproc > gpurun_out/r2_nproc.txt; free -g >> gpurun_out/r2_nproc.txt
timeout 1800 python -m pytest tests -m gpu -q -rf --durations=25 > gpurun_out/r2_pytest1.log 2>&1
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/r2_bench1.json 2> gpurun_out/r2_bench1.err
timeout 300 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r2_ref1.json 2> gpurun_out/r2_ref1.err
timeout 600 ncu --set full --import-source on --kernel-name regex:foreground_tc -c 1 -f -o gpurun_out/r2_fg1 python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --lanes 1 --graph-reps 10 > gpurun_out/r2_ncu1.log 2>&1
echo done
