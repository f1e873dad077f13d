cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -q -rf -x -k "fused or full_size or small or no_out_of or repeatable or c2 or frequency or gavish or streaming or two_rank" > gpurun_out/r2_pytest2.log 2>&1
for ew in 8 16; do
CDMD_FG_EW=$ew timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --lanes 1 > gpurun_out/r2_bench2_ew$ew.json 2> gpurun_out/r2_bench2_ew$ew.err
done
timeout 600 ncu --set full --import-source on --kernel-name regex:"foreground_tc|fused_fg" -c 2 -f -o gpurun_out/r2_fg2 python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --lanes 1 --graph-reps 10 > gpurun_out/r2_ncu2.log 2>&1
echo done
