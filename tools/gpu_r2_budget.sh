cd $GRAFT_REPO_ROOT
for B in 0 4 8 16; do
  export CDMD_TILE_BUDGET=$B
  timeout 300 python tools/fg_time.py c4_1080p_sparse 20 > gpurun_out/bud_fg_$B.log 2>&1
  timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/bud_$B.json 2> gpurun_out/bud_$B.err
done
