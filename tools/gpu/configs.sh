# GPU-box script: one quick bench line per config (regression sweep)
cd $GRAFT_REPO_ROOT
for c in c1_32x24_sparse c2_320x240_spixel c3_720x480_rademacher c4_1080p_gaussian c5_4k_sparse; do
  timeout 600 python bench.py --config $c --steps 6 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/cfg_$c.json 2> gpurun_out/cfg_$c.err
  echo "$c rc $?" >> gpurun_out/cfg_rc.log
done
