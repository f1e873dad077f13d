# GPU-box script: foreground ablations (build with -DCDMD_ABLATIONS): 0 full, 1 no mask
# arithmetic (TMEM/X loads kept), 2 no MMAs, 3 neither
cd $GRAFT_REPO_ROOT
for D in 0 1 2 3; do
  echo "dbg=$D" >> gpurun_out/fg_ablate.log
  CDMD_FG_DBG=$D timeout 300 python tools/fg_time.py c4_1080p_sparse 20 >> gpurun_out/fg_ablate.log 2>&1
done
