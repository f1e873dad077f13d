# GPU-box script: timing of the passes, then one ncu --set full capture of the fused pass (N11)
# and of the dynamic foreground pass.
cd $GRAFT_REPO_ROOT
timeout 300 python tools/fg_time.py c4_1080p_sparse 20 > gpurun_out/fu_plain.log 2>&1 &&
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"fused_fg_kernel|foreground_tc_kernel" -s 2 -c 2 -f -o gpurun_out/fu_prof python tools/fg_time.py c4_1080p_sparse 3 > gpurun_out/fu_ncu.log 2>&1
echo done
