cd $GRAFT_REPO_ROOT
timeout 120 python tools/probe_r2.py fused > gpurun_out/r2_probe10_fused.log 2>&1; echo "fused rc=$?" >> gpurun_out/r2_probe10_fused.log
CDMD_PROFILE_FIT=1 timeout 120 python tools/probe_r2.py fit > gpurun_out/r2_probe10_fit.log 2>&1; echo "fit rc=$?" >> gpurun_out/r2_probe10_fit.log
timeout 300 ncu --set full --import-source on --kernel-name regex:"fused_fg" --launch-skip 6 -c 1 -f -o gpurun_out/r2_fused10 python tools/probe_r2.py fused > gpurun_out/r2_ncu10.log 2>&1
echo done
