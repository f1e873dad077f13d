cd $GRAFT_REPO_ROOT
CDMD_PROFILE_FIT=1 timeout 120 python tools/probe_r2.py fit > gpurun_out/r2_probe7_fit.log 2>&1; echo "fit rc=$?" >> gpurun_out/r2_probe7_fit.log
timeout 300 ncu --set full --import-source on --kernel-name regex:"fused_fg" -c 1 -f -o gpurun_out/r2_fused7 python tools/probe_r2.py fused > gpurun_out/r2_ncu7.log 2>&1
echo done
