cd $GRAFT_REPO_ROOT
timeout 120 python tools/probe_mismatch.py > gpurun_out/r2_mismatch.log 2>&1; echo "rc=$?" >> gpurun_out/r2_mismatch.log
timeout 300 ncu --set full --import-source on --kernel-name regex:"foreground_tc" --launch-skip 3 -c 1 -f -o gpurun_out/r2_fg11 python tools/probe_r2.py fused > gpurun_out/r2_ncu11.log 2>&1
echo done
