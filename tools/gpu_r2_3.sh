cd $GRAFT_REPO_ROOT
timeout 120 python tools/probe_r2.py sparse > gpurun_out/r2_probe3_sparse.log 2>&1; echo "sparse rc=$?" >> gpurun_out/r2_probe3_sparse.log
timeout 120 python tools/probe_r2.py fit > gpurun_out/r2_probe3_fit.log 2>&1; echo "fit rc=$?" >> gpurun_out/r2_probe3_fit.log
timeout 120 python tools/probe_r2.py fused > gpurun_out/r2_probe3_fused.log 2>&1; echo "fused rc=$?" >> gpurun_out/r2_probe3_fused.log
echo done
