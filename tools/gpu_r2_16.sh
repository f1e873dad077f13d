cd $GRAFT_REPO_ROOT
for d in 0 1 2; do CDMD_FU_MED_DBG=$d timeout 120 python tools/probe_r2.py fused > gpurun_out/r2_probe16_$d.log 2>&1; done
echo done
