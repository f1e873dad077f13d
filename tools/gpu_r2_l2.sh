cd $GRAFT_REPO_ROOT
for G in 0 32 64; do
  if [ "$G" = "0" ]; then unset CDMD_L2_FETCH; else export CDMD_L2_FETCH=$G; fi
  echo "== L2 fetch $G" >> gpurun_out/l2.log
  timeout 200 python tools/probe_r2.py sparse >> gpurun_out/l2.log 2>&1
  timeout 300 ncu --metrics dram__bytes_read.sum,gpu__time_duration.sum --kernel-name regex:"sketch_sparse_sorted" -c 3 python tools/probe_r2.py sparse 2>&1 | grep -E "dram__bytes_read|gpu__time_duration" >> gpurun_out/l2.log
done
