# GPU-box script (run via gpurun from the repo root): the bench's kernel launch list and
# ncu captures of the small solve's two longest kernels (Lanczos, Francis QR).
cd $GRAFT_REPO_ROOT
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 700 --csv --log-file gpurun_out/r2p_launches.csv python bench.py --steps 2 --warmup 3 --lanes 1 --no-cpu-baseline --no-e2e --graph-reps 10 > gpurun_out/r2p_ncu_launch.log 2>&1
timeout 300 ncu --set full --import-source on --kernel-name regex:"lz_kernel" -c 1 -f -o gpurun_out/r2p_lz python tools/probe_fit.py c4_1080p_sparse 1 > /dev/null 2>&1
timeout 300 ncu --set full --import-source on --kernel-name regex:"hqrv_kernel" -c 1 -f -o gpurun_out/r2p_hqr python tools/probe_fit.py c4_1080p_sparse 1 > /dev/null 2>&1
echo done
