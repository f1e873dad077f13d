cd $GRAFT_REPO_ROOT
timeout 600 python bench.py --config c4_1080p_gaussian --steps 6 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/gauss_bench.json 2> gpurun_out/gauss_bench.err
timeout 300 ncu --set full --import-source on --kernel-name regex:"sketch_gaussian" -c 1 -f -o gpurun_out/r2g_gauss python tools/probe_r2.py gauss > gpurun_out/gauss_ncu.log 2>&1
echo done
