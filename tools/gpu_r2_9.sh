cd $GRAFT_REPO_ROOT
timeout 300 ncu --set full --import-source on --kernel-name regex:"fused_fg" --launch-skip 3 -c 1 -f -o gpurun_out/r2_fused9 python tools/probe_r2.py fused > gpurun_out/r2_ncu9.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q -rf --durations=15 > gpurun_out/r2_pytest9.log 2>&1
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/r2_bench9.json 2> gpurun_out/r2_bench9.err
echo done
