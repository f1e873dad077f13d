cd $GRAFT_REPO_ROOT
for i in 1 2; do
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/b2_$i.json 2> gpurun_out/b2_$i.err
done
