# GPU-box script: a quick default bench line (no CPU baseline / e2e)
cd $GRAFT_REPO_ROOT
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/bq.json 2> gpurun_out/bq.err
