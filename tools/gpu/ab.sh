# GPU-box script: A/B of library variants in paper_1512_04205_b200/lib/variants/*.so —
# the Gaussian sketch, modes / foreground / fused pass, the c4 fit, a short bench.
cd $GRAFT_REPO_ROOT
L=paper_1512_04205_b200/lib
cp $L/libcdmd.so /tmp/libcdmd.keep
for v in ${@:-$(ls $L/variants | sed 's/\.so$//')}; do
  cp $L/variants/$v.so $L/libcdmd.so
  {
    echo "=== $v"
    timeout 200 python tools/gauss_probe.py c4_1080p_gaussian 10
    timeout 200 python tools/fg_time.py c4_1080p_sparse 20
    CDMD_PROFILE_FIT=0 timeout 200 python tools/probe_fit.py c4_1080p_sparse 8
    timeout 400 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --graph-reps 10 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('bench value', d['value'], 'stage', d['stage_ms'], 'per_batch', d['per_batch']['ms_median'], 'passes', d['passes_only']['ms_median'], 'fused_stream', d['streaming'].get('fused_frames_per_s'))"
  } >> gpurun_out/ab.log 2>&1
done
cp /tmp/libcdmd.keep $L/libcdmd.so
echo done
