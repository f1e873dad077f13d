cd $GRAFT_REPO_ROOT
for R in 0 16 20 32; do
for L in 10 16; do
CDMD_PERSIST_RESERVE=$R timeout 300 python bench.py --steps 32 --warmup 5 --lanes $L --no-cpu-baseline --no-e2e > gpurun_out/sw_${R}_${L}.json 2> gpurun_out/sw_${R}_${L}.err
python - <<PY
import json
d=json.load(open("gpurun_out/sw_${R}_${L}.json"))
print("R=${R} L=${L}", d["value"], d["ms_per_step"], d["streaming"].get("fused_ms_per_batch"), d["stage_ms"]["fit"])
PY
done
done > gpurun_out/sweep.txt 2>&1
timeout 300 python tools/stream_timeline.py --lanes 10 --batches 40 > gpurun_out/timeline.txt 2>&1
echo done
