# GPU-box script: streaming throughput with a green-context SM partition for the solves
cd $GRAFT_REPO_ROOT
for F in 0 16 20 24 32; do
  timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --fit-sms $F > gpurun_out/fs_$F.json 2> gpurun_out/fs_$F.err
done
python - <<'PY' > gpurun_out/fitsms_probe.log 2>&1
import sys, torch
sys.path.insert(0, ".")
from paper_1512_04205_b200 import cdmd as C
print(C.cdmd_sm_partition(0, 20, 2))
PY
