"""Gaussian / SRFT sketch timing (diagnostic): python tools/gauss_probe.py [config] [reps].
Times P.sketch alone with CUDA events (median), checks determinism across calls."""
import sys

import torch

sys.path.insert(0, ".")
from paper_1512_04205_b200 import cdmd as C  # noqa: E402
from synth.scene import config_by_name, video_for  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c4_1080p_gaussian"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 10
kind = sys.argv[3] if len(sys.argv) > 3 else None
cfg = config_by_name(name)
X = video_for(cfg)
m, n = X.shape
ld = ((n + 15) // 16) * 16
Xd = torch.zeros((m, ld), dtype=torch.uint8, device="cuda")
Xd[:, :n] = torch.from_numpy(X).cuda()
H = C.Handle(0)
P = C.Pipeline(H, n, n, m, kind or cfg.kind, cfg.p, cfg.k, cfg.K, seed=cfg.sensing_seed)
Y0 = P.sketch(Xd).clone()
ts = []
for _ in range(reps):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    P.sketch(Xd)
    b.record()
    torch.cuda.synchronize()
    ts.append(a.elapsed_time(b))
ts.sort()
same = bool(torch.equal(P.Y, Y0))
flops = 2.0 * cfg.p * n * m
print(f"{name} {kind or cfg.kind}: sketch ms median {ts[len(ts) // 2]:.4f} min {ts[0]:.4f} "
      f"TFLOP/s {flops / ts[len(ts) // 2] / 1e9:.1f} deterministic {same} Ysum {float(P.Y.double().abs().sum()):.6e}")
