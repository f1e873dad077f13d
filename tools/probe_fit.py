"""Fit timing on a config's sketch (diagnostic): python tools/probe_fit.py [config] [reps].
Set CDMD_PROFILE_FIT=1 for the per-stage event times, CDMD_SYEV to pick the eigensolver."""
import sys
import time

import torch

sys.path.insert(0, ".")
from paper_1512_04205_b200 import cdmd as C  # noqa: E402
from synth.scene import config_by_name, video_for  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c4_1080p_sparse"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
cfg = config_by_name(name)
X = video_for(cfg)
m, n = X.shape
ld = ((n + 15) // 16) * 16
Xd = torch.zeros((m, ld), dtype=torch.uint8, device="cuda")
Xd[:, :n] = torch.from_numpy(X).cuda()
H = C.Handle(0)
P = C.Pipeline(H, n, n, m, cfg.kind, cfg.p, cfg.k, cfg.K, seed=cfg.sensing_seed)
P.sketch(Xd)
ts = []
for r in range(reps):
    torch.cuda.synchronize()
    a = time.perf_counter()
    P.fit()
    torch.cuda.synchronize()
    ts.append((time.perf_counter() - a) * 1e3)
print(name, "fit ms", " ".join(f"{t:.3f}" for t in ts), "eigensolver stats", C.cdmd_eigensolver_stats(H),
      "sigma[0], sigma[-1]", C.model_to_host(P.model)["sigma"][[0, -1]])
