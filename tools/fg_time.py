"""Foreground / fused pass timing on a config (diagnostic): python tools/fg_time.py [config] [reps]
Prints median CUDA-event times of the foreground (dynamic), the fused pass and modes, and a
checksum of the mask (to compare builds)."""
import sys
import zlib

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_1512_04205_b200 import cdmd as C  # noqa: E402
from synth.scene import config_by_name, video_for  # noqa: E402


def med(fn, reps):
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        b.synchronize()
        ts.append(a.elapsed_time(b))
    return float(np.median(ts))


name = sys.argv[1] if len(sys.argv) > 1 else "c4_1080p_sparse"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 20
cfg = config_by_name(name)
X = video_for(cfg)
m, n = X.shape
ld = ((n + 15) // 16) * 16
Xd = torch.zeros((m, ld), dtype=torch.uint8, device="cuda")
Xd[:, :n] = torch.from_numpy(X).cuda()
H = C.Handle(0)
P = C.Pipeline(H, n, n, m, cfg.kind, cfg.p, cfg.k, cfg.K, seed=cfg.sensing_seed)
P.sketch(Xd)
P.fit()
P.modes(Xd)
P.foreground(Xd, cfg.tau, C.BG_DYNAMIC)
torch.cuda.synchronize()
crc = zlib.crc32(P.mask.cpu().numpy().tobytes())
t_fg = med(lambda: P.foreground(Xd, cfg.tau, C.BG_DYNAMIC), reps)
t_md = med(lambda: P.modes(Xd), reps)
t_fu = med(lambda: P.foreground(Xd, cfg.tau, C.BG_DYNAMIC, fused=True), reps)
gb = (n * m + n * m / 8) / 1e9
print(f"{name}: foreground {t_fg:.4f} ms ({gb / t_fg * 1e3:.0f} GB/s)  modes {t_md:.4f} ms  fused {t_fu:.4f} ms  "
      f"mask crc {crc:08x}")
