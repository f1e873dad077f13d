"""Wait-time profile of the one-pass modes + foreground kernel (diagnostic; needs a
-DCDMD_FF_PROF build: CTA 0's warps print their clock64 totals per wait site)."""
import sys

import torch

sys.path.insert(0, ".")
from paper_1512_04205_b200 import cdmd as C  # noqa: E402
from synth.scene import config_by_name, video_for  # noqa: E402

cfg = config_by_name(sys.argv[1] if len(sys.argv) > 1 else "c4_1080p_sparse")
X = video_for(cfg)
m, n = X.shape
Xd = torch.from_numpy(X).cuda()
H = C.Handle(0)
P = C.Pipeline(H, n, n, m, cfg.kind, cfg.p, cfg.k, cfg.K, seed=cfg.sensing_seed)
P.run(Xd, cfg.tau, C.BG_DYNAMIC)
torch.cuda.synchronize()
P.modes_foreground(Xd, cfg.tau, C.BG_DYNAMIC)
torch.cuda.synchronize()
