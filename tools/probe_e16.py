"""Debug probe for the symmetric eigensolver paths (run under timeout)."""
import os
import sys
import numpy as np
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1512_04205_b200 import cdmd as C  # noqa: E402
from synth.scene import make_video  # noqa: E402
X = make_video(64, 48, int(sys.argv[1]) if len(sys.argv) > 1 else 24, seed=3, noise=2.0, n_rects=1)
m, n = X.shape
Xd = torch.zeros((m, ((n + 15) // 16) * 16), dtype=torch.uint8, device="cuda")
Xd[:, :n] = torch.from_numpy(X).cuda()
H = C.Handle(0)
P = C.Pipeline(H, n, n, m, "sparse", 200, 8, 2)
P.sketch(Xd)
torch.cuda.synchronize()
print("fit start", flush=True)
P.fit()
torch.cuda.synchronize()
from oracle import cdmd as OD, sensing as OS
om = OD.fit(OS.sketch(X, OS.SPARSE, 200, 0), 8, 2)
gm = C.model_to_host(P.model)
print("sigma", gm["sigma"][:4], om["sigma"][:4], flush=True)
print("fit ok", flush=True)
