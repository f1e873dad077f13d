"""Where do the fused (N11) and two-pass masks differ at the bench size?"""
import os
import sys
import numpy as np
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1512_04205_b200 import cdmd as C  # noqa: E402
from synth.scene import make_video  # noqa: E402
X = make_video(1920, 1080, 500, seed=3, noise=2.0, n_rects=2)
m, n = X.shape
Xd = torch.zeros((m, n), dtype=torch.uint8, device="cuda")
Xd.copy_(torch.from_numpy(X))
H = C.Handle(0)
P = C.Pipeline(H, n, n, m, "sparse", 600, 20, 6)
P.run(Xd, 25.0, C.BG_DYNAMIC)
for mode, name in ((C.BG_DYNAMIC, "dyn"), (C.BG_STATIC, "sta")):
    a = P.foreground(Xd, 25.0, mode).clone()
    reps = []
    for r in range(3):
        reps.append(P.foreground(Xd, 25.0, mode, fused=True).clone())
    torch.cuda.synchronize()
    for r, b in enumerate(reps):
        diff = (a != b).nonzero().cpu().numpy()
        print(name, "rep", r, "differing words", len(diff), diff[:5].tolist(), flush=True)
        for t, w in diff[:3]:
            print("   two-pass %08x fused %08x" % (a[t, w].item() & 0xffffffff, b[t, w].item() & 0xffffffff), flush=True)
    print(name, "fused reps identical:", all(torch.equal(reps[0], x) for x in reps[1:]), flush=True)
