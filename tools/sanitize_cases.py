"""Small cases of the whole hot path for compute-sanitizer (memcheck / synccheck /
initcheck / racecheck): C1 and the ragged cases (n not a multiple of 128, odd m),
every entry point of libcdmd once.  Prints "cases ok" at the end.

    compute-sanitizer --tool memcheck --kernel-regex kns=cdmd python tools/sanitize_cases.py [c1 ...]
"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_1512_04205_b200 import cdmd as C   # noqa: E402
from synth.scene import config_by_name, make_video, video_for   # noqa: E402

CASES = {
    # name: (video, kind, p, k, K)
    "c1": (lambda: video_for(config_by_name("c1_32x24_sparse")), "sparse", 50, 10, 2),
    "ragged_sparse": (lambda: make_video(100, 37, 33, seed=5, noise=2.0, n_rects=1), "sparse", 120, 12, 5),
    "ragged_spixel": (lambda: make_video(97, 61, 45, seed=6, noise=2.0, n_rects=2), "spixel", 400, 15, 6),
    "rademacher": (lambda: make_video(180, 120, 60, seed=7, noise=2.0, n_rects=2), "rademacher", 300, 20, 6),
    "gaussian": (lambda: make_video(160, 100, 50, seed=8, noise=2.0, n_rects=1), "gaussian", 256, 16, 6),
}


def run(name):
    mk, kind, p, k, K = CASES[name]
    X = mk()
    m, n = X.shape
    ld = ((n + 15) // 16) * 16
    Xd = torch.zeros((m, ld), dtype=torch.uint8, device="cuda")
    Xd[:, :n] = torch.from_numpy(X).cuda()
    H = C.Handle(0)
    P = C.Pipeline(H, n, n, m, kind, p, k, K)
    P.run(Xd, 25.0, C.BG_DYNAMIC)
    P.foreground(Xd, 25.0, C.BG_STATIC)
    if hasattr(P, "Phi"):
        try:
            P.foreground(Xd, 25.0, C.BG_DYNAMIC, fused=True)
        except TypeError:
            pass
    P.background(C.BG_DYNAMIC)
    P.amplitudes(Xd)
    if name == "c1":
        P.median3(32, 24)
        P.foreground_median3(Xd, 25.0, 32, 24)
    torch.cuda.synchronize()
    print(name, "k_eff", P.model.k_eff, "K_eff", P.model.K_eff, flush=True)


if __name__ == "__main__":
    names = sys.argv[1:] or list(CASES)
    for nm in names:
        run(nm)
    print("cases ok", flush=True)
