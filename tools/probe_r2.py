"""Quick GPU probe of new kernels (run under `timeout`): prints progress as it goes so a
hang shows where it happened.  python tools/probe_r2.py [fused] [fit] [sparse]"""
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1512_04205_b200 import cdmd as C  # noqa: E402
from synth.scene import config_by_name, make_video, video_for  # noqa: E402


def dev(X):
    m, n = X.shape
    ld = ((n + 15) // 16) * 16
    Xd = torch.zeros((m, ld), dtype=torch.uint8, device="cuda")
    Xd[:, :n] = torch.from_numpy(X).cuda()
    return Xd


def say(*a):
    print(*a, flush=True)


def probe_fused(H):
    for (W, Hh, m) in [(64, 48, 40), (180, 120, 60), (400, 300, 130), (1920, 1080, 500)]:
        X = make_video(W, Hh, m, seed=3, noise=2.0, n_rects=2)
        n = X.shape[1]
        Xd = dev(X)
        P = C.Pipeline(H, n, n, m, "sparse", min(600, n // 4), 20, 6)
        P.run(Xd, 25.0, C.BG_DYNAMIC)
        ref = P.mask.clone()
        torch.cuda.synchronize()
        say(f"fused {W}x{Hh}x{m}: n_coef={P.model.n_coef} launching", time.strftime("%X"))
        P.foreground(Xd, 25.0, C.BG_DYNAMIC, fused=True)
        torch.cuda.synchronize()
        same = float((P.mask == ref).float().mean())
        say(f"  words equal to the two-pass mask: {same:.7f}")
        ref_s = P.foreground(Xd, 25.0, C.BG_STATIC).clone()
        P.foreground(Xd, 25.0, C.BG_STATIC, fused=True)
        torch.cuda.synchronize()
        say(f"  static: words equal to the two-pass static mask: {float((P.mask == ref_s).float().mean()):.7f}")
        if W == 1920:
            ts = []
            for _ in range(10):
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record()
                P.foreground(Xd, 25.0, C.BG_DYNAMIC, fused=True)
                b.record()
                b.synchronize()
                ts.append(a.elapsed_time(b))
            t2 = []
            for _ in range(10):
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record()
                P.foreground(Xd, 25.0, C.BG_DYNAMIC)
                b.record()
                b.synchronize()
                t2.append(a.elapsed_time(b))
            say(f"  fused {np.median(ts):.4f} ms, two-pass foreground {np.median(t2):.4f} ms")
            ts = []
            for _ in range(10):
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record()
                P.foreground(Xd, 25.0, C.BG_STATIC, fused=True)
                b.record()
                b.synchronize()
                ts.append(a.elapsed_time(b))
            say(f"  fused static {np.median(ts):.4f} ms")
            ts = []
            for _ in range(10):
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record()
                P.foreground_median3(Xd, 25.0, W, Hh, C.BG_DYNAMIC)
                b.record()
                b.synchronize()
                ts.append(a.elapsed_time(b))
            say(f"  fused + median {np.median(ts):.4f} ms")


def probe_fit(H):
    from oracle import cdmd as OD
    from oracle import sensing as OS
    cfg = config_by_name("c4_1080p_sparse")
    X = video_for(cfg)
    m, n = X.shape
    Xd = dev(X)
    P = C.Pipeline(H, n, n, m, "sparse", cfg.p, cfg.k, cfg.K)
    P.sketch(Xd)
    torch.cuda.synchronize()
    say("fit launching", time.strftime("%X"))
    P.fit()
    torch.cuda.synchronize()
    say("fit done")
    ts = []
    for _ in range(5):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        P.fit()
        b.record()
        b.synchronize()
        ts.append(a.elapsed_time(b))
    say(f"fit median {np.median(ts):.3f} ms")
    gm = C.model_to_host(P.model)
    om = OD.fit(OS.sketch(X, OS.SPARSE, cfg.p, 0), cfg.k, cfg.K)
    srel = np.max(np.abs(gm["sigma"] - om["sigma"]) / om["sigma"])
    lam_err = max(min(abs(l - om["lam"])) / abs(l) for l in gm["lam"])
    say(f"k_eff {gm['k_eff']} vs {om['k_eff']}, sigma rel {srel:.2e}, lambda rel {lam_err:.2e}")
    os.environ["CDMD_PROFILE_FIT"] = "1"
    P.fit()
    torch.cuda.synchronize()


def probe_sparse(H):
    cfg = config_by_name("c4_1080p_sparse")
    X = video_for(cfg)
    m, n = X.shape
    Xd = dev(X)
    P = C.Pipeline(H, n, n, m, "sparse", cfg.p, cfg.k, cfg.K)
    say("sparse sorted launching", time.strftime("%X"))
    a = P.sketch(Xd).clone()
    torch.cuda.synchronize()
    os.environ["CDMD_SPARSE_ELL"] = "1"
    b = P.sketch(Xd).clone()
    del os.environ["CDMD_SPARSE_ELL"]
    torch.cuda.synchronize()
    say("sorted == ELL:", bool(torch.equal(a, b)))
    for name, env in (("sorted", None), ("ell", "1")):
        if env:
            os.environ["CDMD_SPARSE_ELL"] = env
        ts = []
        for _ in range(10):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            P.sketch(Xd)
            e1.record()
            e1.synchronize()
            ts.append(e0.elapsed_time(e1))
        os.environ.pop("CDMD_SPARSE_ELL", None)
        say(f"  {name}: {np.median(ts):.4f} ms")


def probe_gauss(H):
    cfg = config_by_name("c4_1080p_gaussian")
    X = video_for(cfg)
    m, n = X.shape
    Xd = dev(X)
    P = C.Pipeline(H, n, n, m, "gaussian", cfg.p, cfg.k, cfg.K)
    P.sketch(Xd)
    torch.cuda.synchronize()
    ts = []
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        P.sketch(Xd)
        e1.record()
        e1.synchronize()
        ts.append(e0.elapsed_time(e1))
    say(f"gaussian sketch {np.median(ts):.4f} ms")


if __name__ == "__main__":
    H = C.Handle(0)
    what = sys.argv[1:] or ["fused", "fit", "sparse"]
    for w in what:
        {"fused": probe_fused, "fit": probe_fit, "sparse": probe_sparse, "gauss": probe_gauss}[w](H)
    say("probe done")
