"""Time the full-state amplitudes b = lstsq(Phi, x_1) (Alg. 1 step 9) at the
bench's c4 shape (1920x1080x500, sparse p=2000, k=50): the Gram pass over Phi and
the fp64 Cholesky solve, CUDA events on the launching stream, after warm-up.
Algorithmic bytes of the Gram pass: n k 4 (folded fp32 Phi) + n (x_1)."""
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1512_04205_b200 import cdmd as C  # noqa: E402
from synth.scene import config_by_name, video_for  # noqa: E402


def main():
    cfg = config_by_name("c4_1080p_sparse")
    X = torch.from_numpy(video_for(cfg)).cuda()
    m, n = X.shape
    H = C.Handle(0)
    P = C.Pipeline(H, n, n, m, cfg.kind, cfg.p, cfg.k, cfg.K)
    P.sketch(X)
    P.fit()
    P.modes(X)
    ke = P.model.k_eff
    v = C.video(X, n, 0, n)
    ws = torch.empty(C.cdmd_amplitudes_workspace_bytes(H, ke), dtype=torch.uint8, device="cuda")
    G = torch.empty((ke + 1, ke), dtype=torch.float64, device="cuda")
    b = torch.empty((ke, 2), dtype=torch.float64, device="cuda")
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    st = torch.cuda.current_stream()
    for _ in range(3):
        C.cdmd_amplitudes_gram(H, v, P.model, P.Phi, G, ws)
        C.cdmd_amplitudes_solve(H, P.model, G, b)
    torch.cuda.synchronize()
    reps, tg, ts = 10, 0.0, 0.0
    for _ in range(reps):
        flush.zero_()
        e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
        e0.record(st)
        C.cdmd_amplitudes_gram(H, v, P.model, P.Phi, G, ws)
        e1.record(st)
        C.cdmd_amplitudes_solve(H, P.model, G, b)
        e2.record(st)
        torch.cuda.synchronize()
        tg += e0.elapsed_time(e1) / reps
        ts += e1.elapsed_time(e2) / reps
    algo = n * ke * 4 + n
    peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    hbm = float(peaks["hbm_gbs"])
    out = dict(workload="c4_1080p_sparse", k_eff=ke, gram_ms=round(tg, 4), solve_ms=round(ts, 4),
               gram_GBps=round(algo / tg / 1e6, 1), hbm_peak_GBps=hbm, gram_frac=round(algo / tg / 1e6 / hbm, 4),
               algorithmic_bytes=algo)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
