"""Throughput of the two halves of a streaming step in isolation (diagnostics).

    python tools/throughput_probe.py [--lanes 16] [--batches 64]

passes: sketch + modes + foreground of `batches` batches round-robin over `lanes`
        streams from one host thread (each lane's model fitted once beforehand);
fits:   `batches` small solves from `lanes` host threads, nothing else running.
"""
import argparse
import concurrent.futures as cf
import os
import sys

os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")   # as bench.py
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_1512_04205_b200 import cdmd as C  # noqa: E402
from synth.scene import config_by_name, video_for  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c4_1080p_sparse")
    ap.add_argument("--lanes", type=int, default=16)
    ap.add_argument("--batches", type=int, default=64)
    a = ap.parse_args()
    cfg = config_by_name(a.config)
    X = video_for(cfg)
    m, n = X.shape
    ld = ((n + 15) // 16) * 16
    Xd = torch.zeros((m, ld), dtype=torch.uint8, device="cuda")
    Xd[:, :n] = torch.from_numpy(X).cuda()
    L = a.lanes
    lanes = []
    for _ in range(L):
        h = C.Handle(0)
        st = torch.cuda.Stream()
        with torch.cuda.stream(st):
            P = C.Pipeline(h, n, n, m, cfg.kind, cfg.p, cfg.k, cfg.K, seed=cfg.sensing_seed)
            P.run(Xd, cfg.tau)
        lanes.append((h, st, P))
    Xs = [Xd] + [Xd.clone() for _ in range(L - 1)]
    torch.cuda.synchronize()

    def passes(nb):
        for b in range(nb):
            _, st, P = lanes[b % L]
            P.sketch(Xs[b % L], st)
            P.modes(Xs[b % L], st)
            P.foreground(Xs[b % L], cfg.tau, C.BG_DYNAMIC, st)

    def fits(nb):
        def work(li):
            _, st, P = lanes[li]
            with torch.cuda.stream(st):
                for _ in range(li, nb, L):
                    P.fit(st)
        with cf.ThreadPoolExecutor(L) as ex:
            for f in [ex.submit(work, i) for i in range(L)]:
                f.result()

    for name, fn in (("passes", passes), ("fits", fits)):
        fn(L)
        torch.cuda.synchronize()
        t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0.record()
        for _, st, _ in lanes:
            st.wait_event(t0)
        fn(a.batches)
        for _, st, _ in lanes:
            ev = torch.cuda.Event()
            ev.record(st)
            torch.cuda.current_stream().wait_event(ev)
        t1.record()
        torch.cuda.synchronize()
        ms = t0.elapsed_time(t1)
        print(f"{name}: {a.batches} batches over {L} lanes: {ms:.2f} ms -> {ms / a.batches:.3f} ms/batch")


if __name__ == "__main__":
    main()
