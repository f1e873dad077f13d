"""Per-lane stage timeline of the streaming driver (diagnostics, not a benchmark).

    python tools/stream_timeline.py [--lanes 8] [--batches 48]

Records CUDA events around every stage of every batch and prints, per stage, the
mean device duration under load and the mean gap a lane waits between stages.
"""
import argparse
import os
import sys

import numpy as np
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")   # as bench.py
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_1512_04205_b200 import cdmd as C  # noqa: E402
from synth.scene import config_by_name, video_for  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c4_1080p_sparse")
    ap.add_argument("--lanes", type=int, default=8)
    ap.add_argument("--batches", type=int, default=48)
    ap.add_argument("--fit-sms", type=int, default=0)
    a = ap.parse_args()
    cfg = config_by_name(a.config)
    X = video_for(cfg)
    m, n = X.shape
    ld = ((n + 15) // 16) * 16
    Xd = torch.zeros((m, ld), dtype=torch.uint8, device="cuda")
    Xd[:, :n] = torch.from_numpy(X).cuda()
    S = C.Streaming(0, n, n, m, cfg.kind, cfg.p, cfg.k, cfg.K, lanes=a.lanes, seed=cfg.sensing_seed,
                    fit_sms=a.fit_sms)
    Xs = [Xd] + [Xd.clone() for _ in range(a.lanes - 1)]
    ev = {}

    orig = {name: getattr(C.Pipeline, name) for name in ("sketch", "fit", "modes", "foreground")}

    def wrap(name):
        def f(self, *args, **kw):
            st = kw.get("stream") if "stream" in kw else (args[-1] if args else None)
            if name == "foreground":
                st = args[3] if len(args) > 3 else kw.get("stream")
            elif name in ("sketch", "modes"):
                st = args[1] if len(args) > 1 else kw.get("stream")
            else:
                st = args[0] if args else kw.get("stream")
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            r = orig[name](self, *args, **kw)
            e1.record(st)
            ev.setdefault((id(self), name), []).append((e0, e1))
            return r
        return f

    start = torch.cuda.Event(enable_timing=True)
    S.run([Xs[b % a.lanes] for b in range(2 * a.lanes)], cfg.tau)   # warm-up
    torch.cuda.synchronize()
    for name in orig:
        setattr(C.Pipeline, name, wrap(name))
    start.record()
    ends = S.run([Xs[b % a.lanes] for b in range(a.batches)], cfg.tau, start_event=start)
    for e in ends:
        torch.cuda.current_stream().wait_event(e)
    stop = torch.cuda.Event(enable_timing=True)
    stop.record()
    torch.cuda.synchronize()
    total = start.elapsed_time(stop)
    print(f"{a.batches} batches, {a.lanes} lanes: {total:.2f} ms -> {total / a.batches:.3f} ms/batch")
    dur = {}
    gaps = []
    for (pid, name), lst in ev.items():
        for e0, e1 in lst:
            dur.setdefault(name, []).append(e0.elapsed_time(e1))
    for name in ("sketch", "fit", "modes", "foreground"):
        d = np.array(dur[name])
        print(f"  {name:10s} under load: mean {d.mean():7.3f} ms  min {d.min():7.3f}  max {d.max():7.3f}")
    # per-lane: time from foreground end to next sketch start (lane idle / host gap)
    pids = sorted({pid for pid, _ in ev})
    for pid in pids[:2]:
        sk = ev[(pid, "sketch")]
        fg = ev[(pid, "foreground")]
        g = [sk[i + 1][0].elapsed_time(fg[i][1]) * -1 for i in range(len(fg) - 1)]
        gaps += g
    if gaps:
        print(f"  fg end -> next sketch start (lanes 0-1): mean {np.mean(gaps):.3f} ms")


if __name__ == "__main__":
    main()
