#!/usr/bin/env python
"""Throughput benchmark of the cDMD hot path on B200 (BASELINE.json metric).

metric : "1080p frames/sec (sketch+modes+fg mask) at 1/2/4/8 B200; % of HBM roofline"
step   : one pass of the whole hot path over one batch:
         cdmd_sketch -> all_reduce(Y) -> cdmd_fit -> cdmd_modes -> cdmd_foreground
workload (N=1): c4_1080p_sparse = 1920x1080, m = 500 frames, sparse C (s = n/ln n),
         p = 2000, k = 50, K = 10, tau = 25, dynamic background (north_star (3)).
value  : frames / device time per step (max over ranks), inputs resident in HBM;
         X (1.04 GB) is larger than L2, so no flush is needed between steps.
         Streaming (default): K batches flow through `lanes` lanes (own handle, CUDA
         stream, buffers and copy of X), so one batch's latency-bound small solve
         overlaps other batches' HBM passes -- the paper's batch decomposition of a long
         video.  lanes <= K/2, so every lane runs >= 2 batches (steady state).
Also reported:
  latency_ms_per_batch  one batch at a time, eager, with per-stage CUDA events;
  per_batch             one batch at a time, the whole step (sketch + fit + modes +
                        foreground) replayed from ONE CUDA graph (cdmd_fit reads nothing back
                        under capture; the replays' self-check flag is verified), median of
                        >= 10 runs; eager_fit_ms_median: the same with the fit eager;
  passes_only           sketch + modes + foreground in one CUDA graph (the replicated
                        small solve excluded), median of >= 10 runs, with its HBM fraction;
  e2e_fused             the same with the fused single pass (N11: cdmd_foreground(Phi=NULL)).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config NAME] [--bg dynamic|static]
    python -m torch.distributed.run --nproc-per-node N --master-addr 127.0.0.1 bench.py --gpus N
    python bench.py --impl reference     # the CPU oracle (test infrastructure) as the baseline arm
"""

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

# Streaming runs 2 streams per lane.  With the default 8 hardware work queues, streams
# share queues and a lane's queued solve kernel blocks unrelated streams behind it
# (measured: 16 concurrent solves 0.79 -> 0.51 ms/batch with 32).  Must be set before
# the CUDA context exists.
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

FALLBACK_HBM_GBS = 6650.0   # B200_PROFILING.md fallback, used only without MEASURED_PEAKS.json
FALLBACK_BF16_TFLOPS = 1590.0
METRIC = "1080p frames/sec (sketch+modes+fg mask) at 1/2/4/8 B200; % of HBM roofline"
KINDS = {"spixel": 0, "sparse": 1, "rademacher": 2, "gaussian": 3, "srft": 4}


def peaks():
    """(HBM GB/s, dense bf16 TFLOP/s burst, source): MEASURED_PEAKS.json, else the recipe's fallback."""
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d["hbm_gbs"]), float(d["bf16_tflops"]), "measured"
    return FALLBACK_HBM_GBS, FALLBACK_BF16_TFLOPS, "fallback"


def int8_peak_tops(torch):
    """Dense int8 tensor-core peak measured here: torch._int_mm (cuBLASLt int8 GEMM,
    tcgen05 kind::i8 on sm_100a) 8192^3, 2 N^3 ops, best of 10 (burst)."""
    try:
        a = torch.randint(-128, 127, (8192, 8192), dtype=torch.int8, device="cuda")
        b = torch.randint(-128, 127, (8192, 8192), dtype=torch.int8, device="cuda").t()
        for _ in range(3):
            torch._int_mm(a, b)
        best = 1e30
        for _ in range(10):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            torch._int_mm(a, b)
            e1.record()
            torch.cuda.synchronize()
            best = min(best, e0.elapsed_time(e1))
        del a, b
        return 2 * 8192 ** 3 / (best * 1e-3) / 1e12
    except Exception:
        return None


class ClockSampler:
    """nvidia-smi samples of SM clock and throttle reasons during the timed region."""
    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu):
        self.gpu, self.rows, self.proc = gpu, [], None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def __exit__(self, *a):
        if self.proc:
            time.sleep(0.25)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        rows = [r for r in self.rows if len(r) == 6 and r[0].isdigit()]
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[2 + i].lower().startswith("active")})
        return {"sm_mhz": statistics.median(float(r[0]) for r in rows),
                "sm_max_mhz": max(float(r[1]) for r in rows), "reasons": reasons, "samples": len(rows)}


def sector_bytes_sparse(n_local, pix0, n_total, p, seed, m):
    """Algorithmic bytes of the sparse sketch: distinct 32-B sectors of X gathered per
    frame x m frames (the sector is the HBM access granule) + the p x m int32 Y."""
    from oracle.sensing import default_s, sparse_rows   # counting only; not on the timed path
    rows = sparse_rows(n_total, p, default_s(n_total), seed)
    pos = np.concatenate([r[0] for r in rows])
    pos = pos[(pos >= pix0) & (pos < pix0 + n_local)] - pix0
    return int(np.unique(pos // 32).size) * 32 * m + 4 * p * m


# ------------------------------------------------------------- the oracle as a baseline
class OracleStep:
    """One step of the oracle (test infrastructure) on the whole workload, on this
    host's cores: the sketch and the fit in this process, then modes + background +
    mask of EVERY pixel, the oracle's own per-pixel functions fanned over pixel slabs in
    worker processes (oracle/runner.py; no arithmetic of its own).  Dense sensings
    (Rademacher / Gaussian) sketch in the workers as well (slabs sum to Y)."""

    def __init__(self, cfg, bg):
        from oracle.runner import PixelPool
        from synth.scene import video_for
        self.cfg, self.dynamic = cfg, bg == "dynamic"
        self.kind = KINDS[cfg.kind]
        self.X = video_for(cfg) if self.kind in (0, 1) else None
        self.pool = PixelPool(cfg)
        self.cores = len(os.sched_getaffinity(0))

    def step(self):
        from oracle import cdmd as OD
        from oracle import sensing as OS
        from oracle.runner import parallel_sketch
        cfg = self.cfg
        t0 = time.perf_counter()
        if self.X is not None:
            Y = OS.sketch(self.X, self.kind, cfg.p, cfg.sensing_seed)
        else:
            Y = parallel_sketch(cfg, self.kind)
        t1 = time.perf_counter()
        model = OD.fit(Y, cfg.k, cfg.K)
        t2 = time.perf_counter()
        self.pool.run(model, cfg.tau, dynamic=self.dynamic)
        t3 = time.perf_counter()
        return t3 - t0, {"sketch_s": round(t1 - t0, 3), "fit_s": round(t2 - t1, 3), "pixels_s": round(t3 - t2, 3)}

    def close(self):
        self.pool.close()


def run_reference(args):
    """--impl reference: the oracle as it stands, timed over --warmup + --steps full
    steps of the same workload on this host's cores (rank 0 only)."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from synth.scene import config_by_name
    cfg = config_by_name(args.config)
    o = OracleStep(cfg, args.bg)
    try:
        for _ in range(args.warmup):
            o.step()
        times, parts = [], None
        for _ in range(args.steps):
            t, parts = o.step()
            times.append(t)
    finally:
        o.close()
    t = sum(times) / len(times)
    val = cfg.m / t
    line = {
        "impl": "reference", "metric": METRIC, "value": round(val, 3), "unit": "frames/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(t * 1e3, 1), "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": cfg.name, "video": f"{cfg.width}x{cfg.height}x{cfg.m}", "sensing": cfg.kind,
                   "p": cfg.p, "k": cfg.k, "K": cfg.K, "tau": cfg.tau, "background": args.bg},
        "cpu_baseline": {"value": round(val, 3), "unit": "frames/s", "cores": o.cores, "kind": "oracle",
                         "sample": f"the whole workload every step (no extrapolation): sketch + fit in one "
                                   f"process, modes+background+mask of all {cfg.n} px over {o.pool.cores} "
                                   f"worker processes; last step {parts}"},
        "e2e": {"value": round(val, 3), "unit": "frames/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def cpu_baseline(cfg, args):
    """The oracle as it stands, one full step of the workload (about 10-30 s of CPU work
    on the box's cores), after one untimed step."""
    o = OracleStep(cfg, args.bg)
    try:
        o.step()
        t, parts = o.step()
    finally:
        o.close()
    return {"value": round(cfg.m / t, 3), "unit": "frames/s", "cores": o.cores, "kind": "oracle",
            "sample": f"{cfg.name}: one whole step, no extrapolation ({parts}; pixels over "
                      f"{o.pool.cores} worker processes)"}


# --------------------------------------------------------------------------- helpers
def median_ms(torch, fn, reps, stream):
    """Median over `reps` runs of fn() timed with CUDA events on `stream`."""
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        fn()
        b.record(stream)
        b.synchronize()
        ts.append(a.elapsed_time(b))
    return statistics.median(ts), ts


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="cdmd", choices=["cdmd", "reference"])
    ap.add_argument("--config", default="c4_1080p_sparse")
    ap.add_argument("--bg", default="dynamic", choices=["dynamic", "static"])
    ap.add_argument("--rank", default="fixed", choices=["fixed", "gd"],
                    help="target rank: the config's k, or Gavish-Donoho (Remark 2, P:361) with k as the cap")
    ap.add_argument("--partition", default="pixel", choices=["pixel", "batch"],
                    help="N > 1: pixel-row slabs + all-reduce of Y (north_star), or batch-parallel "
                         "replicas (P:573; whole frames per rank, no collective)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--lanes", type=int, default=16,
                    help="batches in flight (streaming, P:573), capped at steps/2; 1 = one batch at a time")
    ap.add_argument("--fused", action="store_true",
                    help="streaming value through the fused single pass (N11) instead of modes + foreground")
    ap.add_argument("--graph-reps", type=int, default=20)
    ap.add_argument("--fit-sms", type=int, default=0,
                    help="streaming: SMs reserved for the small solves (green-context partition; 0 = shared)")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)

    import torch
    import torch.distributed as dist

    from paper_1512_04205_b200 import cdmd as C
    from paper_1512_04205_b200.dist import slab
    from synth.scene import config_by_name, video_for

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # CDMD_DIST_BACKEND=gloo (with more ranks than GPUs: ranks share devices) is only for
    # exercising the multi-rank code path on a one-GPU box; its numbers mean nothing
    backend = os.environ.get("CDMD_DIST_BACKEND", "nccl")
    if backend != "nccl":
        local = local % torch.cuda.device_count()
    torch.cuda.set_device(local)
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    cfg = config_by_name(args.config)
    n, m = cfg.n, cfg.m
    pixel = world > 1 and args.partition == "pixel"
    pix0, nl = slab(n, world, rank) if pixel else (0, n)
    X_host = video_for(cfg, pix0=pix0, n_local=nl)
    ld = ((nl + 15) // 16) * 16
    Xd = torch.zeros((m, ld), dtype=torch.uint8, device="cuda")
    Xd[:, :nl] = torch.from_numpy(X_host).cuda()
    H = C.Handle(local)
    P = C.Pipeline(H, n, nl, m, cfg.kind, cfg.p, cfg.k, cfg.K, seed=cfg.sensing_seed, pix0=pix0, rank=args.rank)
    mode = C.BG_DYNAMIC if args.bg == "dynamic" else C.BG_STATIC
    stream = torch.cuda.current_stream()
    allreduce = (lambda Y: dist.all_reduce(Y, op=dist.ReduceOp.SUM)) if pixel else None
    ev = {s: [] for s in ("sketch", "allreduce", "fit", "modes", "foreground")}

    def step(record=False):
        marks = [torch.cuda.Event(enable_timing=True) for _ in range(6)] if record else None
        if record:
            marks[0].record(stream)
        P.sketch(Xd)
        if record:
            marks[1].record(stream)
        if allreduce is not None:
            allreduce(P.Y)
        if record:
            marks[2].record(stream)
        P.fit()
        if record:
            marks[3].record(stream)
        P.modes(Xd)
        if record:
            marks[4].record(stream)
        P.foreground(Xd, cfg.tau, mode)
        if record:
            marks[5].record(stream)
            for i, s in enumerate(ev):
                ev[s].append((marks[i], marks[i + 1]))

    # ---- 1. one batch at a time, eager, per-stage events
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    start, stop = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        n0 = C.cdmd_kernel_launches()
        start.record(stream)
        for _ in range(args.steps):
            step(record=True)
        stop.record(stream)
        launches = C.cdmd_kernel_launches() - n0
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()

    def max_over_ranks(x):
        t = torch.tensor([x], dtype=torch.float64, device="cuda")
        if world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    latency_ms = max_over_ranks(start.elapsed_time(stop) / args.steps)
    stage_ms = {s: sum(a.elapsed_time(b) for a, b in v) / len(v) for s, v in ev.items()}
    ms_max, value, launches_seq = latency_ms, m / (latency_ms * 1e-3), launches
    hbm, bf16, peak_src = peaks()
    step_bytes = nl * m + nl * m // 8          # X read once + the bit mask (north_star)

    # ---- 2. CUDA graphs: passes captured, the fit eager between replays
    graphs = {}
    s_cap = torch.cuda.Stream()
    s_cap.wait_stream(stream)

    def capture(fn):
        g = torch.cuda.CUDAGraph()
        with torch.cuda.stream(s_cap):
            fn()                                   # warm (outside the capture)
            torch.cuda.synchronize()
            with torch.cuda.graph(g, stream=s_cap):
                fn()
        torch.cuda.synchronize()
        return g

    try:
        graphs["sketch"] = capture(lambda: P.sketch(Xd))
        graphs["passes_mf"] = capture(lambda: (P.modes(Xd), P.foreground(Xd, cfg.tau, mode)))
        graphs["passes_all"] = capture(lambda: (P.sketch(Xd), P.modes(Xd), P.foreground(Xd, cfg.tau, mode)))
    except Exception as e:   # report, do not hide: the eager numbers above still stand
        graphs = {"error": repr(e)}
    step_graph_err = None
    if "error" not in graphs and allreduce is None:
        try:   # the whole step in one graph: cdmd_fit has no host read-back under capture
            graphs["step"] = capture(lambda: (P.sketch(Xd), P.fit(), P.modes(Xd), P.foreground(Xd, cfg.tau, mode)))
        except Exception as e:
            step_graph_err = repr(e)
    fused_ok = True
    try:
        P.foreground(Xd, cfg.tau, mode, fused=True)
        torch.cuda.synchronize()
        if "error" not in graphs:
            graphs["passes_fused"] = capture(lambda: (P.sketch(Xd), P.foreground(Xd, cfg.tau, mode, fused=True)))
            graphs["fg_fused"] = capture(lambda: P.foreground(Xd, cfg.tau, mode, fused=True))
    except Exception as e:
        fused_ok = repr(e)
    reps = max(10, args.graph_reps)
    per_batch = passes_only = e2e_fused = None
    if "error" not in graphs:
        def one_batch():
            graphs["sketch"].replay()
            if allreduce is not None:
                with torch.cuda.stream(s_cap):
                    allreduce(P.Y)
            with torch.cuda.stream(s_cap):
                P.fit()
            graphs["passes_mf"].replay()

        with torch.cuda.stream(s_cap):
            for _ in range(3):
                one_batch()
            med, _ = median_ms(torch, one_batch, reps, s_cap)
            med = max_over_ranks(med)
            per_batch = {"ms_median": round(med, 4), "frames_per_s": round(m / (med * 1e-3), 1), "runs": reps,
                         "mode": "sketch graph | fit (eager: it reads the model sizes back once) | "
                                 "modes+foreground graph"}
            if "step" in graphs:
                for _ in range(3):
                    graphs["step"].replay()
                gmed, _ = median_ms(torch, graphs["step"].replay, reps, s_cap)
                torch.cuda.synchronize()
                if not P.graph_stale():   # the replays' self-check (sizes as captured, no fallback)
                    gmed = max_over_ranks(gmed)
                    per_batch = {"ms_median": round(gmed, 4), "frames_per_s": round(m / (gmed * 1e-3), 1),
                                 "runs": reps, "mode": "one CUDA graph: sketch + fit + modes + foreground",
                                 "eager_fit_ms_median": per_batch["ms_median"]}
                else:
                    per_batch["step_graph"] = "stale: a replay disagreed with the captured sizes"
            elif step_graph_err:
                per_batch["step_graph"] = step_graph_err
            for _ in range(3):
                graphs["passes_all"].replay()
            med, _ = median_ms(torch, graphs["passes_all"].replay, reps, s_cap)
            med = max_over_ranks(med)
            passes_only = {"ms_median": round(med, 4), "frames_per_s": round(m / (med * 1e-3), 1), "runs": reps,
                           "step_hbm_frac": round(step_bytes / (med * 1e-3) / 1e9 / hbm, 4),
                           "graph": "sketch + modes + foreground (fit excluded: the replicated small solve)"}
            if "passes_fused" in graphs:
                for _ in range(3):
                    graphs["passes_fused"].replay()
                med, _ = median_ms(torch, graphs["passes_fused"].replay, reps, s_cap)
                med = max_over_ranks(med)
                fmed, _ = median_ms(torch, graphs["fg_fused"].replay, reps, s_cap)
                fmed = max_over_ranks(fmed)
                fg_bytes = nl * m + 4 * m * ((nl + 31) // 32)
                e2e_fused = {"passes_ms_median": round(med, 4), "passes_frames_per_s": round(m / (med * 1e-3), 1),
                             "step_hbm_frac": round(step_bytes / (med * 1e-3) / 1e9 / hbm, 4),
                             "fused_kernel_ms": round(fmed, 4),
                             "fused_kernel_hbm_frac": round(fg_bytes / (fmed * 1e-3) / 1e9 / hbm, 4),
                             "graph": "sketch + fused foreground (N11: the support's modes in-slab, no Phi "
                                      "written; fit excluded)"}
        torch.cuda.synchronize()

    # ---- 3. streaming (the value): lanes reused, steady state
    streaming = None
    lanes = max(1, min(args.lanes, args.steps // 2))
    if args.lanes > 1 and lanes > 1:
        S = C.Streaming(local, n, nl, m, cfg.kind, cfg.p, cfg.k, cfg.K, lanes=lanes, seed=cfg.sensing_seed,
                        pix0=pix0, rank=args.rank, fit_sms=args.fit_sms, fused=args.fused and fused_ok is True)
        Xs = [Xd] + [Xd.clone() for _ in range(lanes - 1)]

        def stream_run(nb):
            a = torch.cuda.Event(enable_timing=True)
            a.record(stream)
            ends = S.run([Xs[b % lanes] for b in range(nb)], cfg.tau, mode, allreduce=allreduce, start_event=a)
            for e in ends:
                stream.wait_event(e)
            b_ = torch.cuda.Event(enable_timing=True)
            b_.record(stream)
            return a, b_

        stream_run(max(args.warmup, lanes))
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        with ClockSampler(local) as clk:
            n0 = C.cdmd_kernel_launches()
            a, b_ = stream_run(args.steps)
            torch.cuda.synchronize()
            launches = C.cdmd_kernel_launches() - n0
        if world > 1:
            dist.barrier()
        ms_max = max_over_ranks(a.elapsed_time(b_) / args.steps)
        value = m / (ms_max * 1e-3)
        streaming = {"lanes": lanes, "batches": args.steps, "ms_per_batch": round(ms_max, 4),
                     "sm_partition": S.sms, "fused": S.fused,
                     "step_hbm_frac": round(step_bytes / (ms_max * 1e-3) / 1e9 / hbm, 4),
                     "note": "batches pipelined across lanes (own handle, stream, buffers, copy of X); "
                             "each lane runs >= 2 batches"}
        # the same lanes through the fused single pass (N11: no cdmd_modes; the support's
        # modes in-slab) -- the E2E-fused variant of SURVEY.md §8(d), reported alongside
        if fused_ok is True and not args.fused:
            S.fused = True
            stream_run(max(args.warmup, lanes))
            torch.cuda.synchronize()
            if world > 1:
                dist.barrier()
            a2, b2 = stream_run(args.steps)
            torch.cuda.synchronize()
            S.fused = False
            msf = max_over_ranks(a2.elapsed_time(b2) / args.steps)
            streaming["fused_ms_per_batch"] = round(msf, 4)
            streaming["fused_frames_per_s"] = round(m / (msf * 1e-3) * (world if not pixel and world > 1 else 1), 1)
    if not pixel and world > 1:
        value *= world      # batch-parallel replicas: every rank processes its own batches

    # ---- roofline of the dominant kernel: HBM-bound passes (algorithmic bytes per
    # launch) and, for the dense sensings, the tensor-core sketch (2 p n m per launch)
    ke, nc = P.model.k_eff, P.model.n_coef
    algo = {
        "modes": nl * (m - 1) + 4 * nl * ke,
        "foreground": nl * m + 4 * m * ((nl + 31) // 32) + 4 * nl * nc,
    }
    if cfg.kind in ("sparse", "spixel"):
        algo["sketch"] = (sector_bytes_sparse(nl, pix0, n, cfg.p, cfg.sensing_seed, m)
                          if cfg.kind == "sparse" else 32 * cfg.p * m + 4 * cfg.p * m)
    elif cfg.kind in ("rademacher", "gaussian"):
        algo["sketch"] = 2 * cfg.p * nl * m
    i8 = int8_peak_tops(torch) if cfg.kind == "rademacher" else None
    tensor_peak = (i8 if i8 else 2.0 * bf16) if cfg.kind == "rademacher" else bf16
    tensor_src = ("measured here: torch._int_mm int8 8192^3 (burst)" if i8 else
                  "2 x measured bf16 (nominal ratio)") if cfg.kind == "rademacher" else peak_src

    def stage_roof(s):
        if s == "sketch" and cfg.kind in ("rademacher", "gaussian"):
            return algo[s] / (stage_ms[s] * 1e-3) / 1e12, tensor_peak, "tensor", "TFLOP/s"
        return algo[s] / (stage_ms[s] * 1e-3) / 1e9, hbm, "hbm", "GB/s"

    cand = {s: stage_ms[s] for s in algo}
    dom = max(cand, key=cand.get)
    achieved, peak, bound, unit = stage_roof(dom)
    traffic = None
    tp = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tp) and cfg.name == "c4_1080p_sparse" and world == 1 and mode:
        traffic = json.load(open(tp)).get(dom)
    sk_kernel = {"sparse": "sketch_sparse_kernel", "spixel": "sketch_spixel_kernel",
                 "rademacher": "sketch_rademacher_tc_kernel",
                 "gaussian": "sketch_gaussian_tc_kernel" if os.environ.get("CDMD_GAUSS_1CTA")
                 else "sketch_gaussian_tc2_kernel"}[cfg.kind]
    vq = C.video(Xd, n, pix0, nl)
    md_kernel = {1: "modes_tc_kernel", 2: "modes_tc_mc_kernel"}.get(C.cdmd_modes_path(P.model), "modes_simt_kernel")
    fg_kernel = {2: "foreground_tc_kernel", 1: "foreground_dynamic_kernel", 0: "foreground_static_kernel"}[
        C.cdmd_foreground_path(vq, P.model, mode)]
    roof = {"kernel": {"sketch": sk_kernel, "modes": md_kernel, "foreground": fg_kernel}[dom],
            "bound": bound, "achieved": round(achieved, 1), "peak": round(peak, 1), "unit": unit,
            "frac": round(achieved / peak, 4), "traffic": traffic,
            "peak_source": tensor_src if bound == "tensor" else peak_src,
            ("algorithmic_flops_per_launch" if bound == "tensor" else "algorithmic_bytes_per_launch"): algo[dom],
            "launch_ms": round(stage_ms[dom], 4),
            "stage_roofline": {s: round(stage_roof(s)[0] / stage_roof(s)[1], 4) for s in algo}}

    # Alg. 1 step 9 full-state amplitudes b = lstsq(Phi, x_1): measured on the
    # modes of the last step, after (and outside) the timed region -- the step's
    # background amplitudes are Remark 3's OMP ones, so this is a reported extra.
    amplitudes = None
    if ke <= 128:
        P.sketch(Xd)
        if allreduce is not None:
            allreduce(P.Y)
        P.fit()
        P.modes(Xd)
        va = C.video(Xd, n, pix0, nl)
        ws_a = torch.empty(max(C.cdmd_amplitudes_workspace_bytes(P.h, ke), 256), dtype=torch.uint8, device="cuda")
        Ga = torch.empty((ke + 1, ke), dtype=torch.float64, device="cuda")
        ba = torch.empty((ke, 2), dtype=torch.float64, device="cuda")

        def amp_once(marks=None):
            if marks:
                marks[0].record(stream)
            C.cdmd_amplitudes_gram(P.h, va, P.model, P.Phi, Ga, ws_a, stream)
            if marks:
                marks[1].record(stream)
            if pixel:
                dist.all_reduce(Ga, op=dist.ReduceOp.SUM)
            if marks:
                marks[2].record(stream)
            C.cdmd_amplitudes_solve(P.h, P.model, Ga, ba, None, stream)
            if marks:
                marks[3].record(stream)

        for _ in range(3):
            amp_once()
        torch.cuda.synchronize()
        reps_a, tg_, ts_ = 10, 0.0, 0.0
        for _ in range(reps_a):
            mk = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
            amp_once(mk)
            torch.cuda.synchronize()
            tg_ += mk[0].elapsed_time(mk[1]) / reps_a
            ts_ += mk[2].elapsed_time(mk[3]) / reps_a
        abytes = 4 * nl * ke + nl
        amplitudes = {"step": "Alg. 1 step 9, b = lstsq(Phi, x_1), not in the timed step",
                      "gram_kernel": "amp_gram_kernel", "gram_ms": round(tg_, 4), "solve_ms": round(ts_, 4),
                      "algorithmic_bytes_per_launch": abytes,
                      "gram_frac_hbm": round(abytes / (tg_ * 1e-3) / 1e9 / hbm, 4)}

    # e2e: host (pinned) video in, mask out, through the same public calls -- through the
    # streaming lanes when they are in use (each batch's H2D copy and mask read-back run
    # on its lane's stream and overlap other batches' work), else one batch at a time
    e2e = None
    if not args.no_e2e:
        Xh = torch.from_numpy(np.ascontiguousarray(np.pad(X_host, ((0, 0), (0, ld - nl))))).pin_memory()
        mask_shape, mask_dtype = P.mask.shape, P.mask.dtype
        if streaming is not None:
            mhs = [torch.empty(mask_shape, dtype=mask_dtype).pin_memory() for _ in range(lanes)]
            e_steps = max(args.steps, 2 * lanes)

            def e2e_run(nb):
                a = torch.cuda.Event(enable_timing=True)
                a.record(stream)
                ends = S.run([Xs[b % lanes] for b in range(nb)], cfg.tau, mode, allreduce=allreduce, start_event=a,
                             host_video=Xh, host_masks=mhs)
                for e in ends:
                    stream.wait_event(e)
                b_ = torch.cuda.Event(enable_timing=True)
                b_.record(stream)
                return a, b_

            e2e_run(lanes)
            torch.cuda.synchronize()
            if world > 1:
                dist.barrier()
            a, b = e2e_run(e_steps)
            torch.cuda.synchronize()
        else:
            mh = torch.empty(mask_shape, dtype=mask_dtype).pin_memory()
            e_steps = max(3, min(10, args.steps))

            def e2e_step():
                Xd.copy_(Xh, non_blocking=True)
                step()
                mh.copy_(P.mask, non_blocking=True)
            e2e_step()
            torch.cuda.synchronize()
            if world > 1:
                dist.barrier()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            for _ in range(e_steps):
                e2e_step()
            b.record(stream)
            torch.cuda.synchronize()
        te = max_over_ranks(a.elapsed_time(b) / e_steps)
        ev_ = m / (te * 1e-3) * (world if not pixel and world > 1 else 1)
        e2e = {"value": round(ev_, 1), "unit": "frames/s",
               "h2d_bytes_per_step": int(Xh.numel()) * world,
               "d2h_bytes_per_step": int(P.mask.numel() * P.mask.element_size()) * world,
               "mode": "streaming lanes" if streaming is not None else "one batch at a time"}

    if rank == 0:
        cpu = None
        if not args.no_cpu_baseline and world == 1:
            cpu = cpu_baseline(cfg, args)
        par = (f"pixel-rows x{world}" if pixel else f"batch replicas x{world}") if world > 1 else "1 GPU"
        line = {
            "metric": METRIC, "value": round(value, 2), "unit": "frames/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms_max, 4),
            "higher_is_better": True, "scaling": "weak" if (world > 1 and not pixel) else "strong",
            "vs_baseline": None, "dtype": "u8", "data": "synthetic",
            "config": {"workload": cfg.name, "video": f"{cfg.width}x{cfg.height}x{m}", "sensing": cfg.kind,
                       "p": cfg.p, "k": cfg.k, "K": cfg.K, "tau": cfg.tau, "background": args.bg, "rank": args.rank,
                       "parallelism": par, "l2": "inputs larger than L2 (X = %.2f GB)" % (n * m / 1e9),
                       "k_eff": ke, "K_eff": P.model.K_eff, "n_coef": nc},
            "stage_ms": {s: round(v, 4) for s, v in stage_ms.items()},
            "latency_ms_per_batch": round(latency_ms, 4),
            "per_batch": per_batch,
            "passes_only": passes_only,
            "e2e_fused": e2e_fused if e2e_fused else {"unavailable": str(fused_ok)},
            "streaming": streaming,
            "roofline": roof,
            "amplitudes": amplitudes,
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": launches,   # libcdmd kernels launched in the timed region (cdmd_kernel_launches)
            "gpu_launches_sequential": launches_seq,
            "clocks": clk.summary(),
        }
        if "error" in graphs:
            line["graph_error"] = graphs["error"]
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
