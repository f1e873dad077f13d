#!/usr/bin/env python
"""Throughput benchmark of the cDMD hot path on B200 (BASELINE.json metric).

metric : "1080p frames/sec (sketch+modes+fg mask) at 1/2/4/8 B200; % of HBM roofline"
step   : one pass of the whole hot path over one batch:
         cdmd_sketch -> all_reduce(Y) -> cdmd_fit -> cdmd_modes -> cdmd_foreground
workload (N=1): c4_1080p_sparse = 1920x1080, m = 500 frames, sparse C (s = n/ln n),
         p = 2000, k = 50, K = 10, tau = 25, dynamic background (north_star (3)).
value  : frames / device time per step (max over ranks), inputs resident in HBM;
         X (1.04 GB) is larger than L2, so no flush is needed between steps.
         Streaming (default, --lanes 24): K batches flow through 24 lanes (own handle,
         CUDA stream, buffers and copy of X), so one batch's latency-bound small solve
         overlaps other batches' HBM passes -- the paper's batch decomposition of a long
         video.  `latency_ms_per_batch` reports one batch at a time (--lanes 1).

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

# Streaming runs 2 streams per lane (24 lanes by default).  With the default 8 hardware
# work queues, streams share queues and a lane's queued solve kernel blocks unrelated
# streams behind it (measured: 16 concurrent solves 0.79 -> 0.51 ms/batch with 32).
# Must be set before the CUDA context exists.
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

FALLBACK_HBM_GBS = 6650.0   # B200_PROFILING.md fallback, used only without MEASURED_PEAKS.json
FALLBACK_BF16_TFLOPS = 1590.0
METRIC = "1080p frames/sec (sketch+modes+fg mask) at 1/2/4/8 B200; % of HBM roofline"


def peaks():
    """(HBM GB/s, dense bf16 TFLOP/s burst, source): MEASURED_PEAKS.json, else the recipe's fallback."""
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d["hbm_gbs"]), float(d["bf16_tflops"]), "measured"
    return FALLBACK_HBM_GBS, FALLBACK_BF16_TFLOPS, "fallback"


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


def run_reference(args):
    """The oracle (test infrastructure) timed as it stands on this host's cores, on a
    bounded sample of the same workload: the full sketch + fit, then modes + dynamic
    background + mask on 1/`frac` of the pixels, extrapolated to the whole frame."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from oracle import cdmd as OD
    from oracle import sensing as OS
    from synth.scene import config_by_name, video_for
    cfg = config_by_name(args.config)
    X = video_for(cfg)
    m, n = X.shape
    kind = {"spixel": 0, "sparse": 1, "rademacher": 2, "gaussian": 3}[cfg.kind]
    frac = args.ref_frac
    rng = np.random.default_rng(0)
    pix = np.sort(rng.choice(n, n // frac, replace=False))
    times = []
    for _ in range(max(1, args.steps if args.steps <= 3 else 1)):
        t0 = time.perf_counter()
        if kind in (0, 1):
            Y = OS.sketch(X, kind, cfg.p, cfg.sensing_seed)
            t_sk = time.perf_counter() - t0
        else:  # dense sketches: a sample of rows, extrapolated
            rows = np.arange(0, cfg.p, max(1, cfg.p // 16))
            OS.sketch(X, kind, cfg.p, cfg.sensing_seed, rows=rows)
            t_sk = (time.perf_counter() - t0) * cfg.p / len(rows)
            Y = None
        t1 = time.perf_counter()
        if Y is None:
            raise SystemExit("reference arm: dense-C configs need the full oracle sketch (not sampled here)")
        model = OD.fit(Y, cfg.k, cfg.K)
        t_fit = time.perf_counter() - t1
        t2 = time.perf_counter()
        Xs = X[:, pix]
        Phi = OD.modes(Xs, model["M"])
        L = OD.background_dynamic(Phi, model) if args.bg == "dynamic" else OD.background_static(Phi, model)
        OD.mask(Xs, L, cfg.tau)
        t_px = (time.perf_counter() - t2) * frac
        times.append(t_sk + t_fit + t_px)
    t = min(times)
    cores = len(os.sched_getaffinity(0))
    val = m / t
    line = {
        "impl": "reference", "metric": METRIC, "value": val, "unit": "frames/s", "n_gpus": args.gpus,
        "steps": len(times), "warmup": 0, "ms_per_step": t * 1e3, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": cfg.name, "video": f"{cfg.width}x{cfg.height}x{cfg.m}", "sensing": cfg.kind,
                   "p": cfg.p, "k": cfg.k, "K": cfg.K, "tau": cfg.tau, "background": args.bg},
        "cpu_baseline": {"value": val, "unit": "frames/s", "cores": cores, "kind": "oracle",
                         "sample": f"full sketch+fit; modes+background+mask on 1/{frac} of the pixels "
                                   f"({len(pix)} px), extrapolated x{frac}"},
        "e2e": {"value": val, "unit": "frames/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="cdmd", choices=["cdmd", "reference"])
    ap.add_argument("--config", default="c4_1080p_sparse")
    ap.add_argument("--bg", default="dynamic", choices=["dynamic", "static"])
    ap.add_argument("--rank", default="fixed", choices=["fixed", "gd"],
                    help="target rank: the config's k, or Gavish-Donoho (Remark 2, P:361) with k as the cap")
    ap.add_argument("--ref-frac", type=int, default=32)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--lanes", type=int, default=24,
                    help="batches in flight (streaming, P:573); 1 = one batch at a time")
    ap.add_argument("--replicated-fits", action="store_true",
                    help="N > 1 streaming: every rank solves every batch (north_star's redundant solve) "
                         "instead of rank b mod N solving batch b and broadcasting the model")
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
    pix0, nl = slab(n, world, rank)
    X_host = video_for(cfg, pix0=pix0, n_local=nl)
    ld = ((nl + 15) // 16) * 16
    Xd = torch.zeros((m, ld), dtype=torch.uint8, device="cuda")
    Xd[:, :nl] = torch.from_numpy(X_host).cuda()
    H = C.Handle(local)
    P = C.Pipeline(H, n, nl, m, cfg.kind, cfg.p, cfg.k, cfg.K, seed=cfg.sensing_seed, pix0=pix0, rank=args.rank)
    mode = C.BG_DYNAMIC if args.bg == "dynamic" else C.BG_STATIC
    stream = torch.cuda.current_stream()
    ev = {s: [] for s in ("sketch", "allreduce", "fit", "modes", "foreground")}

    def step(record=False):
        marks = [torch.cuda.Event(enable_timing=True) for _ in range(6)] if record else None
        if record:
            marks[0].record(stream)
        P.sketch(Xd)
        if record:
            marks[1].record(stream)
        if world > 1:
            dist.all_reduce(P.Y, op=dist.ReduceOp.SUM)
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
    ms = start.elapsed_time(stop) / args.steps
    stage_ms = {s: sum(a.elapsed_time(b) for a, b in v) / len(v) for s, v in ev.items()}
    t = torch.tensor([ms], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_max = float(t.item())
    value = m / (ms_max * 1e-3)
    latency_ms = ms_max

    streaming = None
    if args.lanes > 1:
        # K batches through `lanes` concurrent lanes; each lane reads its own copy of X
        S = C.Streaming(local, n, nl, m, cfg.kind, cfg.p, cfg.k, cfg.K, lanes=args.lanes,
                        seed=cfg.sensing_seed, pix0=pix0, rank=args.rank, fit_sms=args.fit_sms,
                        shard_fit=not args.replicated_fits)
        Xs = [Xd] + [Xd.clone() for _ in range(args.lanes - 1)]
        ar = (lambda Y: dist.all_reduce(Y, op=dist.ReduceOp.SUM)) if world > 1 else None

        def stream_run(nb):
            a = torch.cuda.Event(enable_timing=True)
            a.record(stream)
            ends = S.run([Xs[b % args.lanes] for b in range(nb)], cfg.tau, mode, allreduce=ar, start_event=a)
            for e in ends:
                stream.wait_event(e)
            b_ = torch.cuda.Event(enable_timing=True)
            b_.record(stream)
            return a, b_

        stream_run(max(args.warmup, args.lanes))
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
        ts = torch.tensor([a.elapsed_time(b_) / args.steps], dtype=torch.float64, device="cuda")
        if world > 1:
            dist.all_reduce(ts, op=dist.ReduceOp.MAX)
        ms_max = float(ts.item())
        value = m / (ms_max * 1e-3)
        streaming = {"lanes": args.lanes, "ms_per_batch": round(ms_max, 4), "sm_partition": S.sms,
                     "fits": "sharded: batch b solved on rank b mod N, model broadcast" if S.shard_fit
                     else "every rank",
                     "note": "batches pipelined across lanes (own handle, stream, buffers, copy of X)"}

    # roofline of the dominant kernel: HBM-bound passes (algorithmic bytes per launch) and,
    # for the dense sensings, the tensor-core sketch (algorithmic 2 p n m flops per launch)
    hbm, bf16, peak_src = peaks()
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
    # kind::f16 runs at the bf16 rate; kind::i8 at twice it (the guide's nominal 4.5 / 2.25 ratio)
    tensor_peak = bf16 * (2.0 if cfg.kind == "rademacher" else 1.0)

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
            "bound": bound, "achieved": round(achieved, 1), "peak": peak, "unit": unit,
            "frac": round(achieved / peak, 4), "traffic": traffic, "peak_source": peak_src,
            ("algorithmic_flops_per_launch" if bound == "tensor" else "algorithmic_bytes_per_launch"): algo[dom],
            "launch_ms": round(stage_ms[dom], 4),
            "stage_roofline": {s: round(stage_roof(s)[0] / stage_roof(s)[1], 4) for s in algo}}

    # Alg. 1 step 9 full-state amplitudes b = lstsq(Phi, x_1): measured on the
    # modes of the last step, after (and outside) the timed region -- the step's
    # background amplitudes are Remark 3's OMP ones, so this is a reported extra.
    # Phi (n_local x k_eff fp32) is larger than L2 at the bench sizes.
    amplitudes = None
    if ke <= 128:
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
            if world > 1:
                dist.all_reduce(Ga, op=dist.ReduceOp.SUM)
            if marks:
                marks[2].record(stream)
            C.cdmd_amplitudes_solve(P.h, P.model, Ga, ba, None, stream)
            if marks:
                marks[3].record(stream)

        for _ in range(3):
            amp_once()
        torch.cuda.synchronize()
        reps, tg_, ts_ = 10, 0.0, 0.0
        for _ in range(reps):
            mk = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
            amp_once(mk)
            torch.cuda.synchronize()
            tg_ += mk[0].elapsed_time(mk[1]) / reps
            ts_ += mk[2].elapsed_time(mk[3]) / reps
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
            mhs = [torch.empty(mask_shape, dtype=mask_dtype).pin_memory() for _ in range(args.lanes)]
            e_steps = max(args.steps, 2 * args.lanes)

            def e2e_run(nb):
                a = torch.cuda.Event(enable_timing=True)
                a.record(stream)
                ends = S.run([Xs[b % args.lanes] for b in range(nb)], cfg.tau, mode, allreduce=ar, start_event=a,
                             host_video=Xh, host_masks=mhs)
                for e in ends:
                    stream.wait_event(e)
                b_ = torch.cuda.Event(enable_timing=True)
                b_.record(stream)
                return a, b_

            e2e_run(args.lanes)
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
        te = torch.tensor([a.elapsed_time(b) / e_steps], dtype=torch.float64, device="cuda")
        if world > 1:
            dist.all_reduce(te, op=dist.ReduceOp.MAX)
        e2e = {"value": m / (float(te.item()) * 1e-3), "unit": "frames/s",
               "h2d_bytes_per_step": int(Xh.numel()) * world,
               "d2h_bytes_per_step": int(P.mask.numel() * P.mask.element_size()) * world,
               "mode": "streaming lanes" if streaming is not None else "one batch at a time"}

    if rank == 0:
        cpu = None
        if not args.no_cpu_baseline and world == 1:
            cpu = cpu_baseline(cfg, X_host, args)
        line = {
            "metric": METRIC, "value": round(value, 2), "unit": "frames/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms_max, 4),
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "u8",
            "data": "synthetic",
            "config": {"workload": cfg.name, "video": f"{cfg.width}x{cfg.height}x{m}", "sensing": cfg.kind,
                       "p": cfg.p, "k": cfg.k, "K": cfg.K, "tau": cfg.tau, "background": args.bg, "rank": args.rank,
                       "parallelism": f"pixel-rows x{world}", "l2": "inputs larger than L2 (X = %.2f GB)" % (n * m / 1e9),
                       "k_eff": ke, "K_eff": P.model.K_eff, "n_coef": nc},
            "stage_ms": {s: round(v, 4) for s, v in stage_ms.items()},
            "latency_ms_per_batch": round(latency_ms, 4),
            "streaming": streaming,
            "roofline": roof,
            "amplitudes": amplitudes,
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": launches,   # libcdmd kernels launched in the timed region (cdmd_kernel_launches)
            "clocks": clk.summary(),
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def cpu_baseline(cfg, X, args):
    """The oracle as it stands, on a bounded sample (about 10-30 s of CPU work)."""
    from oracle import cdmd as OD
    from oracle import sensing as OS
    m, n = X.shape
    frac = args.ref_frac
    rng = np.random.default_rng(0)
    pix = np.sort(rng.choice(n, n // frac, replace=False))
    kind = {"spixel": 0, "sparse": 1, "rademacher": 2, "gaussian": 3}[cfg.kind]
    dense = cfg.kind in ("rademacher", "gaussian")
    t0 = time.perf_counter()
    if dense:
        # a dense C row costs a full pass over X on the CPU: time every frac-th row and
        # extrapolate; the fit runs on those rows (a p/frac x m sketch)
        rstep = frac * (2 if cfg.kind == "gaussian" else 1)
        Y = OS.sketch(X, kind, cfg.p, cfg.sensing_seed, rows=np.arange(0, cfg.p, rstep))
        t_sk = (time.perf_counter() - t0) * rstep
    else:
        Y = OS.sketch(X, kind, cfg.p, cfg.sensing_seed)
        t_sk = time.perf_counter() - t0
    t1 = time.perf_counter()
    model = OD.fit(Y, min(cfg.k, Y.shape[0]), cfg.K)
    t_fit = time.perf_counter() - t1
    t2 = time.perf_counter()
    Xs = X[:, pix]
    Phi = OD.modes(Xs, model["M"])
    L = OD.background_dynamic(Phi, model) if args.bg == "dynamic" else OD.background_static(Phi, model)
    OD.mask(Xs, L, cfg.tau)
    t_px = (time.perf_counter() - t2) * frac
    total = t_sk + t_fit + t_px
    return {"value": round(m / total, 3), "unit": "frames/s", "cores": len(os.sched_getaffinity(0)),
            "kind": "oracle",
            "sample": f"{cfg.name}: " + (f"sketch of every {rstep}th row ({t_sk / rstep:.1f}s) extrapolated x{rstep}"
                                         f" + fit of that {Y.shape[0]}-row sketch ({t_fit:.1f}s)" if dense else
                                         f"full sketch ({t_sk:.1f}s) + fit ({t_fit:.1f}s)") + "; modes+background+mask "
                      f"on 1/{frac} of the pixels ({len(pix)} px, {t_px / frac:.1f}s) extrapolated x{frac}"}


if __name__ == "__main__":
    main()
