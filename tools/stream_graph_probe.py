"""Streaming with per-lane whole-step CUDA graphs (diagnostic): compares the batches/s of
cdmd.Streaming (eager fit) with lanes replaying a captured step graph each.
python tools/stream_graph_probe.py [lanes] [batches]"""
import os
import sys
import threading

os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")
import torch

sys.path.insert(0, ".")
from paper_1512_04205_b200 import cdmd as C  # noqa: E402
from synth.scene import config_by_name, video_for  # noqa: E402

lanes = int(sys.argv[1]) if len(sys.argv) > 1 else 10
batches = int(sys.argv[2]) if len(sys.argv) > 2 else 40
cfg = config_by_name("c4_1080p_sparse")
X = video_for(cfg)
m, n = X.shape
ld = ((n + 15) // 16) * 16
X0 = torch.zeros((m, ld), dtype=torch.uint8, device="cuda")
X0[:, :n] = torch.from_numpy(X).cuda()
vids = [X0.clone() for _ in range(lanes)]
mode = C.BG_DYNAMIC

# eager streaming (the library)
S = C.Streaming(0, n, n, m, "sparse", cfg.p, cfg.k, cfg.K, lanes=lanes, seed=cfg.sensing_seed)
work = [vids[b % lanes] for b in range(batches)]
S.run(work[:lanes], cfg.tau, mode)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
ends = S.run(work, cfg.tau, mode, start_event=e0)
for e in ends:
    torch.cuda.current_stream().wait_event(e)
e1.record()
torch.cuda.synchronize()
t_eager = e0.elapsed_time(e1) / batches

# graph lanes: each lane captures sketch + fit + modes + foreground once
graphs = []
for li, (h, st, st_fit, pipe) in enumerate(S.lanes):
    Xl = vids[li]
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(st):
        pipe.run(Xl, cfg.tau, mode)
        torch.cuda.synchronize()
        with torch.cuda.graph(g, stream=st):
            pipe.sketch(Xl)
            pipe.fit()
            pipe.modes(Xl)
            pipe.foreground(Xl, cfg.tau, mode)
    graphs.append(g)
torch.cuda.synchronize()
start = torch.cuda.Event(enable_timing=True)
endev = [None] * lanes


def lane(li):
    h, st, st_fit, pipe = S.lanes[li]
    with torch.cuda.stream(st):
        st.wait_event(start)
        for b in range(li, batches, lanes):
            graphs[li].replay()
        ev = torch.cuda.Event(enable_timing=True)
        ev.record(st)
        endev[li] = ev


start.record()
ths = [threading.Thread(target=lane, args=(i,)) for i in range(lanes)]
for t in ths:
    t.start()
for t in ths:
    t.join()
e1 = torch.cuda.Event(enable_timing=True)
for e in endev:
    torch.cuda.current_stream().wait_event(e)
e1.record()
torch.cuda.synchronize()
t_graph = start.elapsed_time(e1) / batches
stale = sum(int(p.graph_stale()) for (_, _, _, p) in S.lanes)
print(f"lanes {lanes} batches {batches}: eager {t_eager:.4f} ms/batch ({m / t_eager * 1e3:.0f} frames/s), "
      f"graphs {t_graph:.4f} ms/batch ({m / t_graph * 1e3:.0f} frames/s), stale lanes {stale}")
