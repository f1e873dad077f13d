import sys, numpy as np, torch
sys.path.insert(0, ".")
from paper_1512_04205_b200 import cdmd as C
from synth.scene import config_by_name, video_for
cfg = config_by_name("c4_1080p_sparse"); X = video_for(cfg); m, n = X.shape
Xd = torch.from_numpy(X).cuda(); H = C.Handle(0)
P = C.Pipeline(H, n, n, m, cfg.kind, cfg.p, cfg.k, cfg.K, seed=cfg.sensing_seed)
P.run(Xd, cfg.tau, C.BG_DYNAMIC); torch.cuda.synchronize()
def med(fn, reps=15):
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); fn(); b.record(); b.synchronize(); ts.append(a.elapsed_time(b))
    return float(np.median(ts))
t1 = med(lambda: P.foreground(Xd, cfg.tau, C.BG_DYNAMIC, fused=True))
t2 = med(lambda: P.median3(1920, 1080))
t3 = med(lambda: P.foreground_median3(Xd, cfg.tau, 1920, 1080))
print(f"fused pass {t1:.4f} ms + separate median3 {t2:.4f} ms = {t1+t2:.4f};  in-launch fused+median {t3:.4f} ms")
