"""Times candidate small dense solvers for the cDMD fit on the GPU (diagnostic only)."""
import time
import torch

def t(fn, reps=5):
    fn(); torch.cuda.synchronize()
    a = time.perf_counter()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - a) / reps * 1e3

torch.manual_seed(0)
for n1, p in [(199, 1000), (499, 2000), (999, 4000)]:
    Y = torch.randn(p, n1, dtype=torch.float64, device="cuda")
    G = Y.T @ Y
    A = torch.randn(50, 50, dtype=torch.float64, device="cuda")
    print(f"n1={n1} p={p}")
    print("  eigh(G)            %.3f ms" % t(lambda: torch.linalg.eigh(G)))
    print("  eigvalsh(G)        %.3f ms" % t(lambda: torch.linalg.eigvalsh(G)))
    print("  svd(Y) gesvdj?     %.3f ms" % t(lambda: torch.linalg.svd(Y, full_matrices=False)))
    for drv in ["gesvd", "gesvdj", "gesvda"]:
        try:
            print(f"  svd(Y,{drv:6s})     %.3f ms" % t(lambda: torch.linalg.svd(Y, full_matrices=False, driver=drv)))
        except Exception as e:
            print("  ", drv, "failed", str(e)[:60])
    print("  qr(Y)              %.3f ms" % t(lambda: torch.linalg.qr(Y)))
    print("  eig(A 50x50)       %.3f ms" % t(lambda: torch.linalg.eig(A)))
    A100 = torch.randn(100, 100, dtype=torch.float64, device="cuda")
    print("  eig(A 100x100)     %.3f ms" % t(lambda: torch.linalg.eig(A100)))
