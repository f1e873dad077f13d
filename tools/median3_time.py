import torch, sys
sys.path.insert(0, '.')
from paper_1512_04205_b200 import cdmd as C
W, H, m = 1920, 1080, 500
n = W * H
ldw = (n + 31) // 32
mask = torch.randint(-2**31, 2**31 - 1, (m, ldw), dtype=torch.int32, device="cuda")
out = torch.empty_like(mask)
for _ in range(3): C.cdmd_mask_median3(mask, W, H, out)
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(20): C.cdmd_mask_median3(mask, W, H, out)
b.record(); torch.cuda.synchronize()
ms = a.elapsed_time(b) / 20
print(f"median3 1080p x 500: {ms:.4f} ms, {2 * mask.numel() * 4 / ms / 1e6:.1f} GB/s (read + write)")
