"""Pixel-row sharding of the cDMD hot path across GPUs.

Every per-pixel pass is independent ("embarrassingly parallel"): rank g
owns global pixels [pix0_g, pix0_g + n_g) of every frame.  The sketch is linear
in the pixels (Y = C D = sum_g C[:, slab_g] D[slab_g, :]), so each rank sketches
its slab with C's GLOBAL columns and one all-reduce(SUM) of the small p x m Y
gives every rank the full sketch (int32 sums: exact and order-independent).
The fit is then replicated bit-identically on every rank, and modes + mask run
communication-free on each slab.  This module holds only the host logic.
"""

import math


def slab(n_total, world, rank, align=128):
    """Near-equal slabs whose boundaries are multiples of `align` pixels (the
    C ABI requires pix0 % 128 == 0).  Returns (pix0, n_local)."""
    blocks = math.ceil(n_total / align)
    b0 = (blocks * rank) // world
    b1 = (blocks * (rank + 1)) // world
    p0 = min(n_total, b0 * align)
    p1 = min(n_total, b1 * align)
    return p0, p1 - p0


def allreduce_sum(tensor, group=None):
    """The one data-path collective: SUM of the per-slab partial sketches."""
    import torch.distributed as dist
    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(tensor, op=dist.ReduceOp.SUM, group=group)
    return tensor
