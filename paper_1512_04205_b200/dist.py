"""Pixel-row sharding of the cDMD hot path across GPUs.

Every per-pixel pass is independent ("embarrassingly parallel"): rank g
owns global pixels [pix0_g, pix0_g + n_g) of every frame.  The sketch is linear
in the pixels (Y = C D = sum_g C[:, slab_g] D[slab_g, :]), so each rank sketches
its slab with C's GLOBAL columns and one all-reduce(SUM) of the small p x m Y
gives every rank the full sketch (int32 sums: exact and order-independent).
One batch at a time the fit is then replicated bit-identically on every rank;
the streaming lanes instead solve batch b on rank b mod world and broadcast the
model (OrderedCollectives).  Modes + mask run communication-free on each slab.
This module holds only the host logic.
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


def fit_owner(batch, world):
    """Rank that runs the small solve of `batch` when fits are sharded (round robin)."""
    return batch % world


class OrderedCollectives:
    """Batch-ordered collectives for the streaming lanes (host logic only).

    Lane threads reach their collectives in any order; NCCL (and gloo) need every rank
    to issue the collectives of one communicator in the same order.  Each kind of
    collective has its own ticket sequence in batch order and its own communicator:
    the all-reduce of the partial sketches on `ar_group`, the broadcast of a fitted
    model from its owner (fit_owner) on `bc_group`, so the two sequences never have to
    interleave identically across ranks.  With sharded fits each rank runs 1/world of
    the small solves (the per-batch work is independent) instead of all of them."""

    def __init__(self, ar_group=None, bc_group=None):
        import threading
        self.ar_group, self.bc_group = ar_group, bc_group
        # one lock per sequence: a thread blocked inside one kind of collective (gloo
        # calls block until the peers join) must not stop the other sequence
        self._cv = {"ar": threading.Condition(), "bc": threading.Condition()}
        self._next = {"ar": 0, "bc": 0}

    def reset(self):
        for kind, cv in self._cv.items():
            with cv:
                self._next[kind] = 0
                cv.notify_all()

    def _ordered(self, kind, b, fn):
        cv = self._cv[kind]
        with cv:
            cv.wait_for(lambda: self._next[kind] == b)
            try:
                fn()
            finally:
                self._next[kind] += 1
                cv.notify_all()

    def allreduce(self, b, tensor):
        import torch.distributed as dist
        self._ordered("ar", b, lambda: dist.all_reduce(tensor, op=dist.ReduceOp.SUM, group=self.ar_group))

    def broadcast(self, b, tensor, src):
        import torch.distributed as dist
        self._ordered("bc", b, lambda: dist.broadcast(tensor, src=src, group=self.bc_group))
