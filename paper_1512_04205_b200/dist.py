"""Pixel-row sharding of the cDMD hot path across GPUs.

Every per-pixel pass is independent ("embarrassingly parallel"): rank g
owns global pixels [pix0_g, pix0_g + n_g) of every frame.  The sketch is linear
in the pixels (Y = C D = sum_g C[:, slab_g] D[slab_g, :]), so each rank sketches
its slab with C's GLOBAL columns and one all-reduce(SUM) of the small p x m Y
gives every rank the full sketch (int32 sums: exact and order-independent).
The fit is then replicated bit-identically on every rank; modes + mask run
communication-free on each slab.  The streaming lanes issue the per-batch
all-reduces in batch order (OrderedAllreduce).  For long videos the alternative is
batch-parallel replicas: whole batches per rank, no collective at all
(batch_owner).  This module holds only the host logic.
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


def batch_owner(batch, world):
    """Batch-parallel replicas (a long video is "split into batches of 200
    consecutive frames" whose decompositions are "computed for each batch
    independently"): rank b mod world runs batch b end to end on whole frames, with no
    collective at all."""
    return batch % world


def my_batches(nb, world, rank):
    """The batches of a batch-parallel run that this rank owns, in order."""
    return [b for b in range(nb) if batch_owner(b, world) == rank]


class LaneAbort(RuntimeError):
    """Raised in a lane that was waiting for a collective ticket when another lane failed."""


class OrderedAllreduce:
    """Batch-ordered all-reduces of the per-slab partial sketches for the streaming
    lanes of a pixel-sharded run (host logic only).

    Lane threads reach their all-reduce in any order, but every rank must issue the
    collectives of a communicator in the same order.  One ticket sequence in batch
    order over the one communicator gives exactly that: batch b's all-reduce is issued
    once batches 0..b-1 have issued theirs, on every rank.  It is the only collective of
    the data path (the fits are replicated: every rank gets bit-identical Y).
    If a lane fails, abort() wakes every waiter with LaneAbort instead of leaving them
    blocked on a ticket that will never come."""

    def __init__(self, group=None):
        import threading
        self.group = group
        self._cv = threading.Condition()
        self._next = 0
        self._abort = None

    def reset(self):
        with self._cv:
            self._next, self._abort = 0, None
            self._cv.notify_all()

    def abort(self, exc):
        with self._cv:
            if self._abort is None:
                self._abort = exc
            self._cv.notify_all()

    def run(self, b, fn):
        """Run fn() as the b-th collective of the sequence."""
        with self._cv:
            self._cv.wait_for(lambda: self._next == b or self._abort is not None)
            if self._abort is not None:
                raise LaneAbort(f"batch {b}: another lane failed: {self._abort!r}")
            try:
                fn()
            finally:
                self._next += 1
                self._cv.notify_all()

    def allreduce(self, b, tensor):
        import torch.distributed as dist
        self.run(b, lambda: dist.all_reduce(tensor, op=dist.ReduceOp.SUM, group=self.group))
