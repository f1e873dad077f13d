"""Multi-process (gloo, world_size 2, CPU) coverage of the pixel-sharded path's
host logic: slab partition + the one all-reduce of the partial sketches.  The
per-slab partial sketches come from the oracle here (no GPU); the GPU ranks run
the same partition with libcdmd."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1512_04205_b200.dist import allreduce_sum, slab


def test_slab_partition_properties():
    for n in [768, 76800, 345600, 2073600, 8294400, 1000, 129]:
        for world in [1, 2, 3, 4, 8]:
            parts = [slab(n, world, r) for r in range(world)]
            assert parts[0][0] == 0
            for (a, na), (b, _) in zip(parts, parts[1:]):
                assert a + na == b
            assert parts[-1][0] + parts[-1][1] == n
            assert all(p0 % 128 == 0 for p0, _ in parts)
            sizes = [na for _, na in parts]
            assert max(sizes) - min(sizes) <= 128
    assert slab(2073600, 8, 3) == (3 * 259200, 259200)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, kind, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import sensing as S
        from synth.scene import make_video
        W, H, m, p = 48, 40, 12, 30
        n = W * H
        pix0, nl = slab(n, world, rank)
        Xs = make_video(W, H, m, seed=3, noise=2.0, n_rects=1, pix0=pix0, n_local=nl)
        Y = S.sketch(Xs, kind, p, seed=7, n_total=n, pix0=pix0)
        t = torch.from_numpy(np.ascontiguousarray(Y))
        allreduce_sum(t)
        if rank == 0:
            out.put(t.numpy())
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("kind", [0, 1, 2])
def test_two_rank_allreduce_equals_single_rank(kind):
    from oracle import sensing as S
    from synth.scene import make_video
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, 2, port, kind, q)) for r in range(2)]
    for p_ in ps:
        p_.start()
    got = q.get(timeout=120)
    for p_ in ps:
        p_.join(timeout=60)
        assert p_.exitcode == 0
    X = make_video(48, 40, 12, seed=3, noise=2.0, n_rects=1)
    want = S.sketch(X, kind, 30, seed=7)
    assert np.array_equal(got, want)   # integer sketches: bit-identical across world sizes


def test_slab_generation_is_consistent():
    # each rank generates exactly its own bytes of the same global video
    from synth.scene import make_video
    X = make_video(200, 70, 6, seed=5, noise=2.0, n_rects=2)
    n = X.shape[1]
    for world in (2, 3):
        parts = [make_video(200, 70, 6, seed=5, noise=2.0, n_rects=2, pix0=p0, n_local=nl)
                 for p0, nl in (slab(n, world, r) for r in range(world))]
        assert np.array_equal(np.concatenate(parts, axis=1), X)


def _ordered_worker(rank, world, port, out):
    import random
    import threading
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1512_04205_b200.dist import OrderedAllreduce
        coll = OrderedAllreduce()
        nb, lanes = 12, 5
        res = {}
        rng = random.Random(rank)

        def lane(li):
            for b in range(li, nb, lanes):
                threading.Event().wait(rng.random() * 0.01)   # lanes arrive in random order
                y = torch.full((7,), float(rank + 1) * (b + 1))
                coll.allreduce(b, y)                          # sum over ranks: (1 + 2) (b + 1)
                res[b] = y.tolist()

        ts = [threading.Thread(target=lane, args=(li,)) for li in rng.sample(range(lanes), lanes)]
        for t in ts:
            t.start()
        for t in ts:
            t.join(timeout=120)
        out.put((rank, res))
    finally:
        dist.destroy_process_group()


def test_ordered_allreduce_two_ranks():
    """Streaming's batch-ordered all-reduces (dist.OrderedAllreduce): lanes reach their
    all-reduce in any order on each rank; one ticket sequence on one communicator issues
    them in batch order, so every batch is summed with the same batch of the peer."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_ordered_worker, args=(r, 2, port, q)) for r in range(2)]
    for p_ in ps:
        p_.start()
    got = dict(q.get(timeout=180) for _ in range(2))
    for p_ in ps:
        p_.join(timeout=60)
        assert p_.exitcode == 0
    for rank in (0, 1):
        res = got[rank]
        assert sorted(res) == list(range(12))
        for b, y in res.items():
            assert y == [3.0 * (b + 1)] * 7


def test_ordered_allreduce_abort_wakes_waiters():
    """A failed lane aborts the sequence: lanes waiting for a later ticket raise
    LaneAbort instead of waiting forever (no process group needed: fn is local)."""
    import threading
    from paper_1512_04205_b200.dist import LaneAbort, OrderedAllreduce
    coll = OrderedAllreduce()
    seen, errs = [], []

    def waiter(b):
        try:
            coll.run(b, lambda: seen.append(b))
        except LaneAbort as e:
            errs.append((b, str(e)))

    ts = [threading.Thread(target=waiter, args=(b,)) for b in (1, 2, 3)]
    for t in ts:
        t.start()
    coll.abort(RuntimeError("cdmd_fit failed on batch 0"))   # batch 0 never issues its ticket
    for t in ts:
        t.join(timeout=10)
        assert not t.is_alive()
    assert seen == [] and sorted(b for b, _ in errs) == [1, 2, 3]
    coll.reset()
    coll.run(0, lambda: seen.append(0))
    assert seen == [0]


def test_batch_replicas_partition():
    """Batch-parallel replicas: every batch has exactly one owner rank, owners
    round-robin, and a rank's batches are in order."""
    from paper_1512_04205_b200.dist import batch_owner, my_batches
    for world in (1, 2, 3, 8):
        for nb in (0, 1, 7, 24):
            got = sorted(b for r in range(world) for b in my_batches(nb, world, r))
            assert got == list(range(nb))
            for r in range(world):
                mb = my_batches(nb, world, r)
                assert mb == sorted(mb) and all(batch_owner(b, world) == r for b in mb)


def _amp_worker(rank, world, port, out):
    # Alg. 1 step 9 sharded by pixel rows: each rank forms its slab's normal
    # equations [Phi_s^H Phi_s | Phi_s^H x_1,s], one all-reduce sums them, every rank
    # solves (the protocol of cdmd_amplitudes_gram -> all-reduce -> cdmd_amplitudes_solve)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import cdmd as D
        from oracle import sensing as S
        from synth.scene import make_video
        W, H, m, p, k = 48, 40, 12, 30, 6
        n = W * H
        pix0, nl = slab(n, world, rank)
        Xs = make_video(W, H, m, seed=3, noise=2.0, n_rects=1, pix0=pix0, n_local=nl)
        Y = torch.from_numpy(np.ascontiguousarray(S.sketch(Xs, 1, p, seed=7, n_total=n, pix0=pix0)))
        allreduce_sum(Y)
        model = D.fit(Y.numpy(), k, 2)
        Phi_s = D.modes(Xs, model["M"])                               # nl x k complex
        G = np.concatenate([Phi_s.conj().T @ Phi_s, Phi_s.conj().T @ Xs[0].astype(np.float64)[:, None]], 1)
        t = torch.view_as_real(torch.from_numpy(np.ascontiguousarray(G))).contiguous()
        allreduce_sum(t)
        Gs = torch.view_as_complex(t).numpy()
        b = np.linalg.solve(Gs[:, :-1], Gs[:, -1])
        out.put((rank, b))
    finally:
        dist.destroy_process_group()


def test_two_rank_amplitudes_equal_single_rank_lstsq():
    from oracle import cdmd as D
    from oracle import sensing as S
    from synth.scene import make_video
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_amp_worker, args=(r, 2, port, q)) for r in range(2)]
    for p_ in ps:
        p_.start()
    got = dict(q.get(timeout=120) for _ in range(2))
    for p_ in ps:
        p_.join(timeout=60)
        assert p_.exitcode == 0
    X = make_video(48, 40, 12, seed=3, noise=2.0, n_rects=1)
    model = D.fit(S.sketch(X, 1, 30, seed=7), 6, 2)
    want = D.amplitudes(X, D.modes(X, model["M"]))
    for r in (0, 1):
        assert np.max(np.abs(got[r] - want)) <= 1e-8 * np.max(np.abs(want))
    assert np.array_equal(got[0], got[1])    # every rank solves the same summed system
