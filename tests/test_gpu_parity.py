"""GPU (libcdmd, sm_100a) vs CPU oracle parity on identical seeded inputs.

Every call goes through the C ABI (paper_1512_04205_b200.cdmd is ctypes only).
Tolerances: tests/parity.py (north_star).  Sizes: small cases the oracle runs in
seconds that still span several tiles and ragged tails, plus the bench's full
1080p configuration checked exactly (integer sketch) or on sampled outputs.
"""

import os
import zlib

import numpy as np
import pytest
import torch

from oracle import cdmd as OD
from oracle import sensing as OS
from synth.scene import config_by_name, make_video, video_for
import parity as PT  # tests/parity.py (tests/ is on sys.path under pytest)

pytestmark = pytest.mark.gpu

KIND = {"spixel": 0, "sparse": 1, "rademacher": 2, "gaussian": 3, "srft": 4}


@pytest.fixture(scope="module")
def C():
    from paper_1512_04205_b200 import cdmd
    return cdmd


@pytest.fixture(scope="module")
def H(C):
    return C.Handle(0)


def to_dev(X, ld=None):
    m, n = X.shape
    ld = ((n + 15) // 16) * 16 if ld is None else ld
    buf = torch.zeros((m, ld), dtype=torch.uint8, device="cuda")
    buf[:, :n] = torch.from_numpy(X).cuda()
    return buf


def gpu_run(C, H, X, kind, p, k, K, tau, s=0.0, seed=0, modes_simt=False, ld=None, rank="fixed", omega_eps=0.0):
    m, n = X.shape
    Xd = to_dev(X, ld)
    P = C.Pipeline(H, n, n, m, kind, p, k, K, s=s, seed=seed, rank=rank, omega_eps=omega_eps)
    Y = P.sketch(Xd).cpu().numpy().T.copy()          # p x m
    P.fit()
    mh = C.model_to_host(P.model)
    Phi = P.modes(Xd, simt=modes_simt).cpu().numpy()  # k_eff x n folded
    out = dict(Y=Y, model=mh, Phi=Phi)
    for mode, name in ((C.BG_DYNAMIC, "dyn"), (C.BG_STATIC, "sta")):
        Wd = P.foreground(Xd, tau, mode).cpu().numpy().view(np.uint32)
        out["mask_" + name] = OD.unpack_mask(Wd, n)
        out["L_" + name] = P.background(mode).cpu().numpy()   # (m, n) frame-major
    fused = fused_mask(C, P, Xd, tau)
    if fused is not None:
        out["mask_fus"] = OD.unpack_mask(fused, n)
    torch.cuda.synchronize()
    out["P"], out["Xd"] = P, Xd
    return out


def fused_mask(C, P, Xd, tau):
    """The fused single pass N11 (cdmd_foreground with Phi = NULL): packed mask words, or
    None where it is not supported (CDMD_ERR_UNSUPPORTED: n_coef > 16 or m > 512)."""
    try:
        return P.foreground(Xd, tau, C.BG_DYNAMIC, fused=True).cpu().numpy().view(np.uint32).copy()
    except C.CdmdError as e:
        if e.code == 6:
            return None
        raise


def oracle_run(X, kind, p, k, K, tau, s=None, seed=0, rank="fixed", omega_eps=None, Y=None):
    Y = OS.sketch(X, KIND[kind], p, seed, s=s) if Y is None else Y
    model = OD.fit(Y, k, K, rank=rank, omega_eps=omega_eps)
    Phi = OD.modes(X, model["M"])
    Ld = OD.background_dynamic(Phi, model)          # n x m
    Ls = OD.background_static(Phi, model)           # n
    Xf = X.astype(np.float64)
    return dict(Y=Y, model=model, Phi=Phi, L_dyn=Ld.T, L_sta=Ls,
                res_dyn=np.abs(Xf - Ld.T), res_sta=np.abs(Xf - Ls[None, :]),
                mask_dyn=OD.mask(X, Ld, tau), mask_sta=OD.mask(X, Ls, tau))


def check_all(g, o, kind, tau):
    # sketch
    if kind in ("gaussian", "srft"):
        d = np.linalg.norm(g["Y"] - o["Y"], axis=0) / np.linalg.norm(o["Y"], axis=0)
        assert d.max() <= PT.RTOL_Y_GAUSS, d.max()
    else:
        assert g["Y"].dtype == np.int32 or g["Y"].dtype == np.int64
        assert np.array_equal(g["Y"].astype(np.int64), o["Y"])
    gm, om = g["model"], o["model"]
    assert gm["k_eff"] == om["k_eff"]
    perm, err = PT.match_eigs(gm["lam"], om["lam"])
    assert err <= PT.RTOL_EIG, err
    s_rel = np.abs(gm["sigma"] - om["sigma"]) / om["sigma"]
    assert s_rel.max() <= 1e-6, s_rel.max()
    assert list(gm["pair"]) == list(om["pair"]) or sorted(gm["pair"]) == sorted(om["pair"])
    # modes, per column after phase alignment, well-separated eigenvalues only
    Pg = PT.unfold(g["Phi"], gm["pair"])
    for i in range(gm["k_eff"]):
        j = perm[i]
        if not PT.well_separated(om["lam"], j):
            continue
        r = PT.phase_aligned_rel(Pg[:, i], o["Phi"][:, j])
        assert r <= PT.RTOL_PHI, (i, j, r)
    # OMP support (modulo conjugation)
    assert gm["K_eff"] == len(om["support"])
    assert PT.supports_equal_mod_conj(gm["support"], gm["pair"], perm, om["support"], om["pair"])
    # backgrounds
    scale = max(1.0, np.abs(o["L_dyn"]).max())
    assert np.abs(g["L_dyn"] - o["L_dyn"]).max() <= 1e-4 * scale
    assert np.abs(g["L_sta"][0] - o["L_sta"]).max() <= 1e-4 * scale
    # masks (the fused single pass against the oracle's dynamic mask)
    for name, ref in (("dyn", "dyn"), ("sta", "sta"), ("fus", "dyn")):
        if "mask_" + name not in g:
            continue
        frac, band, nd = PT.mask_agreement(g["mask_" + name], o["mask_" + ref], o["res_" + ref], tau)
        assert frac >= PT.MASK_AGREE and band, (name, frac, nd)


# ------------------------------------------------------------- generator pins
def test_philox_known_answers(C):
    ctr32 = torch.tensor(np.array([[0, 0, 0, 0], [0xffffffff] * 4,
                                   [0x243f6a88, 0x85a308d3, 0x13198a2e, 0x03707344]], dtype=np.uint32).view(np.int32),
                         device="cuda")
    keys = [(0, 0), (0xffffffff, 0xffffffff), (0xa4093822, 0x299f31d0)]
    want = [[0x6627e8d5, 0xe169c58d, 0xbc57ac4c, 0x9b00dbd8], [0x408f276d, 0x41c83b0e, 0xa20bc7c6, 0x6d5451fd],
            [0xd16cfe09, 0x94fdcceb, 0x5001e420, 0x24126ea1]]
    for i, (k0, k1) in enumerate(keys):
        out = torch.zeros(4, dtype=torch.int32, device="cuda")
        C.cdmd_philox(ctr32[i].contiguous(), k0, k1, out)
        assert out.cpu().numpy().view(np.uint32).tolist() == want[i]


def test_philox_random_counters_match_oracle(C):
    from oracle.philox import philox4x32_10
    rng = np.random.default_rng(0)
    c = rng.integers(0, 2 ** 32, size=(4096, 4), dtype=np.uint64)
    out = torch.zeros(4096 * 4, dtype=torch.int32, device="cuda")
    C.cdmd_philox(torch.from_numpy(c.astype(np.uint32).view(np.int32)).cuda().reshape(-1), 123, 456, out)
    got = out.cpu().numpy().view(np.uint32).reshape(4096, 4)
    w = philox4x32_10(c[:, 0], c[:, 1], c[:, 2], c[:, 3], 123, 456)
    assert np.array_equal(got, np.stack(w, 1).astype(np.uint32))


def test_gaussian_table_bit_exact(C, H):
    out = torch.zeros(65536, dtype=torch.int16, device="cuda")
    C.cdmd_gaussian_table(H, out)
    bits = out.cpu().numpy().view(np.uint16).astype(np.uint32) << 16
    got = bits.view(np.float32).astype(np.float64)
    assert np.array_equal(got, OS.gaussian_table())


@pytest.mark.parametrize("n,p,seed", [(1, 1, 0), (768, 768, 3), (76800, 1000, 0), (2073600, 2000, 0),
                                      (8294400, 4000, 9), (1000, 999, 5)])
def test_spixel_rows_bit_exact(C, H, n, p, seed):
    out = torch.zeros(p, dtype=torch.int32, device="cuda")
    C.cdmd_sensing_rows(H, n, C.sensing("spixel", p, 0, seed), out)
    assert np.array_equal(out.cpu().numpy().astype(np.int64), OS.spixel_rows(n, p, seed))


@pytest.mark.parametrize("n,p,s,seed", [(768, 50, 0.0, 0), (3700, 120, 0.0, 1), (2073600, 2000, 0.0, 0),
                                        (5000, 64, 3.5, 2), (8294400, 400, 0.0, 0)])
def test_sparse_rows_bit_exact(C, H, n, p, s, seed):
    cap = C.cdmd_sparse_cap(n, p, s)
    ell = torch.zeros(p * cap, dtype=torch.int32, device="cuda")
    cnt = torch.zeros(p, dtype=torch.int32, device="cuda")
    C.cdmd_sensing_rows(H, n, C.sensing("sparse", p, s, seed), ell, cnt)
    ell = ell.cpu().numpy().reshape(p, cap)
    cnt = cnt.cpu().numpy()
    rows = OS.sparse_rows(n, p, s if s > 0 else OS.default_s(n), seed)
    for r in range(p):
        pos, sg = rows[r]
        assert cnt[r] == len(pos)
        e = ell[r, :cnt[r]].astype(np.int64)
        assert np.array_equal(e >> 1, pos)
        assert np.array_equal(np.where(e & 1, -1, 1), sg)


# ------------------------------------------------------- whole-path parity
CASES = [
    # name, (W, H, m, noise, rects), kind, p, k, K, tau
    ("c1", None, "sparse", 50, 10, 2, 25.0),
    ("ragged_sparse", (100, 37, 33, 2.0, 1), "sparse", 120, 12, 5, 20.0),
    ("ragged_spixel", (97, 61, 45, 2.0, 2), "spixel", 400, 15, 6, 25.0),
    ("rademacher_small", (180, 120, 60, 2.0, 2), "rademacher", 300, 20, 6, 25.0),
    ("gaussian_small", (160, 100, 50, 2.0, 1), "gaussian", 256, 16, 6, 25.0),
    ("srft_small", (160, 100, 50, 2.0, 1), "srft", 256, 16, 6, 25.0),
    ("srft_ragged", (97, 61, 45, 2.0, 2), "srft", 202, 15, 6, 25.0),
]


@pytest.mark.parametrize("case", CASES, ids=[c[0] for c in CASES])
def test_pipeline_parity_small(C, H, case):
    name, shape, kind, p, k, K, tau = case
    if shape is None:
        cfg = config_by_name("c1_32x24_sparse")
        X = video_for(cfg)
    else:
        W, Hh, m, noise, rects = shape
        X = make_video(W, Hh, m, seed=zlib.crc32(name.encode()) % 1000, noise=noise, n_rects=rects)
    g = gpu_run(C, H, X, kind, p, k, K, tau)
    o = oracle_run(X, kind, p, k, K, tau)
    check_all(g, o, kind, tau)


def test_c2_full_parity(C, H):
    cfg = config_by_name("c2_320x240_spixel")
    X = video_for(cfg)
    g = gpu_run(C, H, X, cfg.kind, cfg.p, cfg.k, cfg.K, cfg.tau)
    o = oracle_run(X, cfg.kind, cfg.p, cfg.k, cfg.K, cfg.tau)
    check_all(g, o, cfg.kind, cfg.tau)


def test_modes_tensor_core_equals_simt(C, H):
    X = make_video(333, 200, 77, seed=4, noise=2.0, n_rects=2)   # ragged n, ragged m
    m, n = X.shape
    Xd = to_dev(X)
    P = C.Pipeline(H, n, n, m, "sparse", 200, 24, 6)
    P.sketch(Xd)
    P.fit()
    a = P.modes(Xd).clone()
    b = P.modes(Xd, simt=True).clone()
    assert torch.equal(a, b)


def test_modes_cluster_kernel_equals_simt(C, H):
    """k_eff > 64: the 4-CTA cluster kernel (X' multicast, 32 columns per CTA, the
    last group partly past k_eff) is bit-identical to the dp4a kernel; ragged n and m."""
    X = make_video(333, 120, 161, seed=5, noise=2.0, n_rects=2)
    m, n = X.shape
    Xd = to_dev(X)
    P = C.Pipeline(H, n, n, m, "sparse", 300, 100, 6)
    P.sketch(Xd)
    P.fit()
    assert P.model.k_eff > 64 and C.cdmd_modes_path(P.model) == 2
    a = P.modes(Xd).clone()
    b = P.modes(Xd, simt=True).clone()
    assert torch.equal(a, b)


def test_sketch_slabs_sum_to_full(C, H):
    X = make_video(256, 90, 20, seed=8, noise=2.0, n_rects=1)
    m, n = X.shape
    for kind in ("spixel", "sparse", "rademacher"):
        full = C.Pipeline(H, n, n, m, kind, 64, 8, 2)
        full.sketch(to_dev(X))
        acc = torch.zeros_like(full.Y)
        for p0, nl in [(0, 128 * 60), (128 * 60, n - 128 * 60)]:
            P = C.Pipeline(H, n, nl, m, kind, 64, 8, 2, pix0=p0)
            acc += P.sketch(to_dev(X[:, p0:p0 + nl])).clone()
        assert torch.equal(acc, full.Y)


@pytest.mark.parametrize("W,Hh,m,p,slabs", [(1920, 1080, 500, 2000, 1), (333, 101, 77, 200, 1), (640, 360, 30, 600, 3)])
def test_sparse_sorted_sketch_equals_ell(C, H, W, Hh, m, p, slabs, monkeypatch):
    """The pixel-sorted sparse sketch (C sorted by pixel once per plan, cached by the
    handle; a CTA per 4 frames scattering into Y in shared memory) is bit-identical to the
    row-wise ELL gather kernel, on whole frames and on pixel slabs (pix0 > 0)."""
    X = make_video(W, Hh, m, seed=W + m, noise=2.0, n_rects=2)
    n = X.shape[1]
    from paper_1512_04205_b200.dist import slab
    for q in range(slabs):
        p0, nl = slab(n, slabs, q)
        Xd = to_dev(X[:, p0:p0 + nl])
        P = C.Pipeline(H, n, nl, m, "sparse", p, 8, 2, pix0=p0, seed=q + 3)
        a = P.sketch(Xd).clone()
        a2 = P.sketch(Xd).clone()                 # second call: the cached sorted C
        monkeypatch.setenv("CDMD_SPARSE_ELL", "1")
        b = P.sketch(Xd).clone()
        monkeypatch.delenv("CDMD_SPARSE_ELL")
        torch.cuda.synchronize()
        assert torch.equal(a, b) and torch.equal(a2, b), (q, p0, nl)
        if W < 1000:
            want = OS.sketch(X[:, p0:p0 + nl], OS.SPARSE, p, q + 3, n_total=n, pix0=p0)
            assert np.array_equal(a.cpu().numpy().T.astype(np.int64), want)


def test_srft_table_and_frequencies_bit_exact(C, H):
    """SRFT (reading R25): the device's fp16 quarter-wave table and the frequencies of R
    equal the oracle's bit for bit."""
    out = torch.zeros(16385, dtype=torch.int16, device="cuda")
    C.cdmd_srft_table(H, out)
    got = out.cpu().numpy().view(np.float16).astype(np.float64)
    r = np.arange(16385, dtype=np.float64)
    want = np.cos(2.0 * np.pi * r / 65536.0).astype(np.float16).astype(np.float64)
    assert np.array_equal(got, want)
    for n, p, seed in [(768, 200, 3), (2073600, 2000, 0), (97 * 61, 202, 0), (1000, 2000, 5)]:
        fr = torch.zeros(p // 2, dtype=torch.int32, device="cuda")
        C.cdmd_sensing_rows(H, n, C.sensing("srft", p, 0, seed), fr)
        assert np.array_equal(fr.cpu().numpy().astype(np.int64), OS.srft_freqs(n, p // 2, seed))


@pytest.mark.parametrize("W,Hh,m,p,slabs", [(160, 100, 50, 256, 1), (333, 101, 77, 202, 2), (720, 480, 300, 1500, 1)])
def test_srft_sketch_normwise(C, H, W, Hh, m, p, slabs):
    """The SRFT sketch on fp16 tensor cores (exact fp16 x fp16 products, fp32 sums) against
    the oracle's fp64 product with the same C, per column normwise <= 1e-4, on whole
    frames and on pixel slabs whose partial sketches add up."""
    X = make_video(W, Hh, m, seed=W + p, noise=2.0, n_rects=2)
    n = X.shape[1]
    from paper_1512_04205_b200.dist import slab
    acc = None
    for q in range(slabs):
        p0, nl = slab(n, slabs, q)
        P = C.Pipeline(H, n, nl, m, "srft", p, 8, 2, pix0=p0)
        Y = P.sketch(to_dev(X[:, p0:p0 + nl])).cpu().numpy().T.astype(np.float64)
        acc = Y if acc is None else acc + Y
    rows = np.arange(p) if W < 700 else np.r_[0:8, p // 2:p // 2 + 8, p - 4:p]
    want = OS.sketch(X, OS.SRFT, p, 0, rows=rows)
    d = np.linalg.norm(acc[rows] - want, axis=0) / np.linalg.norm(want, axis=0)
    assert d.max() <= PT.RTOL_Y_GAUSS, d.max()


def test_c3_rademacher_full_size_sampled_rows(C, H):
    cfg = config_by_name("c3_720x480_rademacher")
    X = video_for(cfg)
    m, n = X.shape
    P = C.Pipeline(H, n, n, m, "rademacher", cfg.p, cfg.k, cfg.K)
    Y = P.sketch(to_dev(X)).cpu().numpy().T
    # 64 rows over every 128-row tile of the tensor-core kernel: each tile's first and
    # last row and three random rows inside it (12 tiles at p = 1500, the last ragged)
    rng = np.random.default_rng(3)
    rows = set()
    for r0 in range(0, cfg.p, 128):
        r1 = min(cfg.p, r0 + 128)
        rows |= {r0, r1 - 1, *rng.integers(r0, r1, 3).tolist()}
    rows = sorted(rows)[:64] if len(rows) > 64 else sorted(rows)
    while len(rows) < 64:
        rows = sorted(set(rows) | {int(rng.integers(0, cfg.p))})
    want = OS.sketch(X, OS.RADEMACHER, cfg.p, 0, rows=rows)
    assert len(rows) == 64 and {r // 128 for r in rows} == set(range((cfg.p + 127) // 128))
    assert np.array_equal(Y[rows].astype(np.int64), want)


def test_c3_rademacher_full_pipeline(C, H):
    """BASELINE's C3 (720x480x300, Rademacher p = 1500, k = 30) through the whole path
    against the oracle: ALL 1500 rows of Y bit-exact (the oracle's slab sketches summed,
    computed in worker processes), the fit (sigma 1e-6, lambda 1e-4, supports), Phi on
    every pixel per column and the dynamic mask on every pixel."""
    from oracle.runner import PixelPool, parallel_sketch
    cfg = config_by_name("c3_720x480_rademacher")
    X = video_for(cfg)
    m, n = X.shape
    Xd = to_dev(X)
    P = C.Pipeline(H, n, n, m, "rademacher", cfg.p, cfg.k, cfg.K)
    Yg = P.sketch(Xd).cpu().numpy().T.astype(np.int64)
    P.fit()
    gm = C.model_to_host(P.model)
    Phi = P.modes(Xd).cpu().numpy()
    mask = P.foreground(Xd, cfg.tau, C.BG_DYNAMIC).cpu().numpy().view(np.uint32)
    torch.cuda.synchronize()
    del Xd
    Yo = parallel_sketch(cfg, OS.RADEMACHER)
    assert np.array_equal(Yg, Yo)
    om = OD.fit(Yo, cfg.k, cfg.K)
    assert gm["k_eff"] == om["k_eff"]
    perm, err = PT.match_eigs(gm["lam"], om["lam"])
    assert err <= PT.RTOL_EIG, err
    assert np.max(np.abs(gm["sigma"] - om["sigma"]) / om["sigma"]) <= 1e-6
    assert PT.supports_equal_mod_conj(gm["support"], gm["pair"], perm, om["support"], om["pair"])
    with PixelPool(cfg) as pool:
        ref = pool.run(om, cfg.tau, dynamic=True, want=("Phi", "mask", "band"))
    worst = _phi_columns_parity(PT.unfold(Phi, gm["pair"]), ref["Phi"], perm, om["lam"], gm["k_eff"])
    assert worst <= PT.RTOL_PHI, worst
    frac, outside, nd = _full_frame_mask_parity(mask, n, ref["mask"], ref["band"])
    print(f"c3 rademacher full: phi worst {worst:.2e}, mask agreement {frac:.7f} ({nd} px, {outside} outside band)")
    assert frac >= PT.MASK_AGREE and outside == 0, (frac, nd, outside)
    fm = fused_mask(C, P, to_dev(X), cfg.tau)   # N11 on the same model, when the support fits it
    torch.cuda.synchronize()
    if fm is not None:
        frac, outside, nd = _full_frame_mask_parity(fm, n, ref["mask"], ref["band"])
        print(f"c3 rademacher fused: mask agreement {frac:.7f} ({nd} px, {outside} outside band)")
        assert frac >= PT.MASK_AGREE and outside == 0, (frac, nd, outside)


def _phi_columns_parity(Pg, Po, perm, lam_o, k_eff):
    """Per-column relative error of the folded-then-unfolded device modes against the
    oracle's, after unit-phase alignment, over well-separated eigenvalues; returns the worst."""
    worst = 0.0
    for i in range(k_eff):
        j = perm[i]
        if PT.well_separated(lam_o, j):
            worst = max(worst, PT.phase_aligned_rel(Pg[:, i], Po[:, j]))
    return worst


def _full_frame_mask_parity(mask_words, n, ref_mask, band):
    """Whole-frame mask agreement: >= 99.9 % and every disagreement inside the oracle's
    1e-3 band around tau (band = |resid - tau| <= 1e-3, computed by the oracle)."""
    got = OD.unpack_mask(mask_words, n)
    dis = got != ref_mask
    frac = 1.0 - dis.mean()
    outside = int(np.count_nonzero(dis & ~band))
    return frac, outside, int(dis.sum())


def test_c4_sparse_full_size(C, H):
    """The bench configuration, in the bench's launch configuration, against the oracle
    on EVERY pixel: exact Y, fit parity, all n rows of Phi per column, and the whole
    1080p x 500 mask (the oracle's per-pixel steps fanned over pixel slabs)."""
    from oracle.runner import PixelPool
    cfg = config_by_name("c4_1080p_sparse")
    X = video_for(cfg)
    m, n = X.shape
    Xd = to_dev(X)
    P = C.Pipeline(H, n, n, m, "sparse", cfg.p, cfg.k, cfg.K)
    Yg = P.sketch(Xd).cpu().numpy().T.astype(np.int64)
    Yo = OS.sketch(X, OS.SPARSE, cfg.p, 0)
    assert np.array_equal(Yg, Yo)
    P.fit()
    gm = C.model_to_host(P.model)
    om = OD.fit(Yo, cfg.k, cfg.K)
    assert gm["k_eff"] == om["k_eff"]
    perm, err = PT.match_eigs(gm["lam"], om["lam"])
    assert err <= PT.RTOL_EIG
    assert np.max(np.abs(gm["sigma"] - om["sigma"]) / om["sigma"]) <= 1e-6
    assert PT.supports_equal_mod_conj(gm["support"], gm["pair"], perm, om["support"], om["pair"])
    Phi = P.modes(Xd).cpu().numpy()
    mask = P.foreground(Xd, cfg.tau, C.BG_DYNAMIC).cpu().numpy().view(np.uint32)
    torch.cuda.synchronize()
    del Xd
    with PixelPool(cfg) as pool:
        ref = pool.run(om, cfg.tau, dynamic=True, want=("Phi", "mask", "band"))
    worst = _phi_columns_parity(PT.unfold(Phi, gm["pair"]), ref["Phi"], perm, om["lam"], gm["k_eff"])
    assert worst <= PT.RTOL_PHI, worst
    frac, outside, nd = _full_frame_mask_parity(mask, n, ref["mask"], ref["band"])
    print(f"c4 sparse full frame: phi worst {worst:.2e}, mask agreement {frac:.7f} ({nd} px, {outside} outside band)")
    assert frac >= PT.MASK_AGREE and outside == 0, (frac, nd, outside)
    # N11: the fused single pass (no cdmd_modes call) on the same model, every pixel
    Xd = to_dev(X)
    fm = fused_mask(C, P, Xd, cfg.tau)
    torch.cuda.synchronize()
    assert fm is not None, "fused path unsupported at the bench configuration"
    frac, outside, nd = _full_frame_mask_parity(fm, n, ref["mask"], ref["band"])
    same = float((fm == mask).mean())
    print(f"c4 sparse fused: mask agreement {frac:.7f} ({nd} px, {outside} outside band), "
          f"words equal to the two-pass mask {same:.7f}")
    assert frac >= PT.MASK_AGREE and outside == 0, (frac, nd, outside)


def test_c4_gaussian_full_pipeline(C, H):
    """BASELINE's 1080p Gaussian(bf16) configuration through the whole path against the
    oracle: all 2000 rows of Y normwise per column (the oracle's sketch summed over pixel
    slabs computed in worker processes), then
      (a) the device fit on the device's fp32 Y against the oracle fit of that same Y:
          sigma to 1e-6, lambda to 1e-4, supports equal;
      (b) the Gaussian sketch's own effect, oracle fit of the oracle Y against oracle fit
          of the device Y: |d sigma_j| <= ||dY||_2 (Weyl) and lambda to 1e-4;
      (c) Phi (every pixel, per column) and the dynamic mask (every pixel) against the
          oracle with the model of (a)."""
    from oracle.runner import PixelPool, parallel_sketch
    cfg = config_by_name("c4_1080p_gaussian")
    X = video_for(cfg)
    m, n = X.shape
    Xd = to_dev(X)
    P = C.Pipeline(H, n, n, m, "gaussian", cfg.p, cfg.k, cfg.K)
    Yg = P.sketch(Xd).cpu().numpy().T.astype(np.float64)          # p x m
    P.fit()
    gm = C.model_to_host(P.model)
    Phi = P.modes(Xd).cpu().numpy()
    mask = P.foreground(Xd, cfg.tau, C.BG_DYNAMIC).cpu().numpy().view(np.uint32)
    torch.cuda.synchronize()
    del Xd
    Yo = parallel_sketch(cfg, OS.GAUSSIAN)
    d = np.linalg.norm(Yg - Yo, axis=0) / np.linalg.norm(Yo, axis=0)
    assert d.max() <= PT.RTOL_Y_GAUSS, d.max()
    # (a) the fit on identical input
    oa = OD.fit(Yg, cfg.k, cfg.K)
    assert gm["k_eff"] == oa["k_eff"]
    perm, err = PT.match_eigs(gm["lam"], oa["lam"])
    assert err <= PT.RTOL_EIG, err
    assert np.max(np.abs(gm["sigma"] - oa["sigma"]) / oa["sigma"]) <= 1e-6
    assert PT.supports_equal_mod_conj(gm["support"], gm["pair"], perm, oa["support"], oa["pair"])
    # (b) what the fp32 sketch changes (perturbation bounds on the same oracle)
    ob = OD.fit(Yo, cfg.k, cfg.K)
    dY2 = np.linalg.norm(Yg - Yo, 2)
    ks = min(oa["k_eff"], ob["k_eff"])
    assert np.all(np.abs(oa["sigma"][:ks] - ob["sigma"][:ks]) <= 2 * dY2)
    print(f"c4 gaussian: Y normwise max {d.max():.2e}, fit lambda {err:.2e}, "
          f"oracle(Yg) vs oracle(Yo) lambda {PT.match_eigs(oa['lam'], ob['lam'])[1]:.2e}")
    # (c) every pixel
    with PixelPool(cfg) as pool:
        ref = pool.run(oa, cfg.tau, dynamic=True, want=("Phi", "mask", "band"))
    worst = _phi_columns_parity(PT.unfold(Phi, gm["pair"]), ref["Phi"], perm, oa["lam"], gm["k_eff"])
    assert worst <= PT.RTOL_PHI, worst
    frac, outside, nd = _full_frame_mask_parity(mask, n, ref["mask"], ref["band"])
    print(f"c4 gaussian full frame: phi worst {worst:.2e}, mask agreement {frac:.7f} ({nd} px, {outside} outside band)")
    assert frac >= PT.MASK_AGREE and outside == 0, (frac, nd, outside)


def test_errors_are_reported_not_launched(C, H):
    X = to_dev(make_video(64, 32, 10, seed=1, noise=1.0, n_rects=0))
    v = C.video(X)
    Y = torch.zeros((10, 100), dtype=torch.int32, device="cuda")
    ws = torch.zeros(1 << 20, dtype=torch.uint8, device="cuda")
    with pytest.raises(C.CdmdError) as e:
        C.cdmd_sketch(H, v, C.sensing("sparse", 5000), Y, ws)     # p > n
    assert e.value.code == 2
    with pytest.raises(C.CdmdError) as e:
        C.cdmd_sketch(H, v, C.sensing("sparse", 50, 0.5), Y, ws)  # s <= 1
    assert e.value.code == 2
    P = C.Pipeline(H, 2048, 2048, 10, "sparse", 50, 8, 2)
    P.sketch(X)
    with pytest.raises(C.CdmdError) as e:
        C.cdmd_fit(H, P.Y, "sparse", 50, 10, 10, 2, P.model, P.ws_fit)   # k > m - 1
    assert e.value.code == 2
    P.fit()
    P.modes(X)
    with pytest.raises(C.CdmdError) as e:
        C.cdmd_foreground(H, v, P.model, P.Phi, C.BG_DYNAMIC, 0.0, P.mask)  # tau <= 0
    assert e.value.code == 2


@pytest.mark.parametrize("k,seed", [(1, 0), (2, 1), (5, 2), (17, 3), (50, 4), (64, 5), (100, 6), (118, 7)])
def test_device_eig_matches_lapack(C, k, seed):
    """The on-device Hessenberg/Francis-QR eigensolver (cdmd_eig) vs LAPACK (numpy)."""
    rng = np.random.default_rng(seed)
    A = rng.standard_normal((k, k))
    if k >= 5:  # plant a few conjugate pairs on the unit circle and a repeated-modulus set
        Q, _ = np.linalg.qr(rng.standard_normal((k, k)))
        D = np.diag(rng.uniform(0.2, 1.0, k))
        for b in range(0, min(k - 1, 8), 2):
            c, s_ = np.cos(0.3 * (b + 1)), np.sin(0.3 * (b + 1))
            D[b:b + 2, b:b + 2] = [[c, -s_], [s_, c]]
        A = Q @ D @ Q.T
    Ad = torch.from_numpy(A.T.copy()).cuda()     # column-major A
    W = torch.zeros(2 * k, dtype=torch.float64, device="cuda")
    VR = torch.zeros(k * k, dtype=torch.float64, device="cuda")
    info = torch.full((1,), -1, dtype=torch.int32, device="cuda")
    C.cdmd_eig(Ad, W, VR, info)
    assert int(info.item()) == 0
    w = W.cpu().numpy().reshape(k, 2)
    lam = w[:, 0] + 1j * w[:, 1]
    V = VR.cpu().numpy().reshape(k, k).T          # column j = VR[:, j]
    ref = np.linalg.eigvals(A)
    perm, err = PT.match_eigs(lam, ref)
    assert err < 1e-10
    j = 0
    while j < k:   # A v = lambda v for every (complex) eigenvector
        if w[j, 1] == 0:
            v = V[:, j]
            jn = 1
        else:
            assert w[j, 1] > 0 and w[j + 1, 1] == -w[j, 1] and w[j + 1, 0] == w[j, 0]
            v = V[:, j] + 1j * V[:, j + 1]
            jn = 2
        res = np.linalg.norm(A @ v - lam[j] * v) / (np.linalg.norm(A) * np.linalg.norm(v))
        assert res < 1e-12, (j, res)
        j += jn


@pytest.mark.parametrize("W,Hh,m,p", [(720, 480, 300, 1500), (333, 101, 77, 200), (128, 8, 600, 130)])
def test_rademacher_tensor_core_sketch_equals_simt(C, H, W, Hh, m, p, monkeypatch):
    """tcgen05 kind::i8 split-K sketch vs the dp4a kernel: both exact int32 -> identical."""
    X = make_video(W, Hh, m, seed=W + m, noise=2.0, n_rects=1)
    n = X.shape[1]
    Xd = to_dev(X)
    P = C.Pipeline(H, n, n, m, "rademacher", p, 8, 2)
    a = P.sketch(Xd).clone()
    monkeypatch.setenv("CDMD_SIMT_SKETCH", "1")
    b = P.sketch(Xd).clone()
    assert torch.equal(a, b)
    rows = [0, p // 2, p - 1]
    want = OS.sketch(X, OS.RADEMACHER, p, 0, rows=rows)
    assert np.array_equal(a.cpu().numpy().T[rows].astype(np.int64), want)


@pytest.mark.parametrize("W,Hh,m,p", [(160, 100, 50, 256), (333, 101, 77, 200), (720, 480, 300, 500)])
def test_gaussian_tensor_core_sketch(C, H, W, Hh, m, p, monkeypatch):
    """tcgen05 kind::f16 sketch (fp32 accumulation) vs the fp64-chunked SIMT kernel and
    the oracle: per-column normwise <= 1e-4 (north_star), in practice ~1e-6."""
    X = make_video(W, Hh, m, seed=W + 3 * m, noise=2.0, n_rects=1)
    n = X.shape[1]
    Xd = to_dev(X)
    P = C.Pipeline(H, n, n, m, "gaussian", p, 8, 2)
    a = P.sketch(Xd).clone().cpu().numpy().T.astype(np.float64)
    monkeypatch.setenv("CDMD_SIMT_SKETCH", "1")
    b = P.sketch(Xd).clone().cpu().numpy().T.astype(np.float64)
    rows = [0, p // 3, p - 1]
    want = OS.sketch(X, OS.GAUSSIAN, p, 0, rows=rows)
    for got in (a, b):
        d = np.linalg.norm(got[rows] - want, axis=1) / np.linalg.norm(want, axis=1)
        assert d.max() <= PT.RTOL_Y_GAUSS, d.max()
    col = np.linalg.norm(a - b, axis=0) / np.linalg.norm(b, axis=0)
    assert col.max() <= 1e-5, col.max()


def test_streaming_lanes_equal_sequential(C, H):
    """The measured path: batches through cdmd.Streaming (lanes with their own handle,
    streams, buffers; the fit on a high-priority stream) give bit-identical sketches,
    limbs of M and masks to one batch at a time through Pipeline, at the bench size."""
    cfg = config_by_name("c4_1080p_sparse")
    X = video_for(cfg)
    m, n = X.shape
    X0 = to_dev(X)
    vids = [X0, X0.flip(0).contiguous(), X0.roll(7, dims=0).contiguous(), X0.flip(0).roll(3, dims=0).contiguous(),
            X0.roll(-11, dims=0).contiguous()]
    S = C.Streaming(0, n, n, m, "sparse", cfg.p, cfg.k, cfg.K, lanes=3, seed=cfg.sensing_seed)
    ends = S.run(vids, cfg.tau, C.BG_DYNAMIC)
    for e in ends:
        torch.cuda.current_stream().wait_event(e)
    torch.cuda.synchronize()
    P = C.Pipeline(H, n, n, m, "sparse", cfg.p, cfg.k, cfg.K, seed=cfg.sensing_seed)
    for li, (_, _, _, pipe) in enumerate(S.lanes):
        last = max(b for b in range(len(vids)) if b % 3 == li)
        mask = P.run(vids[last], cfg.tau, C.BG_DYNAMIC)
        torch.cuda.synchronize()
        assert torch.equal(pipe.Y, P.Y), li
        assert torch.equal(pipe.mask, mask), li
        assert pipe.model.k_eff == P.model.k_eff and pipe.model.K_eff == P.model.K_eff
        assert torch.equal(pipe.Phi, P.Phi), li


def test_gaussian_sketch_deterministic_full_size(C, H, monkeypatch):
    """Split-K partial sums are reduced in a fixed order: the 1080p Gaussian sketch is
    bit-identical from run to run (a race between the CTA pair's producers and the
    leader's MMAs would show up here), for the paired and the single-CTA kernels."""
    cfg = config_by_name("c4_1080p_gaussian")
    X = video_for(cfg)
    m, n = X.shape
    Xd = to_dev(X)
    P = C.Pipeline(H, n, n, m, "gaussian", cfg.p, cfg.k, cfg.K)
    ys = []
    for single in (False, True):
        if single:
            monkeypatch.setenv("CDMD_GAUSS_1CTA", "1")
        runs = [P.sketch(Xd).clone() for _ in range(3)]
        torch.cuda.synchronize()
        for r in runs[1:]:
            assert torch.equal(r, runs[0]), single
        ys.append(runs[0].double())
    # the two kernels differ only in the split-K summation order
    d = torch.linalg.norm(ys[0] - ys[1], dim=1) / torch.linalg.norm(ys[1], dim=1)
    assert float(d.max()) <= PT.RTOL_Y_GAUSS


@pytest.mark.parametrize("case", ["c1", "ragged_sparse", "rademacher_small", "c2", "long_m"])
def test_pipeline_parity_gavish_donoho(C, H, case):
    """Automatic target rank (Remark 2): the device's Gavish-Donoho rank
    (median singular value by bisection on the tridiagonal form) equals the oracle's,
    and the rest of the path keeps parity at that rank."""
    if case == "c2":
        cfg = config_by_name("c2_320x240_spixel")
        X, kind, p, k, K, tau = video_for(cfg), cfg.kind, cfg.p, cfg.k, cfg.K, cfg.tau
    elif case == "long_m":   # m - 1 = 599 > 510: the full cuSOLVER syevd path of the GD rank
        X, kind, p, k, K, tau = make_video(200, 96, 600, seed=21, noise=2.0, n_rects=1), "sparse", 800, 30, 6, 25.0
    else:
        name, shape, kind, p, k, K, tau = next(c for c in CASES if c[0] == case)
        if shape is None:
            X = video_for(config_by_name("c1_32x24_sparse"))
        else:
            W, Hh, m, noise, rects = shape
            X = make_video(W, Hh, m, seed=zlib.crc32(name.encode()) % 1000, noise=noise, n_rects=rects)
    g = gpu_run(C, H, X, kind, p, k, K, tau, rank="gd")
    o = oracle_run(X, kind, p, k, K, tau, rank="gd")
    assert g["model"]["k_eff"] == o["model"]["k_eff"]
    assert 1 <= o["model"]["k_eff"] <= k
    check_all(g, o, kind, tau)


def _omega_gap_eps(omega, want):
    """A threshold between |omega| values with a clear gap, selecting about `want`
    modes (never splitting equal |omega|, e.g. a conjugate pair)."""
    a = np.sort(np.abs(omega))
    for i in list(range(want - 1, len(a) - 1)) + list(range(want - 2, -1, -1)):
        if a[i + 1] - a[i] > 1e-2 * max(1.0, a[i + 1]):
            return 0.5 * (a[i] + a[i + 1])
    pytest.skip("no clear |omega| gap")


@pytest.mark.parametrize("case,want", [("c1", 1), ("ragged_sparse", 3), ("c2", 2)])
def test_pipeline_parity_frequency_background(C, H, case, want):
    """Background by frequency (|omega| < eps instead of OMP): the device selects
    the same modes as the oracle and the amplitudes, backgrounds and masks keep parity.
    eps sits in a clear gap of the oracle's |omega| (a threshold decision: both sides
    see the same gap)."""
    if case == "c2":
        cfg = config_by_name("c2_320x240_spixel")
        X, kind, p, k, K, tau = video_for(cfg), cfg.kind, cfg.p, cfg.k, cfg.K, cfg.tau
    elif case == "c1":
        cfg = config_by_name("c1_32x24_sparse")
        X, kind, p, k, K, tau = video_for(cfg), cfg.kind, cfg.p, cfg.k, cfg.K, cfg.tau
    else:
        name, shape, kind, p, k, K, tau = next(c for c in CASES if c[0] == case)
        W, Hh, m, noise, rects = shape
        X = make_video(W, Hh, m, seed=zlib.crc32(name.encode()) % 1000, noise=noise, n_rects=rects)
    Y = OS.sketch(X, KIND[kind], p, 0)
    eps = _omega_gap_eps(OD.fit(Y, k, K)["omega"], want)
    g = gpu_run(C, H, X, kind, p, k, K, tau, omega_eps=eps)
    o = oracle_run(X, kind, p, k, K, tau, omega_eps=eps, Y=Y)
    assert len(o["model"]["support"]) >= 1
    check_all(g, o, kind, tau)


def test_frequency_background_capped_at_K(C, H):
    """More slow modes than the model's K (reading R24): the device keeps the first K of
    them in mode order, like the oracle, and writes nothing past the model's K-sized
    arrays (the model buffer is followed by a guard region checked unchanged)."""
    cfg = config_by_name("c2_320x240_spixel")
    X = video_for(cfg)
    m, n = X.shape
    k, K = cfg.k, 3
    Y = OS.sketch(X, KIND[cfg.kind], cfg.p, 0)
    om_all = OD.fit(Y, k, K)["omega"]
    eps = float(np.max(np.abs(om_all))) + 1.0          # every mode qualifies
    Xd = to_dev(X)
    P = C.Pipeline(H, n, n, m, cfg.kind, cfg.p, k, K, omega_eps=eps)
    nb = P.model_buf.numel()
    guard = torch.full((nb + 4096,), 0x5A, dtype=torch.uint8, device="cuda")
    guard[:nb] = P.model_buf
    P.model_buf = guard[:nb]                              # rebind the model inside the guarded buffer
    P.model = C.cdmd_model_bind(P.model_buf, k, K, m)
    g = gpu_run_pipeline(C, P, Xd, X, cfg.tau)
    torch.cuda.synchronize()
    assert bool((guard[nb:] == 0x5A).all()), "write past the model buffer"
    o = oracle_run(X, cfg.kind, cfg.p, k, K, cfg.tau, omega_eps=eps, Y=Y)
    assert len(o["model"]["support"]) == K and g["model"]["K_eff"] == K
    check_all(g, o, cfg.kind, cfg.tau)


def gpu_run_pipeline(C, P, Xd, X, tau):
    """gpu_run on an existing Pipeline (same outputs)."""
    m, n = X.shape
    Y = P.sketch(Xd).cpu().numpy().T.copy()
    P.fit()
    out = dict(Y=Y, model=C.model_to_host(P.model), Phi=P.modes(Xd).cpu().numpy())
    for mode, name in ((C.BG_DYNAMIC, "dyn"), (C.BG_STATIC, "sta")):
        out["mask_" + name] = OD.unpack_mask(P.foreground(Xd, tau, mode).cpu().numpy().view(np.uint32), n)
        out["L_" + name] = P.background(mode).cpu().numpy()
    return out


def test_sparse_plan_check_refused_inside_graph_capture(C):
    """The first sketch of a new sparse plan checks the index lists once with a stream
    sync; inside a CUDA graph capture that is refused (CDMD_ERR_ARG) instead of silently
    skipped, and after one eager call the same plan captures fine."""
    H2 = C.Handle(0)
    X = make_video(64, 48, 12, seed=2, noise=1.0, n_rects=1)
    m, n = X.shape
    Xd = to_dev(X)
    P = C.Pipeline(H2, n, n, m, "sparse", 40, 4, 2, seed=77)
    s = torch.cuda.Stream()
    g = torch.cuda.CUDAGraph()
    with pytest.raises(C.CdmdError) as e:
        with torch.cuda.graph(g, stream=s):
            P.sketch(Xd, s)
    assert e.value.code == 1
    torch.cuda.synchronize()
    P.sketch(Xd)
    want = P.Y.clone()
    P.Y.zero_()
    g2 = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g2, stream=s):
        P.sketch(Xd, s)
    g2.replay()
    torch.cuda.synchronize()
    assert torch.equal(P.Y, want)


@pytest.mark.parametrize("W,Hh,m,dens,pad", [(37, 23, 5, 0.35, 3), (64, 16, 3, 0.5, 3), (720, 480, 4, 0.1, 3),
                                             (5, 3, 2, 0.6, 3), (33, 1, 2, 0.5, 3), (1, 40, 2, 0.5, 3),
                                             # word-aligned rows (W % 128 == 0, ldw % 4 == 0): the vectorised kernel
                                             (256, 37, 5, 0.4, 4), (128, 1, 3, 0.5, 0), (384, 2, 2, 0.55, 0),
                                             (1920, 9, 3, 0.2, 0), (512, 64, 2, 0.9, 8)])
def test_mask_median3_bit_exact(C, W, Hh, m, dens, pad):
    """3x3 median post-filter (Fig. 7): bit-exact against the oracle on random
    masks (widths that are not multiples of 32 straddle words across image rows; widths
    that are multiples of 128 take the vectorised word-aligned kernel)."""
    rng = np.random.default_rng(W * 1000 + Hh)
    n = W * Hh
    M = rng.random((m, n)) < dens
    ldw = (n + 31) // 32 + pad
    packed = np.zeros((m, ldw), dtype=np.uint32)
    packed[:, :(n + 31) // 32] = OD.pack_mask(M)
    dev = torch.from_numpy(packed.view(np.int32)).cuda()
    out = torch.full_like(dev, -1)
    C.cdmd_mask_median3(dev, W, Hh, out)
    got = OD.unpack_mask(out.cpu().numpy().view(np.uint32)[:, :(n + 31) // 32], n)
    assert np.array_equal(got, OD.median3(M, W, Hh))


def test_mask_median3_on_the_bench_mask(C, H):
    """The filter applied to the 1080p dynamic-background mask the bench produces."""
    cfg = config_by_name("c4_1080p_sparse")
    X = video_for(cfg)
    m, n = X.shape
    Xd = to_dev(X)
    P = C.Pipeline(H, n, n, m, "sparse", cfg.p, cfg.k, cfg.K)
    P.run(Xd, cfg.tau, C.BG_DYNAMIC)
    filt = P.median3(cfg.width, cfg.height)
    torch.cuda.synchronize()
    raw = OD.unpack_mask(P.mask.cpu().numpy().view(np.uint32), n)
    got = OD.unpack_mask(filt.cpu().numpy().view(np.uint32), n)
    ref = OD.median3(raw, cfg.width, cfg.height)
    assert np.array_equal(got, ref)
    assert got.sum() <= raw.sum() + raw.size // 100    # the filter mostly removes isolated noise bits


def test_c5_4k_full_size_sampled(C, H):
    """BASELINE's 4K configuration (3840x2160, 1000 frames, sparse p = 4000, k = 100) on
    one GPU: exact integer sketch, fit parity (m - 1 = 999: the streamed-G Lanczos variant,
    no fallback; k = 100: the device eig), sigma to 1e-6, modes and mask on sampled pixels
    incl. the ragged tail (k = 100 and m = 1000 take the CUDA-core modes /
    dynamic-foreground kernels)."""
    cfg = config_by_name("c5_4k_sparse")
    X = video_for(cfg)
    m, n = X.shape
    Xd = to_dev(X)
    P = C.Pipeline(H, n, n, m, "sparse", cfg.p, cfg.k, cfg.K)
    Yg = P.sketch(Xd).cpu().numpy().T.astype(np.int64)
    Yo = OS.sketch(X, OS.SPARSE, cfg.p, 0)
    assert np.array_equal(Yg, Yo)
    runs0, fb0 = C.cdmd_eigensolver_stats(H)
    P.fit()
    runs1, fb1 = C.cdmd_eigensolver_stats(H)
    assert (runs1 - runs0, fb1 - fb0) == (1, 0), (runs1 - runs0, fb1 - fb0)
    gm = C.model_to_host(P.model)
    om = OD.fit(Yo, cfg.k, cfg.K)
    assert gm["k_eff"] == om["k_eff"]
    perm, err = PT.match_eigs(gm["lam"], om["lam"])
    assert err <= PT.RTOL_EIG
    assert np.max(np.abs(gm["sigma"] - om["sigma"]) / om["sigma"]) <= 1e-6
    assert PT.supports_equal_mod_conj(gm["support"], gm["pair"], perm, om["support"], om["pair"])
    Phi = P.modes(Xd)
    mask = P.foreground(Xd, cfg.tau, C.BG_DYNAMIC).cpu().numpy().view(np.uint32)
    torch.cuda.synchronize()
    rng = np.random.default_rng(5)
    pix = np.unique(np.concatenate([rng.choice(n, 2048, replace=False), np.arange(n - 40, n)]))
    Po = X[1:, pix].T.astype(np.float64) @ om["M"]
    Pg = PT.unfold(Phi.cpu().numpy()[:, pix], gm["pair"])
    for i in range(gm["k_eff"]):
        j = perm[i]
        if PT.well_separated(om["lam"], j):
            assert PT.phase_aligned_rel(Pg[:, i], Po[:, j]) <= PT.RTOL_PHI
    Ld = OD.background_dynamic(Po, om)
    res = np.abs(X[:, pix].astype(np.float64) - Ld.T)
    mg = OD.unpack_mask(mask, n)[:, pix]
    frac, band, nd = PT.mask_agreement(mg, res > cfg.tau, res, cfg.tau)
    assert frac >= PT.MASK_AGREE and band, (frac, nd)


_PARTITION_SCRIPT = r"""
import os, sys, torch
# the same eigensolver on both sides: the fit partition's green context may not hold a
# 16-SM cluster, where cdmd_fit's Lanczos falls back to the Householder solver
os.environ["CDMD_SYEV"] = "h"
sys.path.insert(0, sys.argv[1])
from paper_1512_04205_b200 import cdmd as C
from synth.scene import config_by_name, video_for
cfg = config_by_name("c4_1080p_sparse")
X = video_for(cfg)
m, n = X.shape
ld = ((n + 15) // 16) * 16
X0 = torch.zeros((m, ld), dtype=torch.uint8, device="cuda")
X0[:, :n] = torch.from_numpy(X).cuda()
vids = [X0, X0.flip(0).contiguous(), X0.roll(5, dims=0).contiguous(), X0.roll(-9, dims=0).contiguous()]
S = C.Streaming(0, n, n, m, "sparse", cfg.p, cfg.k, cfg.K, lanes=2, seed=cfg.sensing_seed, fit_sms=32)
assert S.sms[0] >= 32 and S.sms[0] + S.sms[1] == torch.cuda.get_device_properties(0).multi_processor_count, S.sms
ends = S.run(vids, cfg.tau, C.BG_DYNAMIC)
for e in ends:
    torch.cuda.current_stream().wait_event(e)
torch.cuda.synchronize()
H = C.Handle(0)
P = C.Pipeline(H, n, n, m, "sparse", cfg.p, cfg.k, cfg.K, seed=cfg.sensing_seed)
for li, (_, _, _, pipe) in enumerate(S.lanes):
    mask = P.run(vids[2 + li], cfg.tau, C.BG_DYNAMIC)
    torch.cuda.synchronize()
    assert torch.equal(pipe.Y, P.Y) and torch.equal(pipe.Phi, P.Phi) and torch.equal(pipe.mask, mask), li
print("partition ok", S.sms)
"""


def test_streaming_sm_partition_equal_sequential(tmp_path):
    """cdmd_sm_partition (green contexts: SMs reserved for the small solves, persistent
    grids sized to the rest) changes scheduling only: lanes on the partition streams
    give bit-identical sketches, modes and masks to Pipeline.  Run in a subprocess: the
    partition is process-wide."""
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    script = tmp_path / "partition_check.py"
    script.write_text(_PARTITION_SCRIPT)
    r = subprocess.run([sys.executable, str(script), root], cwd=root, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-4000:]
    assert "partition ok" in r.stdout


_SHARDED_SCRIPT = r"""
import os, sys, numpy as np, torch
import torch.distributed as dist
sys.path.insert(0, sys.argv[1])
out_dir = sys.argv[2]
rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
dist.init_process_group("gloo", rank=rank, world_size=world)
from paper_1512_04205_b200 import cdmd as C
from paper_1512_04205_b200.dist import slab
from synth.scene import make_video
W, H, m, p, k, K, tau = 640, 360, 120, 600, 20, 6, 25.0
n = W * H
pix0, nl = slab(n, world, rank)
Xs = make_video(W, H, m, seed=11, noise=2.0, n_rects=2, pix0=pix0, n_local=nl)
ld = ((nl + 15) // 16) * 16
X0 = torch.zeros((m, ld), dtype=torch.uint8, device="cuda")
X0[:, :nl] = torch.from_numpy(Xs).cuda()
shifts = [0, 5, -9]                      # batch b = the video rolled by shifts[b] frames
vids = [X0.roll(sh, dims=0).contiguous() for sh in shifts]
ar = lambda Y: dist.all_reduce(Y, op=dist.ReduceOp.SUM)
S = C.Streaming(0, n, nl, m, "sparse", p, k, K, lanes=3, pix0=pix0)
ends = S.run(vids, tau, C.BG_DYNAMIC, allreduce=ar)
for e in ends:
    torch.cuda.current_stream().wait_event(e)
torch.cuda.synchronize()
res = {}
for b, (_, _, _, pipe) in enumerate(S.lanes):      # lane b ran batch b (3 lanes, 3 batches)
    mh = C.model_to_host(pipe.model)
    res[f"Y{b}"] = pipe.Y.cpu().numpy()
    res[f"Phi{b}"] = pipe.Phi[:pipe.model.k_eff].cpu().numpy()
    res[f"mask{b}"] = pipe.mask.cpu().numpy()
    for key in ("lam", "sigma", "pair", "support"):
        res[f"{key}{b}"] = np.asarray(mh[key])
np.savez(os.path.join(out_dir, f"rank{rank}.npz"), pix0=pix0, nl=nl, **res)
dist.barrier()
dist.destroy_process_group()
sys.stdout.write(f"sharded ok {rank}\n")
sys.stdout.flush()
"""


def test_two_rank_sharded_path_equals_single_process_oracle(tmp_path):
    """The pixel-row-sharded path through libcdmd on two ranks
    (gloo, both on cuda:0: host-mediated all-reduces, no kernel waits on another rank's):
    each rank sketches its slab with C's global columns, the streaming lanes all-reduce
    Y in batch order, every rank fits, and modes + masks of the two slabs, put side by
    side, are compared with the SINGLE-PROCESS oracle on the whole video, per batch."""
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    script = tmp_path / "sharded_check.py"
    script.write_text(_SHARDED_SCRIPT)
    port = 29500 + (os.getpid() % 1000)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr=127.0.0.1", f"--master-port={port}", str(script), root, str(tmp_path)]
    r = subprocess.run(cmd, cwd=root, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-4000:]
    R = [np.load(tmp_path / f"rank{q}.npz") for q in (0, 1)]
    W, Hh, m, p, k, K, tau = 640, 360, 120, 600, 20, 6, 25.0
    X = make_video(W, Hh, m, seed=11, noise=2.0, n_rects=2)
    n = X.shape[1]
    assert int(R[0]["pix0"]) == 0 and int(R[0]["nl"]) + int(R[1]["nl"]) == n
    for b, sh in enumerate([0, 5, -9]):
        Xb = np.roll(X, sh, axis=0)
        Yo = OS.sketch(Xb, OS.SPARSE, p, 0)
        om = OD.fit(Yo, k, K)
        Phi_o = OD.modes(Xb, om["M"])
        L = OD.background_dynamic(Phi_o, om)
        res = np.abs(Xb.astype(np.float64) - L.T)
        for q in (0, 1):   # every rank holds the same all-reduced Y and the same model
            assert np.array_equal(R[q][f"Y{b}"].T.astype(np.int64), Yo), (b, q)
            assert list(R[q][f"pair{b}"]) == list(R[0][f"pair{b}"])
            assert np.array_equal(R[q][f"lam{b}"], R[0][f"lam{b}"])
        lam_g = R[0][f"lam{b}"]
        perm, err = PT.match_eigs(lam_g, om["lam"])
        assert err <= PT.RTOL_EIG and len(lam_g) == om["k_eff"]
        assert PT.supports_equal_mod_conj(list(R[0][f"support{b}"]), R[0][f"pair{b}"], perm, om["support"], om["pair"])
        Phi_g = np.concatenate([R[q][f"Phi{b}"][:, :int(R[q]["nl"])] for q in (0, 1)], axis=1)
        worst = _phi_columns_parity(PT.unfold(Phi_g, R[0][f"pair{b}"]), Phi_o, perm, om["lam"], len(lam_g))
        assert worst <= PT.RTOL_PHI, (b, worst)
        mg = np.concatenate([OD.unpack_mask(R[q][f"mask{b}"].view(np.uint32), int(R[q]["nl"])) for q in (0, 1)], axis=1)
        frac, band, nd = PT.mask_agreement(mg, res > tau, res, tau)
        assert frac >= PT.MASK_AGREE and band, (b, frac, nd)


# ------------------------------------------- amplitudes b = lstsq(Phi, x_1)
AMP_CASES = [
    # name, (W, H, m, noise, rects) or None (C1), kind, p, k
    ("c1", None, "sparse", 50, 10),
    ("ragged_sparse", (100, 37, 33, 2.0, 1), "sparse", 120, 12),
    ("rademacher_small", (180, 120, 60, 2.0, 2), "rademacher", 300, 20),
    ("k50_ragged", (333, 101, 77, 2.0, 2), "sparse", 200, 50),
    ("k100", (256, 160, 150, 2.0, 2), "sparse", 400, 100),
]


@pytest.mark.parametrize("case", AMP_CASES, ids=[c[0] for c in AMP_CASES])
def test_amplitudes_parity(C, H, case):
    name, shape, kind, p, k = case
    if shape is None:
        X = video_for(config_by_name("c1_32x24_sparse"))
    else:
        W, Hh, m, noise, rects = shape
        X = make_video(W, Hh, m, seed=zlib.crc32(name.encode()) % 1000, noise=noise, n_rects=rects)
    m, n = X.shape
    K = min(2, k)
    Xd = to_dev(X)
    P = C.Pipeline(H, n, n, m, kind, p, k, K)
    P.sketch(Xd)
    P.fit()
    F = P.modes(Xd)
    b, dropped = P.amplitudes(Xd)
    torch.cuda.synchronize()
    mh = C.model_to_host(P.model)
    b = b.cpu().numpy()
    assert int(dropped.item()) == 0
    # (1) step 9 alone: the oracle's lstsq on the GPU's own modes (same input), within
    # north_star's 1e-4 relative for fp32-level quantities
    Phi_g = PT.unfold(F.cpu().numpy(), mh["pair"])
    b_o = OD.amplitudes(X, Phi_g)
    cond = np.linalg.cond(Phi_g)
    err1 = np.linalg.norm(b - b_o) / np.linalg.norm(b_o)
    assert err1 <= PT.RTOL_PHI, (err1, cond)
    for j in np.nonzero(mh["pair"] == 1)[0]:
        assert b[j + 1] == np.conj(b[j])
    # (2) end to end against the oracle's modes: per-mode contributions b_j phi_j
    # (invariant to each mode's phase normalisation) and the reconstruction of x_1
    o = OD.fit(OS.sketch(X, KIND[kind], p, 0), k, K)
    Phi_o = OD.modes(X, o["M"])
    bo = OD.amplitudes(X, Phi_o)
    perm, werr = PT.match_eigs(mh["lam"], o["lam"])
    assert werr <= PT.RTOL_EIG
    x1 = np.linalg.norm(X[0].astype(np.float64))
    rec_g = (Phi_g @ b).real
    rec_o = (Phi_o @ bo).real
    assert np.linalg.norm(rec_g - rec_o) <= 1e-4 * x1, np.linalg.norm(rec_g - rec_o) / x1
    worst = 0.0
    for i, j in enumerate(perm):
        if PT.well_separated(o["lam"], j, 1e-3):
            worst = max(worst, np.linalg.norm(b[i] * Phi_g[:, i] - bo[j] * Phi_o[:, j]) / x1)
    print(f"{name}: k_eff={mh['lam'].size} cond={cond:.3g} step9_rel={err1:.2e} contrib={worst:.2e}")
    assert worst <= PT.RTOL_PHI   # b_j phi_j inherits the north_star modes tolerance


def test_amplitudes_slabs_sum_to_full(C, H):
    # pixel-row sharding: Gram partials of two slabs sum to the whole-video Gram
    X = make_video(320, 120, 60, seed=11, noise=2.0, n_rects=2)
    m, n = X.shape
    Xd = to_dev(X)
    P = C.Pipeline(H, n, n, m, "sparse", 200, 16, 4)
    P.sketch(Xd)
    P.fit()
    F = P.modes(Xd)
    ke = P.model.k_eff
    ws = torch.empty(C.cdmd_amplitudes_workspace_bytes(H, ke), dtype=torch.uint8, device="cuda")
    G = torch.empty((ke + 1, ke), dtype=torch.float64, device="cuda")
    C.cdmd_amplitudes_gram(H, C.video(Xd, n, 0, n), P.model, P.Phi, G, ws)
    with pytest.raises(C.CdmdError):   # CDMD_ERR_WORKSPACE, reported before any launch
        C.cdmd_amplitudes_gram(H, C.video(Xd, n, 0, n), P.model, P.Phi, G, ws[:256])
    n1 = 128 * 97
    Gs = torch.zeros_like(G)
    for pix0, nl in ((0, n1), (n1, n - n1)):
        Gp = torch.empty_like(G)
        C.cdmd_amplitudes_gram(H, C.video(Xd[:, pix0:], n, pix0, nl), P.model, P.Phi[:, pix0:], Gp, ws)
        Gs += Gp
    torch.cuda.synchronize()
    G, Gs = G.cpu().numpy(), Gs.cpu().numpy()
    assert np.max(np.abs(G - Gs)) <= 8e-6 * np.max(np.abs(G))
    # and the Gram itself equals the fp64 product of the (exact) fp32 modes
    Ff = F.cpu().numpy().astype(np.float64)
    ref = np.concatenate([Ff @ Ff.T, Ff @ X[0].astype(np.float64)[:, None]], 1)   # k x (k+1)
    assert np.max(np.abs(G.T - ref)) <= 8e-6 * np.max(np.abs(ref))


def test_amplitudes_c4_full_size(C, H):
    """Step 9 at the bench configuration (1080p x 500, k = 50), in the launch
    configuration bench.py times: device b vs the oracle's lstsq on the same modes."""
    cfg = config_by_name("c4_1080p_sparse")
    X = video_for(cfg)
    m, n = X.shape
    Xd = to_dev(X)
    P = C.Pipeline(H, n, n, m, "sparse", cfg.p, cfg.k, cfg.K)
    P.sketch(Xd)
    P.fit()
    F = P.modes(Xd)
    b, dropped = P.amplitudes(Xd)
    torch.cuda.synchronize()
    assert int(dropped.item()) == 0
    mh = C.model_to_host(P.model)
    Phi_g = PT.unfold(F.cpu().numpy(), mh["pair"])
    del F
    b = b.cpu().numpy()
    b_o = OD.amplitudes(X, Phi_g)
    err = np.linalg.norm(b - b_o) / np.linalg.norm(b_o)
    assert err <= PT.RTOL_PHI, err
    # end to end: per-mode contributions b_j phi_j against the oracle's own modes and
    # amplitudes (full frame, the oracle's modes fanned over pixel slabs)
    from oracle.runner import PixelPool
    o = OD.fit(OS.sketch(X, OS.SPARSE, cfg.p, 0), cfg.k, cfg.K)
    with PixelPool(cfg) as pool:
        Phi_o = pool.run(o, cfg.tau, want=("Phi",))["Phi"]
    bo = OD.amplitudes(X, Phi_o)
    perm, werr = PT.match_eigs(mh["lam"], o["lam"])
    assert werr <= PT.RTOL_EIG
    x1 = np.linalg.norm(X[0].astype(np.float64))
    worst = 0.0
    for i, j in enumerate(perm):
        if PT.well_separated(o["lam"], j, 1e-3):
            worst = max(worst, np.linalg.norm(b[i] * Phi_g[:, i] - bo[j] * Phi_o[:, j]) / x1)
    print(f"c4 amplitudes: step9_rel={err:.2e} contrib={worst:.2e}")
    assert worst <= PT.RTOL_PHI


def test_amplitudes_static_video_single_mode(C, H):
    """Degenerate case: a constant video has one mode (lambda = 1, k_eff = 1) and
    b phi reproduces the frame exactly (up to fp32 Phi)."""
    rng = np.random.default_rng(2)
    n, m = 128 * 5 + 37, 20
    frame = rng.integers(0, 256, size=n, dtype=np.uint8)
    X = np.tile(frame, (m, 1))
    Xd = to_dev(X)
    P = C.Pipeline(H, n, n, m, "sparse", 30, 5, 3, s=5.0)
    P.sketch(Xd)
    P.fit()
    assert P.model.k_eff == 1
    F = P.modes(Xd)
    b, dropped = P.amplitudes(Xd)
    torch.cuda.synchronize()
    assert int(dropped.item()) == 0
    rec = (F.cpu().numpy().astype(np.float64)[0] * b.cpu().numpy()[0]).real
    assert np.max(np.abs(rec - frame)) <= 1e-4 * 255


GUARD = 4096
_CANARY = 0xA5


def _guarded(shape, dtype):
    """A tensor in the middle of a buffer with GUARD canary bytes on both sides."""
    nb = int(np.prod(shape)) * torch.tensor([], dtype=dtype).element_size()
    buf = torch.full((nb + 2 * GUARD,), _CANARY, dtype=torch.uint8, device="cuda")
    return buf, buf[GUARD:GUARD + nb].view(dtype).view(shape)


def _guards_intact(buf):
    return bool((buf[:GUARD] == _CANARY).all()) and bool((buf[-GUARD:] == _CANARY).all())


@pytest.mark.parametrize("case", ["c1", "ragged_sparse", "ragged_spixel", "rademacher", "gaussian"])
def test_no_out_of_bounds_writes(C, H, case):
    """compute-sanitizer is closed on this GPU pool, so out-of-bounds WRITES are caught
    with canaries instead: every caller buffer of every entry point (Y, sketch and fit
    workspaces, the model, Phi, L, the masks of all three foreground paths, the
    amplitudes Gram / b) sits between 4 KB guard regions of 0xA5 that must be intact
    after the whole path ran; small and ragged cases (n not a multiple of 128, odd m)."""
    import importlib.util
    spec = importlib.util.spec_from_file_location(
        "sanitize_cases", os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                       "tools", "sanitize_cases.py"))
    sc = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(sc)
    mk, kind, p, k, K = sc.CASES[case]
    X = mk()
    m, n = X.shape
    Xd = to_dev(X)
    P = C.Pipeline(H, n, n, m, kind, p, k, K)
    bufs = {}

    def swap(name, attr, shape, dtype):
        b, t = _guarded(shape, dtype)
        bufs[name] = b
        setattr(P, attr, t)

    swap("Y", "Y", tuple(P.Y.shape), P.Y.dtype)
    swap("ws_sketch", "ws_sketch", tuple(P.ws_sketch.shape), torch.uint8)
    swap("ws_fit", "ws_fit", tuple(P.ws_fit.shape), torch.uint8)
    swap("model", "model_buf", (P.model_buf.numel(),), torch.uint8)
    # the model must start 256-B aligned: the guard (4096) keeps the alignment
    P.model = C.cdmd_model_bind(P.model_buf, k, K, m)
    swap("Phi", "Phi", tuple(P.Phi.shape), torch.float32)
    swap("mask", "mask", tuple(P.mask.shape), torch.int32)
    P.run(Xd, 25.0, C.BG_DYNAMIC)
    P.foreground(Xd, 25.0, C.BG_STATIC)
    fused_mask(C, P, Xd, 25.0)
    bL, L = _guarded((m, n), torch.float32)
    C.cdmd_background(H, P.Phi, n, P.model, C.BG_DYNAMIC, 0, m, L)
    ke = P.model.k_eff
    bG, G = _guarded((ke + 1, ke), torch.float64)
    bw, ws = _guarded((C.cdmd_amplitudes_workspace_bytes(H, ke),), torch.uint8)
    bb, b = _guarded((ke, 2), torch.float64)
    C.cdmd_amplitudes_gram(H, C.video(Xd, n, 0, n), P.model, P.Phi, G, ws)
    C.cdmd_amplitudes_solve(H, P.model, G, b)
    torch.cuda.synchronize()
    bufs.update(L=bL, G=bG, amp_ws=bw, b=bb)
    bad = [name for name, buf in bufs.items() if not _guards_intact(buf)]
    assert not bad, f"guard regions overwritten: {bad}"


def test_repeatable_under_concurrency(C, H):
    """A race in the persistent kernels' tile schedule or stage hand-offs shows up as
    run-to-run differences: at the bench size, modes, the two-pass mask and the fused
    mask are bit-identical over 12 repetitions, half of them issued from three streams
    at once (different CTA start times and tile claims)."""
    cfg = config_by_name("c4_1080p_sparse")
    X = video_for(cfg)
    m, n = X.shape
    Xd = to_dev(X)
    pipes = [C.Pipeline(H, n, n, m, "sparse", cfg.p, cfg.k, cfg.K) for _ in range(3)]
    P0 = pipes[0]
    P0.run(Xd, cfg.tau, C.BG_DYNAMIC)
    ref = (P0.Phi.clone(), P0.mask.clone())
    ref_f = P0.foreground(Xd, cfg.tau, C.BG_DYNAMIC, fused=True).clone()
    for Pq in pipes[1:]:
        Pq.sketch(Xd)
        Pq.fit()
    streams = [torch.cuda.Stream() for _ in range(3)]
    torch.cuda.synchronize()
    for rep in range(6):
        for Pq, st in zip(pipes, streams):
            with torch.cuda.stream(st):
                Pq.modes(Xd, st)
                Pq.foreground(Xd, cfg.tau, C.BG_DYNAMIC, st)
        torch.cuda.synchronize()
        for Pq in pipes:
            assert torch.equal(Pq.Phi, ref[0]) and torch.equal(Pq.mask, ref[1]), rep
        for Pq, st in zip(pipes, streams):
            with torch.cuda.stream(st):
                Pq.foreground(Xd, cfg.tau, C.BG_DYNAMIC, st, fused=True)
        torch.cuda.synchronize()
        for Pq in pipes:
            assert torch.equal(Pq.mask, ref_f), rep


@pytest.mark.parametrize("partition", ["pixel", "batch"])
def test_bench_two_ranks_runs(partition, tmp_path):
    """bench.py under torchrun with two ranks sharing cuda:0 over gloo (the multi-rank
    code path of the pixel-row split -- slab sketches + batch-ordered all-reduce -- and
    of batch-parallel replicas -- no collective); one JSON line from rank 0."""
    import json
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    port = 29600 + (os.getpid() % 1000) + (7 if partition == "batch" else 0)
    env = dict(os.environ, CDMD_DIST_BACKEND="gloo")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.join(root, "bench.py"), "--gpus", "2",
           "--steps", "4", "--warmup", "3", "--lanes", "2", "--no-cpu-baseline", "--no-e2e", "--graph-reps", "10",
           "--partition", partition, "--config", "c2_320x240_spixel"]
    r = subprocess.run(cmd, cwd=root, capture_output=True, text=True, timeout=900, env=env)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-4000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["value"] > 0
    assert d["scaling"] == ("weak" if partition == "batch" else "strong")
    assert d["config"]["parallelism"].startswith("pixel-rows" if partition == "pixel" else "batch replicas")


@pytest.mark.parametrize("W,Hh,m,p,k,K,mode", [(64, 48, 40, 120, 10, 3, "dyn"), (320, 240, 200, 1000, 20, 10, "dyn"),
                                                (320, 240, 200, 1000, 20, 10, "sta"), (96, 33, 77, 200, 12, 4, "dyn"),
                                                # W % 128 == 0: the banded median phase (H not a multiple of 8)
                                                (256, 45, 60, 300, 12, 4, "dyn"), (384, 19, 33, 300, 12, 4, "sta"),
                                                (1920, 1080, 500, 2000, 50, 10, "dyn")])
def test_fused_median_bit_exact(C, H, W, Hh, m, p, k, K, mode):
    """The 3x3 median folded into the fused pass (Fig. 7): the filtered mask equals
    the oracle's median3 of the raw mask bit for bit (every frame, every pixel, the image
    borders zero-padded), and the raw mask equals the fused pass's own mask."""
    X = make_video(W, Hh, m, seed=W + Hh, noise=2.0, n_rects=2)
    n = W * Hh
    Xd = to_dev(X)
    P = C.Pipeline(H, n, n, m, "sparse", p, k, K)
    P.sketch(Xd)
    P.fit()
    md = C.BG_DYNAMIC if mode == "dyn" else C.BG_STATIC
    plain = P.foreground(Xd, 25.0, md, fused=True).clone()
    raw, out = P.foreground_median3(Xd, 25.0, W, Hh, md)
    torch.cuda.synchronize()
    assert torch.equal(raw, plain)
    rawb = OD.unpack_mask(raw.cpu().numpy().view(np.uint32), n)
    got = OD.unpack_mask(out.cpu().numpy().view(np.uint32), n)
    assert np.array_equal(got, OD.median3(rawb, W, Hh))


def test_fused_median_needs_word_aligned_rows(C, H):
    X = make_video(100, 37, 33, seed=5, noise=2.0, n_rects=1)   # width 100: rows not word-aligned
    n = X.shape[1]
    P = C.Pipeline(H, n, n, 33, "sparse", 120, 12, 5)
    Xd = to_dev(X)
    P.sketch(Xd)
    P.fit()
    with pytest.raises(C.CdmdError) as e:
        P.foreground_median3(Xd, 25.0, 100, 37)
    assert e.value.code == 6


@pytest.mark.parametrize("name", ["c2_320x240_spixel", "c4_1080p_sparse"])
def test_lanczos_eigensolver_matches_oracle_and_householder(C, H, name, monkeypatch):
    """Step 4's k largest Gram eigenpairs by Lanczos (lanczos.cu) pass the residual test
    on the paper-shaped sketches (no Householder fallback), agree with the oracle's
    eigendecomposition (sigma to 1e-6, lambda to RTOL_EIG), and give the same model as
    the Householder cluster solver (CDMD_SYEV=h) up to rounding."""
    cfg = config_by_name(name)
    X = video_for(cfg)
    m, n = X.shape
    Xd = to_dev(X)
    kind = {"sparse": OS.SPARSE, "spixel": OS.SPIXEL}[cfg.kind]
    Yo = OS.sketch(X, kind, cfg.p, cfg.sensing_seed)
    om = OD.fit(Yo, cfg.k, cfg.K)
    models = {}
    for solver in ("lz", "h"):
        if solver == "h":
            monkeypatch.setenv("CDMD_SYEV", "h")
        else:
            monkeypatch.delenv("CDMD_SYEV", raising=False)
        runs0, fb0 = C.cdmd_eigensolver_stats(H)
        P = C.Pipeline(H, n, n, m, cfg.kind, cfg.p, cfg.k, cfg.K, seed=cfg.sensing_seed)
        P.sketch(Xd)
        P.fit()
        torch.cuda.synchronize()
        runs1, fb1 = C.cdmd_eigensolver_stats(H)
        if solver == "lz":
            assert (runs1 - runs0, fb1 - fb0) == (1, 0), (runs1 - runs0, fb1 - fb0)
        else:
            assert runs1 == runs0
        models[solver] = C.model_to_host(P.model)
    for gm in models.values():
        assert gm["k_eff"] == om["k_eff"]
        perm, err = PT.match_eigs(gm["lam"], om["lam"])
        assert err <= PT.RTOL_EIG, err
        assert np.max(np.abs(gm["sigma"] - om["sigma"]) / om["sigma"]) <= 1e-6
        assert PT.supports_equal_mod_conj(gm["support"], gm["pair"], perm, om["support"], om["pair"])
    a, b = models["lz"], models["h"]
    assert np.max(np.abs(a["sigma"] - b["sigma"]) / b["sigma"]) <= 1e-10
    perm, err = PT.match_eigs(a["lam"], b["lam"])
    assert err <= 1e-8, err


def test_lanczos_falls_back_on_an_invariant_subspace(C, H):
    """A rank-one Gram (a constant video): the Krylov space closes after one step, the
    residual test refuses it, and the Householder solver gives k_eff = 1."""
    rng = np.random.default_rng(5)
    n, m = 4096 + 77, 40
    X = np.tile(rng.integers(0, 256, size=n, dtype=np.uint8), (m, 1))
    Xd = to_dev(X)
    runs0, fb0 = C.cdmd_eigensolver_stats(H)
    P = C.Pipeline(H, n, n, m, "sparse", 60, 10, 3, s=5.0)
    P.sketch(Xd)
    P.fit()
    torch.cuda.synchronize()
    runs1, fb1 = C.cdmd_eigensolver_stats(H)
    assert (runs1 - runs0, fb1 - fb0) == (1, 1)
    assert P.model.k_eff == 1


@pytest.mark.parametrize("p,m,k,decay,seed", [(200, 60, 10, 0.8, 0), (600, 200, 40, 0.93, 1), (1500, 513, 30, 0.9, 2),
                                              (1500, 514, 30, 0.9, 3), (2000, 800, 54, 0.95, 4),
                                              (900, 300, 40, 1.0, 5)])
def test_fit_eigensolver_sizes_match_oracle(C, H, p, m, k, decay, seed):
    """cdmd_fit on planted sketches across the eigensolvers' size limits (Lanczos SMALL up
    to m - 1 = 512, BIG beyond; a flat spectrum (decay 1) whose Ritz pairs may fail the
    residual test and fall back): sigma, lambda and k_eff equal the oracle's whichever
    path ran, and Lanczos was attempted where the sizes allow it."""
    rng = np.random.default_rng(100 + seed)
    r = min(p, m)
    U, _ = np.linalg.qr(rng.standard_normal((p, r)))
    V, _ = np.linalg.qr(rng.standard_normal((m, r)))
    s = 1e4 * decay ** np.arange(r) * (1.0 + 0.1 * rng.random(r))
    Yf = ((U * s) @ V.T + rng.standard_normal((p, m))).astype(np.float32)
    P = C.Pipeline(H, 1024, 1024, m, "gaussian", p, k, min(5, k))
    P.Y.copy_(torch.from_numpy(np.ascontiguousarray(Yf.T)).cuda())
    runs0, fb0 = C.cdmd_eigensolver_stats(H)
    P.fit()
    torch.cuda.synchronize()
    runs1, fb1 = C.cdmd_eigensolver_stats(H)
    assert runs1 - runs0 == 1, "Lanczos not attempted"
    gm = C.model_to_host(P.model)
    om = OD.fit(Yf.astype(np.float64), k, min(5, k))
    assert gm["k_eff"] == om["k_eff"]
    assert np.max(np.abs(gm["sigma"] - om["sigma"]) / om["sigma"]) <= 1e-6
    perm, err = PT.match_eigs(gm["lam"], om["lam"])
    assert err <= PT.RTOL_EIG, err
    print(f"p={p} m={m} k={k} decay={decay}: fallback {fb1 - fb0}")


@pytest.mark.parametrize("p,m,k", [(60, 9, 2), (300, 40, 38), (1200, 513, 60), (1200, 513, 61), (3000, 1025, 60)])
def test_fit_eigensolver_edges(C, H, p, m, k):
    """Edge sizes of the eigensolver dispatch: the smallest Lanczos system (m - 1 = 8), a
    Krylov space as large as the matrix (J = m - 1), the k cap of the SMALL variant
    (2.25 k + 9 <= 144: k = 60 Lanczos, k = 61 Householder), and m - 1 = 1024 (BIG's
    limit).  sigma, lambda, k_eff equal the oracle's whichever solver ran."""
    rng = np.random.default_rng(7 + m + k)
    r = min(p, m)
    U, _ = np.linalg.qr(rng.standard_normal((p, r)))
    V, _ = np.linalg.qr(rng.standard_normal((m, r)))
    s = 1e4 * 0.9 ** np.arange(r) * (1.0 + 0.1 * rng.random(r))
    Yf = ((U * s) @ V.T + 0.1 * rng.standard_normal((p, m))).astype(np.float32)
    P = C.Pipeline(H, 1024, 1024, m, "gaussian", p, k, min(3, k))
    P.Y.copy_(torch.from_numpy(np.ascontiguousarray(Yf.T)).cuda())
    runs0, _ = C.cdmd_eigensolver_stats(H)
    P.fit()
    torch.cuda.synchronize()
    runs1, _ = C.cdmd_eigensolver_stats(H)
    expect_lz = (m - 1 >= 8) and (m - 1 <= 1024) and (k + 1 <= m - 1) and \
        (min(9 * k // 4 + 9, m - 1) <= (144 if m - 1 <= 512 else 288))
    assert (runs1 - runs0 == 1) == expect_lz, (runs1 - runs0, expect_lz)
    gm = C.model_to_host(P.model)
    om = OD.fit(Yf.astype(np.float64), k, min(3, k))
    assert gm["k_eff"] == om["k_eff"]
    assert np.max(np.abs(gm["sigma"] - om["sigma"]) / om["sigma"]) <= 1e-6
    perm, err = PT.match_eigs(gm["lam"], om["lam"])
    assert err <= PT.RTOL_EIG, err


def test_whole_step_cuda_graph(C, H):
    """The step sketch -> fit -> modes -> foreground captured in ONE CUDA graph (cdmd_fit
    without host read-backs under stream capture) replays bit-identically to the eager
    step, and its self-check flag stays clear; a Gavish-Donoho fit refuses capture."""
    cfg = config_by_name("c2_320x240_spixel")
    X = video_for(cfg)
    m, n = X.shape
    Xd = to_dev(X)
    P = C.Pipeline(H, n, n, m, cfg.kind, cfg.p, cfg.k, cfg.K, seed=cfg.sensing_seed)
    mask_e = P.run(Xd, cfg.tau, C.BG_DYNAMIC).clone()
    phi_e = P.Phi.clone()
    torch.cuda.synchronize()
    s = torch.cuda.Stream()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s):
        P.run(Xd, cfg.tau, C.BG_DYNAMIC)   # warm the capture stream's handles
        torch.cuda.synchronize()
        with torch.cuda.graph(g, stream=s):
            P.sketch(Xd)
            P.fit()
            P.modes(Xd)
            P.foreground(Xd, cfg.tau, C.BG_DYNAMIC)
    P.mask.zero_()
    P.Phi.zero_()
    for _ in range(3):
        g.replay()
    torch.cuda.synchronize()
    assert not P.graph_stale()
    assert torch.equal(P.mask, mask_e)
    assert torch.equal(P.Phi, phi_e)
    Pg = C.Pipeline(H, n, n, m, cfg.kind, cfg.p, cfg.k, cfg.K, seed=cfg.sensing_seed, rank="gd")
    Pg.run(Xd, cfg.tau, C.BG_DYNAMIC)
    torch.cuda.synchronize()
    g2 = torch.cuda.CUDAGraph()
    with pytest.raises(C.CdmdError):
        with torch.cuda.graph(g2, stream=s):
            Pg.fit()
