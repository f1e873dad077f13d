"""Thin Python binding of libcdmd (include/cdmd.h) — argument marshalling only.

Every step of the hot path runs in libcdmd's CUDA kernels (and cuSOLVER for the
small eigen-solves of cdmd_fit).  PyTorch provides device memory and streams.
There is no CPU fallback: importing this module on a machine without the built
library raises, and every call checks the returned status.

Names follow the C ABI: cdmd_sketch, cdmd_fit, cdmd_modes, cdmd_background,
cdmd_foreground (+ test hooks).  ``Pipeline`` strings them together with
caller-owned torch buffers (the same calls bench.py times).
"""

import ctypes
import math
import os

import torch

from .build import LIB

SPIXEL, SPARSE, RADEMACHER, GAUSSIAN, SRFT = 0, 1, 2, 3, 4
KINDS = {"spixel": SPIXEL, "sparse": SPARSE, "rademacher": RADEMACHER, "gaussian": GAUSSIAN, "srft": SRFT}
BG_STATIC, BG_DYNAMIC = 0, 1
STATUS = {0: "ok", 1: "invalid argument", 2: "argument out of range", 3: "numerical failure",
          4: "CUDA error", 5: "workspace too small", 6: "unsupported device (needs sm_100a)"}


class CdmdError(RuntimeError):
    def __init__(self, where, code):
        super().__init__(f"{where}: {STATUS.get(code, code)} (status {code})")
        self.code = code


class Video(ctypes.Structure):
    _fields_ = [("X", ctypes.c_void_p), ("n_total", ctypes.c_int64), ("pix0", ctypes.c_int64),
                ("n_local", ctypes.c_int64), ("m", ctypes.c_int64), ("ld", ctypes.c_int64)]


class Sensing(ctypes.Structure):
    _fields_ = [("kind", ctypes.c_int32), ("p", ctypes.c_int64), ("s", ctypes.c_double),
                ("seed", ctypes.c_uint64)]


_P = ctypes.c_void_p


class Model(ctypes.Structure):
    _fields_ = [("k", ctypes.c_int32), ("K", ctypes.c_int32), ("limbs", ctypes.c_int32),
                ("kpad", ctypes.c_int32), ("m", ctypes.c_int64), ("mpad", ctypes.c_int64),
                ("lambda_", _P), ("omega", _P), ("pair", _P), ("sigma", _P), ("Mfold", _P),
                ("beta", _P), ("support", _P), ("Mq", _P), ("Mq_scale", _P), ("coef", _P),
                ("coef_col", _P), ("dev_info", _P),
                ("k_eff", ctypes.c_int32), ("K_eff", ctypes.c_int32), ("n_coef", ctypes.c_int32),
                ("info", ctypes.c_int32), ("dt", ctypes.c_double)]


SYMBOLS = ["cdmd_create", "cdmd_destroy", "cdmd_status_str", "cdmd_version", "cdmd_kernel_launches",
           "cdmd_eigensolver_stats",
           "cdmd_sketch_workspace_bytes", "cdmd_sketch", "cdmd_model_bytes", "cdmd_model_bind",
           "cdmd_fit_workspace_bytes", "cdmd_fit", "cdmd_modes", "cdmd_background",
           "cdmd_amplitudes_workspace_bytes", "cdmd_amplitudes_gram", "cdmd_amplitudes_solve",
           "cdmd_foreground", "cdmd_philox", "cdmd_gaussian_table", "cdmd_srft_table", "cdmd_sparse_cap",
           "cdmd_sensing_rows", "cdmd_modes_simt", "cdmd_eig", "cdmd_mask_median3",
           "cdmd_modes_path", "cdmd_foreground_path", "cdmd_sm_partition",
           "cdmd_set_background_selection", "cdmd_foreground_median3", "cdmd_foreground_median3_ws_bytes"]


def _load():
    if not os.path.exists(LIB):
        raise ImportError(f"libcdmd.so not built ({LIB}); run python -m paper_1512_04205_b200.build")
    lib = ctypes.CDLL(LIB)
    V, S, M = ctypes.POINTER(Video), ctypes.POINTER(Sensing), ctypes.POINTER(Model)
    i32, i64, sz, dbl, vp = ctypes.c_int32, ctypes.c_int64, ctypes.c_size_t, ctypes.c_double, ctypes.c_void_p
    sig = {
        "cdmd_create": (i32, [ctypes.c_int, ctypes.POINTER(vp)]),
        "cdmd_destroy": (None, [vp]),
        "cdmd_status_str": (ctypes.c_char_p, [i32]),
        "cdmd_version": (ctypes.c_char_p, []),
        "cdmd_kernel_launches": (ctypes.c_uint64, []),
        "cdmd_eigensolver_stats": (ctypes.c_int, [ctypes.c_void_p, ctypes.POINTER(ctypes.c_uint64),
                                                  ctypes.POINTER(ctypes.c_uint64)]),
        "cdmd_sketch_workspace_bytes": (sz, [V, S]),
        "cdmd_sketch": (i32, [vp, V, S, vp, i64, vp, sz, vp]),
        "cdmd_model_bytes": (sz, [ctypes.c_int, ctypes.c_int, i64]),
        "cdmd_model_bind": (i32, [M, vp, sz, ctypes.c_int, ctypes.c_int, i64]),
        "cdmd_fit_workspace_bytes": (sz, [vp, i64, i64, ctypes.c_int]),
        "cdmd_fit": (i32, [vp, vp, i64, i32, i64, i64, ctypes.c_int, ctypes.c_int, dbl, M, vp, sz, vp]),
        "cdmd_modes": (i32, [vp, V, M, vp, i64, vp]),
        "cdmd_modes_simt": (i32, [vp, V, M, vp, i64, vp]),
        "cdmd_background": (i32, [vp, vp, i64, i64, M, i32, i64, i64, vp, i64, vp]),
        "cdmd_foreground": (i32, [vp, V, M, vp, i64, i32, ctypes.c_float, vp, i64, vp]),
        "cdmd_mask_median3": (i32, [vp, i64, i64, i64, i64, vp, vp]),
        "cdmd_foreground_median3_ws_bytes": (sz, [i64, i64]),
        "cdmd_foreground_median3": (i32, [vp, V, M, i32, ctypes.c_float, i64, i64, vp, vp, i64, vp, sz, vp]),
        "cdmd_set_background_selection": (i32, [vp, dbl]),
        "cdmd_sm_partition": (i32, [ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.POINTER(vp),
                                    ctypes.POINTER(vp), ctypes.POINTER(ctypes.c_int)]),
        "cdmd_modes_path": (i32, [M]),
        "cdmd_foreground_path": (i32, [V, M, i32]),
        "cdmd_philox": (i32, [vp, ctypes.c_uint32, ctypes.c_uint32, vp, i64, vp]),
        "cdmd_gaussian_table": (i32, [vp, vp, vp]),
        "cdmd_srft_table": (i32, [vp, vp, vp]),
        "cdmd_sparse_cap": (i64, [i64, i64, dbl]),
        "cdmd_sensing_rows": (i32, [vp, i64, S, vp, vp, vp]),
        "cdmd_eig": (i32, [vp, ctypes.c_int, vp, vp, vp, vp]),
        "cdmd_amplitudes_workspace_bytes": (sz, [vp, ctypes.c_int]),
        "cdmd_amplitudes_gram": (i32, [vp, V, M, vp, i64, vp, vp, sz, vp]),
        "cdmd_amplitudes_solve": (i32, [vp, M, vp, vp, vp, vp]),
    }
    for name, (res, args) in sig.items():
        f = getattr(lib, name)
        f.restype = res
        f.argtypes = args
    return lib


_lib = _load()


def lib():
    return _lib


def _check(where, code):
    if code != 0:
        raise CdmdError(where, code)


def _stream(stream=None):
    s = stream if stream is not None else torch.cuda.current_stream()
    return ctypes.c_void_p(s.cuda_stream)


def _ptr(t):
    return ctypes.c_void_p(t.data_ptr()) if t is not None else ctypes.c_void_p(0)


class Handle:
    """cdmd_create / cdmd_destroy."""

    def __init__(self, device=0):
        h = ctypes.c_void_p()
        _check("cdmd_create", _lib.cdmd_create(int(device), ctypes.byref(h)))
        self.h = h
        self.device = device

    def __del__(self):
        if getattr(self, "h", None) is not None and _lib is not None:
            _lib.cdmd_destroy(self.h)
            self.h = None


def video(X, n_total=None, pix0=0, n_local=None):
    """cdmd_video over a uint8 CUDA tensor X of shape (m, ld) (frame-major)."""
    assert X.dtype == torch.uint8 and X.is_cuda and X.dim() == 2 and X.stride(1) == 1
    m = X.shape[0]
    n_local = X.shape[1] if n_local is None else n_local
    n_total = n_local if n_total is None else n_total
    return Video(X.data_ptr(), n_total, pix0, n_local, m, X.stride(0))


def sensing(kind, p, s=0.0, seed=0):
    return Sensing(KINDS[kind] if isinstance(kind, str) else int(kind), int(p), float(s or 0.0), int(seed))


def _empty_bytes(n, device):
    return torch.empty(max(int(n), 256), dtype=torch.uint8, device=device)


# ------------------------------------------------------------------ entry points
def cdmd_sketch_workspace_bytes(v, c):
    return _lib.cdmd_sketch_workspace_bytes(ctypes.byref(v), ctypes.byref(c))


def cdmd_sketch(h, v, c, Y, ws, stream=None):
    """Y: (m, ldy) CUDA tensor viewed column-major p x m (Y[t, r] = Y_full[r, t])."""
    _check("cdmd_sketch", _lib.cdmd_sketch(h.h, ctypes.byref(v), ctypes.byref(c), _ptr(Y), Y.stride(0),
                                           _ptr(ws), ws.numel() * ws.element_size(), _stream(stream)))


def cdmd_model_bytes(k, K, m):
    return _lib.cdmd_model_bytes(k, K, m)


def cdmd_model_bind(buf, k, K, m):
    M = Model()
    _check("cdmd_model_bind", _lib.cdmd_model_bind(ctypes.byref(M), _ptr(buf), buf.numel(), k, K, m))
    M._buf = buf
    return M


def cdmd_fit_workspace_bytes(h, p, m, k):
    return _lib.cdmd_fit_workspace_bytes(h.h, p, m, k)


def cdmd_fit(h, Y, kind, p, m, k, K, model, ws, dt=1.0, stream=None):
    kind = KINDS[kind] if isinstance(kind, str) else int(kind)
    _check("cdmd_fit", _lib.cdmd_fit(h.h, _ptr(Y), Y.stride(0), kind, p, m, k, K, dt, ctypes.byref(model),
                                     _ptr(ws), ws.numel(), _stream(stream)))


def cdmd_modes(h, v, model, Phi, stream=None, simt=False):
    """Phi: (k_cols, ldphi) float32 CUDA tensor (column c of the folded modes is Phi[c])."""
    f = _lib.cdmd_modes_simt if simt else _lib.cdmd_modes
    _check("cdmd_modes", f(h.h, ctypes.byref(v), ctypes.byref(model), _ptr(Phi), Phi.stride(0), _stream(stream)))


def cdmd_background(h, Phi, n_local, model, mode, t0, nt, L, stream=None):
    _check("cdmd_background", _lib.cdmd_background(h.h, _ptr(Phi), Phi.stride(0), n_local, ctypes.byref(model),
                                                   mode, t0, nt, _ptr(L), L.stride(0), _stream(stream)))


def cdmd_foreground(h, v, model, Phi, mode, tau, mask, stream=None):
    """mask: (m, ldw) int32/uint32-sized CUDA tensor of packed words.  Phi=None: the
    fused single pass (N11) -- the support's modes are computed in-slab from X."""
    _check("cdmd_foreground", _lib.cdmd_foreground(h.h, ctypes.byref(v), ctypes.byref(model), _ptr(Phi),
                                                   Phi.stride(0) if Phi is not None else 0, mode, float(tau),
                                                   _ptr(mask), mask.stride(0), _stream(stream)))


def cdmd_foreground_median3(h, v, model, mode, tau, width, height, raw, out, ws, stream=None):
    """Fused pass (N11) with the 3x3 median post-filter folded in: raw and filtered
    (m, ldw) masks of whole frames (width % 32 == 0); ws: >= cdmd_foreground_median3_ws_bytes."""
    _check("cdmd_foreground_median3", _lib.cdmd_foreground_median3(
        h.h, ctypes.byref(v), ctypes.byref(model), int(mode), float(tau), int(width), int(height), _ptr(raw),
        _ptr(out), raw.stride(0), _ptr(ws), ws.numel() * ws.element_size(), _stream(stream)))


def cdmd_amplitudes_workspace_bytes(h, k):
    return int(_lib.cdmd_amplitudes_workspace_bytes(h.h, int(k)))


def cdmd_amplitudes_gram(h, v, model, Phi, G, ws, stream=None):
    """G: (k_eff + 1, k_eff) float64 CUDA tensor (column-major k_eff x (k_eff + 1))."""
    _check("cdmd_amplitudes_gram", _lib.cdmd_amplitudes_gram(h.h, ctypes.byref(v), ctypes.byref(model), _ptr(Phi),
                                                             Phi.stride(0), _ptr(G), _ptr(ws), ws.numel(),
                                                             _stream(stream)))


def cdmd_amplitudes_solve(h, model, G, b, dropped=None, stream=None):
    """b: (k_eff, 2) float64 CUDA tensor (re, im); dropped: optional int32 CUDA scalar."""
    _check("cdmd_amplitudes_solve", _lib.cdmd_amplitudes_solve(h.h, ctypes.byref(model), _ptr(G), _ptr(b),
                                                               _ptr(dropped), _stream(stream)))


def cdmd_modes_path(model):
    """1: tcgen05 modes kernel, 0: CUDA-core fallback."""
    return int(_lib.cdmd_modes_path(ctypes.byref(model)))


def cdmd_foreground_path(v, model, mode):
    """2: tcgen05 dynamic, 1: CUDA-core dynamic, 0: static."""
    return int(_lib.cdmd_foreground_path(ctypes.byref(v), ctypes.byref(model), int(mode)))


def cdmd_mask_median3(mask, width, height, out, stream=None):
    """3x3 median post-filter (Fig. 7) of a (m, ldw) packed mask of whole frames."""
    _check("cdmd_mask_median3", _lib.cdmd_mask_median3(_ptr(mask), mask.stride(0), int(width), int(height),
                                                       mask.shape[0], _ptr(out), _stream(stream)))


def cdmd_philox(ctr, k0, k1, out, stream=None):
    _check("cdmd_philox", _lib.cdmd_philox(_ptr(ctr), k0, k1, _ptr(out), ctr.numel() // 4, _stream(stream)))


def cdmd_gaussian_table(h, out, stream=None):
    _check("cdmd_gaussian_table", _lib.cdmd_gaussian_table(h.h, _ptr(out), _stream(stream)))


def cdmd_srft_table(h, out, stream=None):
    _check("cdmd_srft_table", _lib.cdmd_srft_table(h.h, _ptr(out), _stream(stream)))


def cdmd_kernel_launches():
    """libcdmd kernel launches issued by this process so far (cuBLAS/cuSOLVER excluded)."""
    return int(lib().cdmd_kernel_launches())


def cdmd_eigensolver_stats(h):
    """(runs, fallbacks): fits on handle h whose eigenpairs came from Lanczos, and how many
    of them failed the residual test and were recomputed by the Householder solver."""
    runs, fb = ctypes.c_uint64(0), ctypes.c_uint64(0)
    _check("cdmd_eigensolver_stats", _lib.cdmd_eigensolver_stats(h.h, ctypes.byref(runs), ctypes.byref(fb)))
    return int(runs.value), int(fb.value)


_PARTITION = {}


def cdmd_sm_partition(device, fit_sms, n_streams):
    """Split the device's SMs (green contexts) into a solve partition of >= fit_sms SMs
    and a pass partition (the rest), once per process.  Returns (pass_streams,
    fit_streams, (solve_sms, pass_sms)) with the streams as torch ExternalStreams."""
    if device in _PARTITION:
        ps, fs, sms = _PARTITION[device]
        if len(ps) < n_streams:
            raise RuntimeError(f"SM partition on device {device} has {len(ps)} streams, {n_streams} requested")
        return ps[:n_streams], fs[:n_streams], sms
    vp = ctypes.c_void_p
    ps, fs, sms = (vp * n_streams)(), (vp * n_streams)(), (ctypes.c_int * 2)()
    _check("cdmd_sm_partition", lib().cdmd_sm_partition(device, fit_sms, n_streams, ps, fs, sms))
    dev = torch.device("cuda", device)
    out = ([torch.cuda.ExternalStream(ps[i], device=dev) for i in range(n_streams)],
           [torch.cuda.ExternalStream(fs[i], device=dev) for i in range(n_streams)], (sms[0], sms[1]))
    _PARTITION[device] = out
    return out


def cdmd_sparse_cap(n_total, p, s=0.0):
    return _lib.cdmd_sparse_cap(n_total, p, float(s or 0.0))


def cdmd_sensing_rows(h, n_total, c, out, counts=None, stream=None):
    _check("cdmd_sensing_rows", _lib.cdmd_sensing_rows(h.h, n_total, ctypes.byref(c), _ptr(out), _ptr(counts),
                                                       _stream(stream)))


def cdmd_eig(A, W, VR, info, stream=None):
    """A: (k, k) float64 CUDA tensor holding A^T row-major == A column-major."""
    _check("cdmd_eig", _lib.cdmd_eig(_ptr(A), A.shape[0], _ptr(W), _ptr(VR), _ptr(info), _stream(stream)))


# --------------------------------------------------------------- model read-back
def model_to_host(M):
    """Copy the model's device arrays into CPU tensors (for tests / reports)."""
    buf = M._buf
    base = buf.data_ptr()

    def arr(ptr, count, dtype):
        es = torch.tensor([], dtype=dtype).element_size()
        off = ptr - base
        return buf[off:off + count * es].view(dtype).cpu()

    k, K, m, ke, Ke = M.k, M.K, M.m, M.k_eff, M.K_eff
    lam = arr(M.lambda_, 2 * k, torch.float64).view(k, 2)[:ke]
    om = arr(M.omega, 2 * k, torch.float64).view(k, 2)[:ke]
    beta = arr(M.beta, 2 * K, torch.float64).view(K, 2)[:Ke]
    return dict(
        k_eff=ke, K_eff=Ke, n_coef=M.n_coef, info=M.info,
        lam=torch.complex(lam[:, 0], lam[:, 1]).numpy(),
        omega=torch.complex(om[:, 0], om[:, 1]).numpy(),
        pair=arr(M.pair, k, torch.int32)[:ke].numpy(),
        sigma=arr(M.sigma, k, torch.float64)[:ke].numpy(),
        Mfold=arr(M.Mfold, (m - 1) * k, torch.float64)[:(m - 1) * ke].view(ke, m - 1).T.numpy(),
        support=arr(M.support, K, torch.int32)[:Ke].numpy().tolist(),
        beta=torch.complex(beta[:, 0], beta[:, 1]).numpy(),
        coef=arr(M.coef, 2 * K * m, torch.float32)[:M.n_coef * m].view(M.n_coef, m).numpy(),
        coef_col=arr(M.coef_col, 2 * K, torch.int32)[:M.n_coef].numpy(),
        dev_info=arr(M.dev_info, 8, torch.int32).numpy(),
    )


# ---------------------------------------------------------------------- pipeline
class Pipeline:
    """Caller-owned buffers for one (video shape, sensing, k, K) problem, and the
    five-call hot path sketch -> [all-reduce] -> fit -> modes -> foreground."""

    def __init__(self, handle, n_total, n_local, m, kind, p, k, K, s=0.0, seed=0, pix0=0,
                 device="cuda", dt=1.0, rank="fixed", omega_eps=0.0):
        """rank="fixed": target rank k; rank="gd": Gavish-Donoho rank, at most k (Remark 2).
        omega_eps > 0: background = modes with |omega| < omega_eps instead of OMP."""
        if rank not in ("fixed", "gd"):
            raise ValueError(rank)
        self.rank = rank
        self.omega_eps = float(omega_eps)
        self.h = handle
        self.kind = KINDS[kind] if isinstance(kind, str) else int(kind)
        self.n_total, self.n_local, self.m, self.p, self.k, self.K = n_total, n_local, m, p, k, K
        self.pix0, self.dt = pix0, dt
        self.c = sensing(self.kind, p, s, seed)
        ydt = torch.float32 if self.kind in (GAUSSIAN, SRFT) else torch.int32
        self.Y = torch.empty((m, p), dtype=ydt, device=device)          # column-major p x m
        probe = Video(0, n_total, pix0, n_local, m, ((n_local + 15) // 16) * 16)
        self.ws_sketch = _empty_bytes(cdmd_sketch_workspace_bytes(probe, self.c), device)
        self.ws_fit = _empty_bytes(cdmd_fit_workspace_bytes(handle, p, m, k), device)
        self.model_buf = _empty_bytes(cdmd_model_bytes(k, K, m), device)
        self.model = cdmd_model_bind(self.model_buf, k, K, m)
        self.Phi = torch.empty((k, n_local), dtype=torch.float32, device=device)
        self.ldw = (n_local + 31) // 32
        self.mask = torch.empty((m, self.ldw), dtype=torch.int32, device=device)

    def sketch(self, X, stream=None):
        v = video(X, self.n_total, self.pix0, self.n_local)
        cdmd_sketch(self.h, v, self.c, self.Y, self.ws_sketch, stream)
        return self.Y

    def graph_stale(self):
        """After a replay of a captured step: True when the run disagreed with the sizes the
        graph was captured with (k_eff, K_eff, n_coef, an eigensolver fallback or error) --
        refit eagerly and recapture.  One 32-byte device-to-host read."""
        base = self.model_buf.data_ptr()
        off = self.model.dev_info - base
        flags = int(self.model_buf[off + 12:off + 16].view(torch.int32).item())   # dev_info[INFO_FLAGS]
        return bool(flags & 16)

    def fit(self, stream=None):
        k = -self.k if self.rank == "gd" else self.k
        _check("cdmd_set_background_selection", _lib.cdmd_set_background_selection(self.h.h, self.omega_eps))
        cdmd_fit(self.h, self.Y, self.kind, self.p, self.m, k, self.K, self.model, self.ws_fit,
                 self.dt, stream)
        return self.model

    def modes(self, X, stream=None, simt=False):
        v = video(X, self.n_total, self.pix0, self.n_local)
        cdmd_modes(self.h, v, self.model, self.Phi, stream, simt=simt)
        return self.Phi[:self.model.k_eff]

    def foreground(self, X, tau, mode=BG_DYNAMIC, stream=None, fused=False):
        """fused=True: cdmd_foreground(Phi=NULL), the single pass N11 (no modes() call needed)."""
        v = video(X, self.n_total, self.pix0, self.n_local)
        cdmd_foreground(self.h, v, self.model, None if fused else self.Phi, mode, tau, self.mask, stream)
        return self.mask

    def foreground_median3(self, X, tau, width, height, mode=BG_DYNAMIC, stream=None):
        """The fused pass with the 3x3 median folded in (whole frames, width % 32 == 0).
        Returns (raw mask, filtered mask); self.mask holds the raw one."""
        if width * height != self.n_local or self.pix0 != 0:
            raise ValueError("the fused median needs whole frames in this pipeline's slab")
        v = video(X, self.n_total, self.pix0, self.n_local)
        if getattr(self, "_med_out", None) is None:
            self._med_out = torch.empty_like(self.mask)
            self._med_ws = _empty_bytes(_lib.cdmd_foreground_median3_ws_bytes(int(width), int(height)),
                                        self.mask.device)
        cdmd_foreground_median3(self.h, v, self.model, mode, tau, width, height, self.mask, self._med_out,
                                self._med_ws, stream)
        return self.mask, self._med_out

    def median3(self, width, height, stream=None):
        """3x3 median post-filter of the last mask (whole frames: n_local = width * height)."""
        if width * height != self.n_local:
            raise ValueError("median3 needs whole frames in this pipeline's slab")
        out = torch.empty_like(self.mask)
        cdmd_mask_median3(self.mask, width, height, out, stream)
        return out

    def amplitudes(self, X, allreduce=None, stream=None):
        """b = lstsq(Phi, x_1) (Alg. 1 step 9) from the modes of the last
        modes() call: slab Gram [F^T F | F^T x_1] -> [allreduce(G), summing over the
        pixel slabs] -> fp64 Cholesky solve.  Returns (b (k_eff,) complex128 CUDA
        tensor, dropped (int32 CUDA scalar: dependent columns given c_j = 0))."""
        v = video(X, self.n_total, self.pix0, self.n_local)
        ke = self.model.k_eff
        ws = _empty_bytes(cdmd_amplitudes_workspace_bytes(self.h, ke), self.Phi.device)
        G = torch.empty((ke + 1, ke), dtype=torch.float64, device=self.Phi.device)
        cdmd_amplitudes_gram(self.h, v, self.model, self.Phi, G, ws, stream)
        if allreduce is not None:
            allreduce(G)
        b = torch.empty((ke, 2), dtype=torch.float64, device=self.Phi.device)
        dropped = torch.zeros((), dtype=torch.int32, device=self.Phi.device)
        cdmd_amplitudes_solve(self.h, self.model, G, b, dropped, stream)
        return torch.view_as_complex(b), dropped

    def background(self, mode=BG_DYNAMIC, t0=0, nt=None, stream=None):
        nt = self.m - t0 if nt is None else nt
        L = torch.empty((nt, self.n_local), dtype=torch.float32, device=self.Phi.device)
        cdmd_background(self.h, self.Phi, self.n_local, self.model, mode, t0, nt, L, stream)
        return L

    def run(self, X, tau, mode=BG_DYNAMIC, allreduce=None, stream=None, fused=False):
        """sketch -> [allreduce] -> fit -> modes -> foreground (fused: no modes pass;
        the foreground computes the support's modes in-slab, N11)."""
        self.sketch(X, stream)
        if allreduce is not None:
            allreduce(self.Y)
        self.fit(stream)
        if not fused:
            self.modes(X, stream)
        return self.foreground(X, tau, mode, stream, fused=fused)


class Streaming:
    """Multi-batch streaming driver (a long video is decomposed in independent
    consecutive batches).  `lanes` independent (handle, CUDA stream, buffers, host
    thread) sets run batches round-robin, so the latency-bound small solve of one
    batch (cdmd_fit, which blocks its own host thread) overlaps the HBM-bound passes
    and solves of the others.  Each batch runs the same five calls as Pipeline.run.

    Across GPUs (torch.distributed initialised, world > 1) two partitions:
      * pixel-row slabs (run(..., allreduce=fn)): each rank sketches its slab, the
        per-batch all-reduces of Y are issued in batch order on every rank (one ticket
        sequence over one communicator, dist.OrderedAllreduce) and every rank repeats
        the fit (bit-identical Y -> identical model);
      * batch-parallel replicas (no allreduce): each rank runs its own whole-frame
        batches (dist.my_batches), no collective at all.
    A lane that raises aborts the ticket sequence (the other lanes stop waiting) and
    run() re-raises the first error.
    Each lane uses two streams: set CUDA_DEVICE_MAX_CONNECTIONS (up to 32) to at least
    2 x lanes before CUDA initialises, or streams share the default 8 hardware queues
    and a lane's waiting solve stalls other lanes' work (bench.py sets 32)."""

    def __init__(self, device, n_total, n_local, m, kind, p, k, K, lanes=4, s=0.0, seed=0, pix0=0, dt=1.0,
                 rank="fixed", fit_sms=0, fused=False):
        """fused: foreground through cdmd_foreground(Phi=NULL) (N11: modes of the
        support computed in-slab, no cdmd_modes pass) instead of modes + foreground."""
        from .dist import OrderedAllreduce
        self.lanes = []
        self.fused = fused
        self.ordered = OrderedAllreduce()
        self.sms = None
        if fit_sms > 0:
            # spatial partition (cdmd_sm_partition): the solves get SMs of their own
            # instead of queueing behind the persistent full-resolution passes
            pst, fst, self.sms = cdmd_sm_partition(device, fit_sms, lanes)
        lo, hi = torch.cuda.Stream.priority_range()
        for li in range(lanes):
            h = Handle(device)
            if fit_sms > 0:
                st, st_fit = pst[li], fst[li]
            else:
                st = torch.cuda.Stream(device=device)
                # the small solve runs on a high-priority stream of its own: its kernels
                # (the 8-CTA tridiagonalisation cluster above all) get SMs ahead of the
                # next lane's full-resolution pass instead of waiting behind it
                st_fit = torch.cuda.Stream(device=device, priority=hi)
            with torch.cuda.stream(st):
                pipe = Pipeline(h, n_total, n_local, m, kind, p, k, K, s=s, seed=seed, pix0=pix0,
                                device=f"cuda:{device}", dt=dt, rank=rank)
            self.lanes.append((h, st, st_fit, pipe))

    def run(self, videos, tau, mode=BG_DYNAMIC, allreduce=None, start_event=None, host_video=None,
            host_masks=None):
        """videos: list of uint8 CUDA tensors (m, ld), one per batch.  Returns the
        per-lane end events (record them into the caller's stream to join).
        allreduce(Y): the per-batch sum of the slab sketches (pixel-row sharding), issued
        in batch order; None for one GPU or batch-parallel replicas.
        End to end: with `host_video` (a pinned uint8 host tensor like videos[b]) every
        batch first copies it into its device buffer, and with `host_masks` (one pinned
        int32 host tensor per lane, shaped like the mask) every batch copies its mask
        back; the copies run on the lane's stream, overlapping the other lanes' work."""
        import concurrent.futures as cf
        self.ordered.reset()
        L = len(self.lanes)
        ends = [None] * L

        def lane_work(li):
            h, st, st_fit, pipe = self.lanes[li]
            try:
                with torch.cuda.stream(st):
                    if start_event is not None:
                        st.wait_event(start_event)
                    for b in range(li, len(videos), L):
                        X = videos[b]
                        if host_video is not None:
                            X.copy_(host_video, non_blocking=True)
                        pipe.sketch(X, st)
                        if allreduce is not None:
                            self.ordered.run(b, lambda: allreduce(pipe.Y))
                        st_fit.wait_stream(st)
                        pipe.fit(st_fit)
                        st.wait_stream(st_fit)
                        if self.fused:
                            pipe.foreground(X, tau, mode, st, fused=True)
                        else:
                            pipe.modes(X, st)
                            pipe.foreground(X, tau, mode, st)
                        if host_masks is not None:
                            host_masks[li].copy_(pipe.mask, non_blocking=True)
                    ev = torch.cuda.Event(enable_timing=True)
                    ev.record(st)
                    ends[li] = ev
            except BaseException as e:
                self.ordered.abort(e)
                raise

        errs = []
        with cf.ThreadPoolExecutor(L) as ex:
            futs = [ex.submit(lane_work, i) for i in range(L)]
            for f in futs:
                try:
                    f.result()
                except BaseException as e:
                    errs.append(e)
        if errs:
            from .dist import LaneAbort
            first = next((e for e in errs if not isinstance(e, LaneAbort)), errs[0])
            raise first
        return ends


from .dist import slab  # noqa: E402,F401  (re-export)
