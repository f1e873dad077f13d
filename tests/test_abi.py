"""The C-ABI library loads on a CPU-only box and exports every symbol that
include/cdmd.h declares; host-only entry points validate their arguments.
No compute calls (there is no GPU here)."""

import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HDR = os.path.join(ROOT, "include", "cdmd.h")


@pytest.fixture(scope="module")
def libpath():
    from paper_1512_04205_b200.build import build
    return build(verbose=False)


def declared():
    src = open(HDR).read()
    return sorted(set(re.findall(r"CDMD_API[^;]*?\b(cdmd_\w+)\s*\(", src)))


def test_header_declares_the_boundary():
    names = declared()
    for n in ["cdmd_sketch", "cdmd_fit", "cdmd_modes", "cdmd_background", "cdmd_foreground"]:
        assert n in names


def test_library_exports_every_declared_symbol(libpath):
    out = subprocess.run(["nm", "-D", "--defined-only", libpath], capture_output=True, text=True, check=True).stdout
    exported = set(re.findall(r" T (cdmd_\w+)", out))
    assert set(declared()) <= exported
    # and nothing else leaks out of the library
    assert exported <= set(declared())


def test_binding_loads_and_matches_header(libpath):
    from paper_1512_04205_b200 import cdmd
    lib = cdmd.lib()
    for n in declared():
        assert hasattr(lib, n)
    assert set(cdmd.SYMBOLS) == set(declared())
    assert b"sm_100a" in lib.cdmd_version()
    assert lib.cdmd_status_str(5) == b"workspace too small"


def test_sm100a_cubin_only(libpath):
    out = subprocess.run(["cuobjdump", "--list-elf", libpath], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    assert "sm_90" not in out and "sm_80" not in out


def test_host_side_validation_and_sizes(libpath):
    from paper_1512_04205_b200 import cdmd
    lib = cdmd.lib()
    # model buffer size and binding layout (host only)
    nb = lib.cdmd_model_bytes(50, 10, 500)
    assert nb > 0
    M = cdmd.Model()
    buf = ctypes.create_string_buffer(nb + 512)
    base = (ctypes.addressof(buf) + 255) & ~255
    assert lib.cdmd_model_bind(ctypes.byref(M), ctypes.c_void_p(base), nb, 50, 10, 500) == 0
    assert M.k == 50 and M.K == 10 and M.kpad == 64 and M.mpad == 512 and M.limbs == 4
    ptrs = [M.lambda_, M.omega, M.pair, M.sigma, M.Mfold, M.beta, M.support, M.Mq, M.Mq_scale,
            M.coef, M.coef_col, M.dev_info]
    assert all(base <= p < base + nb and p % 256 == 0 for p in ptrs)
    assert ptrs == sorted(ptrs)
    # range errors (SPEC/paper preconditions) are reported before any launch
    assert lib.cdmd_model_bind(ctypes.byref(M), ctypes.c_void_p(base), nb, 50, 51, 500) == 2  # K > k
    assert lib.cdmd_model_bind(ctypes.byref(M), ctypes.c_void_p(base), 16, 50, 10, 500) == 5  # too small
    assert lib.cdmd_model_bind(ctypes.byref(M), ctypes.c_void_p(base + 8), nb, 50, 10, 500) == 1  # misaligned
    # sparse ELL capacity: mean n/s = ln n non-zeros per row plus a wide margin
    cap = lib.cdmd_sparse_cap(2073600, 2000, 0.0)
    assert 60 < cap < 100
    # workspace query for a sparse sketch of 1080p
    v = cdmd.Video(0, 2073600, 0, 2073600, 500, 2073600)
    c = cdmd.sensing("sparse", 2000)
    assert lib.cdmd_sketch_workspace_bytes(ctypes.byref(v), ctypes.byref(c)) >= 2000 * cap * 4
    bad = cdmd.sensing("sparse", 3000000)
    assert lib.cdmd_sketch_workspace_bytes(ctypes.byref(v), ctypes.byref(bad)) == 0   # p > n
    # null handle -> invalid argument, no launch
    assert lib.cdmd_sketch(None, ctypes.byref(v), ctypes.byref(c), None, 2000, None, 0, None) == 1
    # amplitudes (Alg. 1 step 9): host-side validation only, nothing launched
    assert lib.cdmd_amplitudes_workspace_bytes(None, 50) == 0
    assert lib.cdmd_amplitudes_gram(None, ctypes.byref(v), ctypes.byref(M), None, 2073600, None, None, 0,
                                    None) == 1
    assert lib.cdmd_amplitudes_solve(None, ctypes.byref(M), None, None, None, None) == 1


def test_struct_layouts_match_c():
    from paper_1512_04205_b200 import cdmd
    assert ctypes.sizeof(cdmd.Video) == 48
    assert ctypes.sizeof(cdmd.Sensing) == 32
    assert cdmd.Model.k_eff.offset == 4 * 4 + 2 * 8 + 12 * 8
    assert ctypes.sizeof(cdmd.Model) == cdmd.Model.dt.offset + 8
