"""Pins the oracle's Philox4x32-10 to the Random123 known-answer vectors
(tests/golden/philox_kat.txt) — the generator DESIGN.md §3.1 fixes for C."""

import os

import numpy as np

from oracle.philox import philox4x32_10, seed_key

GOLD = os.path.join(os.path.dirname(__file__), "golden", "philox_kat.txt")


def _kat():
    out = []
    for line in open(GOLD):
        line = line.split("#")[0].strip()
        if not line:
            continue
        v = [int(x, 16) for x in line.split()]
        out.append((v[:4], v[4:6], v[6:10]))
    return out


def test_known_answer_vectors():
    kat = _kat()
    assert len(kat) == 3
    for ctr, key, want in kat:
        got = [int(x) for x in philox4x32_10(*ctr, *key)]
        assert got == want


def test_vectorised_matches_scalar_calls():
    c0 = np.arange(17, dtype=np.uint64) * np.uint64(0x9E3779B1)
    vec = philox4x32_10(c0, 5, 7, 3, 11, 13)
    for i in range(17):
        sc = philox4x32_10(int(c0[i]) & 0xFFFFFFFF, 5, 7, 3, 11, 13)
        assert [int(v[i]) for v in vec] == [int(s) for s in sc]


def test_seed_key_split():
    assert seed_key(0) == (0, 0)
    assert seed_key(0x0123456789ABCDEF) == (0x89ABCDEF, 0x01234567)
