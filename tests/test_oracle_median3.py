"""Pins for the 3x3 median post-filter of the foreground mask (Fig. 7)."""

import numpy as np
import pytest
from scipy import ndimage

from oracle import cdmd as OD


def test_isolated_pixel_removed_block_kept():
    W, H = 9, 7
    M = np.zeros((2, W * H), dtype=bool)
    M[0, 3 * W + 4] = True                          # isolated positive -> removed
    for y in range(2, 5):
        for x in range(3, 6):
            M[1, y * W + x] = True                  # 3x3 block -> centre and edge midpoints kept
    R = OD.median3(M, W, H)
    assert not R[0].any()
    kept = {(y, x) for y in range(H) for x in range(W) if R[1, y * W + x]}
    assert kept == {(3, 4), (2, 4), (4, 4), (3, 3), (3, 5)}   # 6 of 9 / 5 of 9 neighbours; corners see 4


def test_equals_scipy_median_filter_zero_padded():
    """The majority rule equals the textbook 3x3 median with constant-0 padding."""
    rng = np.random.default_rng(0)
    for W, H, dens in [(37, 23, 0.3), (64, 16, 0.5), (5, 3, 0.7), (1, 9, 0.6)]:
        M = rng.random((3, W * H)) < dens
        ref = np.stack([ndimage.median_filter(f.reshape(H, W).astype(np.uint8), size=3, mode="constant", cval=0)
                        for f in M]).reshape(3, W * H).astype(bool)
        assert np.array_equal(OD.median3(M, W, H), ref)


def test_idempotent_on_solid_and_empty_frames():
    W, H = 10, 10
    full = np.ones((1, W * H), dtype=bool)
    R = OD.median3(full, W, H)
    # with zero padding only the 4 corners (4 of 9 set) drop
    corners = {0, W - 1, (H - 1) * W, H * W - 1}
    assert set(np.flatnonzero(~R[0])) == corners
    assert not OD.median3(np.zeros((1, W * H), dtype=bool), W, H).any()


def test_rejects_partial_frames():
    with pytest.raises(ValueError):
        OD.median3(np.zeros((1, 10), dtype=bool), 3, 3)
