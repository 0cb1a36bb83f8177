"""Pins for the oracle's integer 2x box downsample (reading Q11)."""
import json
import os

import numpy as np
import pytest

import oracle

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "frame_A.json")))


def test_golden():
    A = np.array(GOLD["A"], dtype=np.uint8)
    np.testing.assert_array_equal(oracle.downsample(A), np.array(GOLD["downsample_A"], dtype=np.uint8))
    f3 = np.array(GOLD["frame_3x3"]["pixels"], dtype=np.uint8)
    np.testing.assert_array_equal(oracle.downsample(f3), np.array(GOLD["frame_3x3"]["downsample"], dtype=np.uint8))


@pytest.mark.parametrize("w,h", [(2, 2), (7, 5), (64, 36), (1, 9), (9, 1)])
def test_constant_closed_form(w, h):
    for v in (0, 1, 128, 255):
        f = np.full((h, w, 3), v, dtype=np.uint8)
        out = oracle.downsample(f)
        assert out.shape == (h // 2, w // 2, 3)
        assert (out == v).all()


@pytest.mark.parametrize("w,h", [(1920, 4), (513, 3), (6, 2)])
def test_xgradient_pins_rounding(w, h):
    # v = x mod 256: block sum = 8x'+2 (mod-256 period is even) -> round-half-up gives 2x'+1, truncation 2x'
    f = np.empty((h, w, 3), dtype=np.uint8)
    f[:] = (np.arange(w) % 256).astype(np.uint8)[None, :, None]
    out = oracle.downsample(f)
    expect = ((2 * np.arange(w // 2) + 1) % 256).astype(np.uint8)
    for c in range(3):
        np.testing.assert_array_equal(out[:, :, c], np.broadcast_to(expect, (h // 2, w // 2)))


def test_float_mean_formulation():
    # second formulation: floor(mean of the 2x2 block + 1/2) in float64 on random odd-sized frames
    rng = np.random.default_rng(11)
    for _ in range(30):
        h, w = rng.integers(1, 30, size=2)
        f = rng.integers(0, 256, size=(h, w, 3), dtype=np.uint8)
        blocks = f[: h // 2 * 2, : w // 2 * 2].astype(np.float64).reshape(h // 2, 2, w // 2, 2, 3)
        ref = np.floor(blocks.mean(axis=(1, 3)) + 0.5).astype(np.uint8)
        np.testing.assert_array_equal(oracle.downsample(f), ref)
