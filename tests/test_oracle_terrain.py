"""Pins of the oracle's world generation (reading R27)
against closed forms, the definition restated in float32 numpy, and distributional checks."""
import math

import numpy as np
import pytest

import oracle

L, C, SEED = 6, 10, 1234


@pytest.fixture(scope="module")
def world():
    return oracle.terrain_generate(L, C, SEED)


def tile(hf, l, c):
    return hf[80 * l:80 * (l + 1), 80 * c:80 * (c + 1)]


def edge_dist64():
    x = (np.arange(80) + 0.5) * 0.1
    d1 = np.minimum(x, 8.0 - x)
    return np.minimum(d1[:, None], d1[None, :])


def word(seed, tile_id, w):
    out = oracle.philox(seed & 0xFFFFFFFF, seed >> 32, [w // 4, tile_id, 0, 8])
    return int(out[w % 4])


def u01(x):
    return np.float32(x >> 8) * np.float32(2.0 ** -24)


def test_shape_layout_and_flat_tiles(world):
    assert world.shape == (80 * L, 80 * C) and world.dtype == np.float32
    for l in range(L):
        for c in range(0, C, 5):  # kind 0 = flat
            assert np.all(tile(world, l, c) == 0.0)


def test_slope_pyramid_closed_form(world):
    e = edge_dist64()
    for l in range(L):
        d = l / (L - 1)
        want = math.tan(math.radians(25.0 * d)) * np.minimum(e, 3.0)
        got = tile(world, l, 1).astype(np.float64)
        assert np.max(np.abs(got - want)) <= 1e-6 * max(1.0, want.max())
        # plateau at the peak height, border ring at tan * 0.05
        assert np.allclose(got[40, 40], math.tan(math.radians(25.0 * d)) * 3.0, rtol=1e-6, atol=1e-7)
    assert np.all(tile(world, 0, 1) == 0.0)  # difficulty 0: flat


def test_stairs_are_integer_risers(world):
    e = edge_dist64()
    k = np.floor(np.minimum(e, 3.0) / 0.3)  # no cell centre sits on a tread edge (0.05 + 0.1 n != 0.3 m)
    for l in range(L):
        d = np.float32(l) / np.float32(L - 1)
        riser = np.float32(0.05) + np.float32(0.15) * d
        got = tile(world, l, 4)
        assert np.array_equal(got, (riser * k.astype(np.float32)).astype(np.float32))
    assert k.max() == 10 and k.min() == 0


def test_rough_uniform_in_range_and_counter_layout(world):
    for l in range(L):
        a = 0.05 * (1.0 + l / (L - 1))
        t = tile(world, l, 2).astype(np.float64)
        assert np.all(np.abs(t) <= a / 2 + 1e-7)
        assert abs(t.mean()) < 5 * (a / math.sqrt(12)) / 80          # 5 sigma of the mean of 6400 draws
        hist, _ = np.histogram(t, bins=10, range=(-a / 2, a / 2))
        chi2 = ((hist - 640.0) ** 2 / 640.0).sum()
        assert chi2 < 40.0                                          # 9 dof: p < 1e-5
    # the counter layout: cell (i, j) of tile (l, c) is word i*80 + j of stream (tile id, 0, tag 8)
    l, c = 3, 7
    half = np.float32(0.5) * (np.float32(0.05) * (np.float32(1.0) + np.float32(l) / np.float32(L - 1)))
    for (i, j) in [(0, 0), (0, 3), (17, 42), (79, 79)]:
        w = word(SEED, l * C + c, i * 80 + j)
        want = half * (np.float32(2.0) * u01(w) - np.float32(1.0))
        assert tile(world, l, c)[i, j] == want


def test_obstacles_restated_in_float32(world):
    e = edge_dist64()
    for l in range(L):
        for c in (3, 8):
            tid = l * C + c
            d = np.float32(l) / np.float32(L - 1)
            hmax = np.float32(0.05) + np.float32(0.15) * d
            want = np.zeros((80, 80), np.float32)
            for b in range(8):
                u = [u01(word(SEED, tid, 5 * b + k)) for k in range(5)]
                w = np.float32(0.5) + np.float32(1.5) * u[0]
                ln = np.float32(0.5) + np.float32(1.5) * u[1]
                x0 = np.float32(8.0) * u[2]
                y0 = np.float32(8.0) * u[3]
                hh = hmax * (np.float32(2.0) * u[4] - np.float32(1.0))
                i0, i1 = int(x0 * np.float32(10)), int(min(np.float32(8), x0 + w) * np.float32(10))
                j0, j1 = int(y0 * np.float32(10)), int(min(np.float32(8), y0 + ln) * np.float32(10))
                want[i0:i1, j0:j1] = hh
            want[e >= 3.0] = 0.0
            got = tile(world, l, c)
            assert np.array_equal(got, want), (l, c)
            assert np.all(np.abs(got) <= hmax)
            assert np.all(got[37:43, 37:43] == 0.0)  # spawn plateau


def test_seed_and_tile_independence():
    a = oracle.terrain_generate(2, 5, 1)
    b = oracle.terrain_generate(2, 5, 2)
    assert np.array_equal(a, oracle.terrain_generate(2, 5, 1))
    assert not np.array_equal(tile(a, 1, 2), tile(b, 1, 2))
    assert not np.array_equal(tile(a, 0, 2), tile(a, 1, 2))      # tiles draw from their own streams


def test_single_level_world_is_difficulty_zero():
    hf = oracle.terrain_generate(1, 5, 3)
    assert np.all(tile(hf, 0, 1) == 0.0)
    riser = np.float32(0.05)
    assert set(np.unique(tile(hf, 0, 4) / riser).round(4)) <= set(float(k) for k in range(11))
