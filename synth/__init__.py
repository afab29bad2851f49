"""synth -- seeded input generators shared by the CUDA path's tests/bench and the oracle's tests.

Holds none of the method's arithmetic: it only synthesises *inputs* shaped like the
paper's workloads --
  * the tiled world heightfield (SPEC terrain module S:25-93: 5 terrain types as columns, difficulty
    levels as rows, 8 m tiles at 0.1 m), generated once on the host;
  * initial network parameters (R19: U(±1/sqrt(fan_in)), log-std 0);
  * synthetic rollout storage for kernel micro-benchmarks and parity cases.
"""
from __future__ import annotations

import math

import numpy as np

TILE_CELLS = 80  # 8 m / 0.1 m
CELL = 0.1


def _tile_rng(seed: int, level: int, col: int) -> np.random.Generator:
    return np.random.default_rng([seed & 0xFFFFFFFF, level, col, 0x7e77a1])


def _edge_dist():
    c = (np.arange(TILE_CELLS) + 0.5) * CELL
    d1 = np.minimum(c, 8.0 - c)
    return np.minimum(d1[:, None], d1[None, :])  # distance of each cell centre to the tile border


def generate_tile(kind: int, level: int, n_levels: int, seed: int, col: int = 0) -> np.ndarray:
    """One 80x80 tile. kind = col mod 5: 0 flat, 1 slope pyramid, 2 rough, 3 obstacles,
    4 stairs pyramid. Difficulty d = level/(L-1): riser 0.05+0.15d, slope 25°·d, rough p-p
    0.05(1+d), obstacles ±(0.05+0.15d)."""
    d = level / max(n_levels - 1, 1)
    rng = _tile_rng(seed, level, col)
    e = _edge_dist()
    plateau = 3.0  # central 2 m x 2 m spawn plateau
    if kind == 0:
        h = np.zeros((TILE_CELLS, TILE_CELLS))
    elif kind == 1:
        h = math.tan(math.radians(25.0 * d)) * np.minimum(e, plateau)
    elif kind == 2:
        a = 0.05 * (1.0 + d)
        h = rng.uniform(-0.5 * a, 0.5 * a, size=(TILE_CELLS, TILE_CELLS))
    elif kind == 3:
        hmax = 0.05 + 0.15 * d
        h = np.zeros((TILE_CELLS, TILE_CELLS))
        for _ in range(8):
            w, l = rng.uniform(0.5, 2.0, size=2)
            x0, y0 = rng.uniform(0.0, 8.0, size=2)
            hh = rng.uniform(-hmax, hmax)
            i0, i1 = int(x0 / CELL), int(min(8.0, x0 + w) / CELL)
            j0, j1 = int(y0 / CELL), int(min(8.0, y0 + l) / CELL)
            h[i0:i1, j0:j1] = hh
        h[e >= plateau] = 0.0
    elif kind == 4:
        riser = 0.05 + 0.15 * d
        h = riser * np.floor(np.minimum(e, plateau) / 0.3)
    else:
        raise ValueError(kind)
    return h.astype(np.float32)


def make_world(n_levels: int = 10, n_cols: int = 20, seed: int = 0, rough: bool = True) -> np.ndarray:
    """Merged world [n_levels*80][n_cols*80] fp32; level along x, column along y (R21)."""
    R, C = n_levels * TILE_CELLS, n_cols * TILE_CELLS
    hf = np.zeros((R, C), np.float32)
    if rough:
        for lv in range(n_levels):
            for c in range(n_cols):
                hf[lv * 80:(lv + 1) * 80, c * 80:(c + 1) * 80] = generate_tile(c % 5, lv, n_levels, seed, c)
    return hf


def init_params(obs_dim: int, hidden=(512, 256, 128), act_dim: int = 12, seed: int = 0,
                logstd: float = 0.0) -> np.ndarray:
    """Flat fp32 θ in the canonical order of DESIGN.md §3.8, U(±1/sqrt(fan_in)) (R19)."""
    rng = np.random.default_rng([seed & 0xFFFFFFFF, 0x5eed])
    parts = []
    for out in (act_dim, 1):
        dims = [obs_dim, *hidden, out]
        for l in range(4):
            bound = 1.0 / math.sqrt(dims[l])
            parts.append(rng.uniform(-bound, bound, size=dims[l + 1] * dims[l]))
            parts.append(rng.uniform(-bound, bound, size=dims[l + 1]))
    parts.append(np.full(act_dim, logstd))
    return np.concatenate(parts).astype(np.float32)


def synthetic_storage(T: int, N: int, obs_dim: int, seed: int = 0, p_term: float = 0.01,
                      p_timeout: float = 0.002):
    """Synthetic rollout batch (SURVEY §8(d) 'kernel microbenchmarks use synthetic storage')."""
    rng = np.random.default_rng([seed & 0xFFFFFFFF, 0x57a6e])
    term = (rng.random((T, N)) < p_term).astype(np.uint8)
    timeout = ((rng.random((T, N)) < p_timeout) & (term == 0)).astype(np.uint8)
    return dict(
        obs=rng.standard_normal((T, N, obs_dim)).astype(np.float32),
        act=rng.standard_normal((T, N, 12)).astype(np.float32),
        mu=(0.3 * rng.standard_normal((T, N, 12))).astype(np.float32),
        logp=(-17.0 + rng.standard_normal((T, N))).astype(np.float32),
        V=rng.standard_normal((T, N)).astype(np.float32),
        r=(0.02 * rng.standard_normal((T, N))).astype(np.float32),
        b=(timeout * rng.standard_normal((T, N))).astype(np.float32),
        term=term, timeout=timeout,
        V_T=rng.standard_normal(N).astype(np.float32),
        logstd_old=np.zeros(12, np.float32),
    )
