"""Seeded synthetic stand-ins for the BASELINE.json configs.

The paper's datasets (US Census 1990, HEPMASS, CORD-19 embeddings, Gisette;
PAPER.md:257-260) are not available; these generators reproduce the stated
shapes, storage types and value distributions of BASELINE.json `configs`
(no dataset items are reproduced).  Every config takes a `scale` in (0, 1]
that shrinks m and s proportionally for parity tests (k, n unchanged).
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

DATA_SEED = 20220415  # fixed generator seed (documented in DESIGN.md)


@dataclass(frozen=True)
class Workload:
    name: str
    m: int
    n: int
    k: int
    s: int
    chunks: int
    dtype: str  # "f64" | "f32"
    seed: int = 0  # Big-means seed (BASELINE.json: seed 0)
    max_iterations: int = 300
    rel_tolerance: float = 1e-4
    candidates: int = 3


CONFIGS = {
    "c1": Workload("c1_gauss_100k_16", 100_000, 16, 10, 10_000, 50, "f64"),
    "c2": Workload("c2_aniso_int_2.5M_68", 2_500_000, 68, 25, 50_000, 200, "f64"),
    "c3": Workload("c3_outliers_10.5M_28_f32", 10_500_000, 28, 20, 100_000, 512, "f32"),
    "c4": Workload("c4_embed_600k_768_f32", 600_000, 768, 15, 20_000, 200, "f32"),
    "c5": Workload("c5_sparse_13.5k_5000", 13_500, 5000, 10, 4_000, 100, "f64"),
}


def scaled(w: Workload, scale: float, chunks: int | None = None) -> Workload:
    if scale >= 1.0 and chunks is None:
        return w
    m = max(int(w.m * scale), w.k * 4)
    s = max(min(int(w.s * scale), m), w.k)
    return Workload(w.name + f"@{scale:g}", m, w.n, w.k, s, chunks or w.chunks, w.dtype, w.seed,
                    w.max_iterations, w.rel_tolerance, w.candidates)


def generate(key: str, m: int | None = None, seed: int = DATA_SEED) -> np.ndarray:
    """Return the (m, n) matrix of config `key` (float64 or float32 storage)."""
    w = CONFIGS[key]
    m = m or w.m
    n = w.n
    rng = np.random.default_rng(seed + int(key[1]))
    if key == "c1":  # 10 centers U[-10,10]^16, equal weights, sigma 1, f64
        centers = rng.uniform(-10, 10, (10, n))
        lab = rng.integers(0, 10, m)
        return centers[lab] + rng.standard_normal((m, n))
    if key == "c2":  # 40 centers U[0,20]^68, per-dim scale log-U[0.1,10], integers, f64
        centers = rng.uniform(0, 20, (40, n))
        scales = np.exp(rng.uniform(np.log(0.1), np.log(10.0), n))
        out = np.empty((m, n), np.float64)
        step = 1 << 18
        for a in range(0, m, step):
            b = min(m, a + step)
            lab = rng.integers(0, 40, b - a)
            out[a:b] = np.rint(centers[lab] + rng.standard_normal((b - a, n)) * scales)
        return out
    if key == "c3":  # centers +-1 per dim, sigma 1, 5% U[-5,5]^28 outliers, f32
        out = np.empty((m, n), np.float32)
        step = 1 << 20
        for a in range(0, m, step):
            b = min(m, a + step)
            sign = np.where(rng.integers(0, 2, b - a) == 0, -1.0, 1.0)[:, None]
            x = sign + rng.standard_normal((b - a, n), dtype=np.float32)
            outl = rng.random(b - a) < 0.05
            x[outl] = rng.uniform(-5, 5, (int(outl.sum()), n))
            out[a:b] = x
        return out
    if key == "c4":  # 30 unit directions + N(0, 0.3^2), L2-normalised, f32
        dirs = rng.standard_normal((30, n))
        dirs /= np.linalg.norm(dirs, axis=1, keepdims=True)
        out = np.empty((m, n), np.float32)
        step = 1 << 15
        for a in range(0, m, step):
            b = min(m, a + step)
            lab = rng.integers(0, 30, b - a)
            x = dirs[lab] + 0.3 * rng.standard_normal((b - a, n))
            x /= np.linalg.norm(x, axis=1, keepdims=True)
            out[a:b] = x
        return out
    if key == "c5":  # 87% zeros; nonzeros integer U[1,999]; mask from 2 latent groups, f64
        groups = rng.integers(0, 2, m)
        active = np.zeros((2, n), bool)
        perm = rng.permutation(n)
        active[0, perm[: n // 2]] = True
        active[1, perm[n // 2:]] = True
        p = np.where(active, 0.26, 0.0)  # 0.5 * 0.26 = 13% nonzero overall
        mask = rng.random((m, n)) < p[groups]
        vals = rng.integers(1, 1000, (m, n)).astype(np.float64)
        return np.where(mask, vals, 0.0)
    raise KeyError(key)
