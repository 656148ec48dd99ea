"""Seeded synthetic inputs for the five BASELINE configurations (C1-C5).

BASELINE.json names synthetic laws only (no dataset), so these generators are
the workload. Draws happen in numpy float64 from ``np.random.default_rng(seed)``
in a fixed order; the point clouds are then rounded to float32 so that the GPU
path and the fp64 CPU oracle see the same representable coordinates
(SURVEY.md §8d "Synthetic inputs").

Variance notation follows SURVEY.md §8d: N(0, 0.01^2) means std 0.01,
N(0, 4I) std 2 per coordinate, N(0, 0.25) std 0.5, N(0, 1/D) std 1/sqrt(D).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

# per-config Sinkhorn/outer settings, as restated in SURVEY.md §8c/§8d
C1_EPS = 0.01
C2_EPS = 0.05
C3_EPS_STAGES = (0.1, 0.05, 0.025, 0.0125, 0.00625, 0.005)
C4_EPS = 0.01
C5_EPS = 0.02


@dataclass
class PointClouds:
    """Source/target point clouds (float32-representable fp64) and weights."""

    x: np.ndarray
    y: np.ndarray
    a: np.ndarray
    b: np.ndarray


@dataclass
class LowRankInstance:
    """C2 micro-benchmark instance: C_ij = a_i + b_j - 2 u_i.v_j, potential g."""

    u: np.ndarray
    v: np.ndarray
    row_sep: np.ndarray
    col_sep: np.ndarray
    g: np.ndarray
    log_wa: np.ndarray
    log_wb: np.ndarray
    eps: float


def _f32(x: np.ndarray) -> np.ndarray:
    return np.asarray(x, dtype=np.float32).astype(np.float64)


def haar_orthogonal(rng, d: int) -> np.ndarray:
    """Haar-distributed orthogonal matrix (QR of a Gaussian with sign fix)."""
    q, r = np.linalg.qr(rng.standard_normal((d, d)))
    return q * np.sign(np.diag(r))[None, :]


def _sphere(rng, n: int) -> np.ndarray:
    p = rng.standard_normal((n, 3))
    p /= np.linalg.norm(p, axis=1, keepdims=True)
    return p + 0.01 * rng.standard_normal((n, 3))


def _max_sq_pair(p: np.ndarray) -> float:
    """Largest pairwise squared distance. O(n^2): numpy up to 50k points (the
    sizes with golden vectors), blocked fp64 on the GPU above that (C1/C3-law
    clouds at 1e5-1e6 points would take hours on the host)."""
    if p.shape[0] > 50_000:
        import torch

        if torch.cuda.is_available():
            t = torch.as_tensor(p, dtype=torch.float64, device="cuda")
            sqt = (t * t).sum(1)
            best = 0.0
            for i0 in range(0, t.shape[0], 1024):
                blk = sqt[i0:i0 + 1024, None] + sqt[None, :] - 2.0 * t[i0:i0 + 1024] @ t.t()
                best = max(best, float(blk.max()))
            return best
    sq = (p**2).sum(axis=1)
    best = 0.0
    for i0 in range(0, p.shape[0], 2048):
        blk = sq[i0 : i0 + 2048, None] + sq[None, :] - 2.0 * p[i0 : i0 + 2048] @ p.T
        best = max(best, float(blk.max()))
    return best


def c1(seed: int = 0, n: int = 1000, m: int | None = None) -> PointClouds:
    """C1: noisy unit spheres in R^3, target Haar-rotated, max sq distance 1."""
    m = n if m is None else m
    rng = np.random.default_rng(seed)
    x = _sphere(rng, n)
    y = _sphere(rng, m) @ haar_orthogonal(rng, 3).T
    x = x / np.sqrt(_max_sq_pair(x))
    y = y / np.sqrt(_max_sq_pair(y))
    return PointClouds(_f32(x), _f32(y), np.full(n, 1.0 / n), np.full(m, 1.0 / m))


def c2(seed: int = 0, n: int = 1 << 20, m: int | None = None, k: int = 16) -> LowRankInstance:
    """C2: u, v ~ N(0, 1/k); separable a, b ~ U[0,1]; g ~ N(0,1); uniform weights."""
    m = n if m is None else m
    rng = np.random.default_rng(seed)
    std = 1.0 / np.sqrt(k)
    u = rng.standard_normal((n, k), dtype=np.float32) * np.float32(std)
    v = rng.standard_normal((m, k), dtype=np.float32) * np.float32(std)
    row_sep = rng.random(n, dtype=np.float32)
    col_sep = rng.random(m, dtype=np.float32)
    g = rng.standard_normal(m, dtype=np.float32)
    return LowRankInstance(
        u=u, v=v, row_sep=row_sep, col_sep=col_sep, g=g,
        log_wa=np.full(n, -np.log(n)), log_wb=np.full(m, -np.log(m)), eps=C2_EPS,
    )


def _torus(rng, n: int) -> np.ndarray:
    th = rng.random(n) * 2.0 * np.pi
    ph = rng.random(n) * 2.0 * np.pi
    rad = 1.0 + 0.3 * np.cos(ph)
    p = np.column_stack([rad * np.cos(th), rad * np.sin(th), 0.3 * np.sin(ph)])
    return p + 0.01 * rng.standard_normal((n, 3))


def c3(seed: int = 0, n: int = 100_000, m: int | None = None) -> PointClouds:
    """C3: noisy torus (R=1, r=0.3); target fresh torus, rotated, x1.2, translated."""
    m = n if m is None else m
    rng = np.random.default_rng(seed)
    x = _torus(rng, n)
    y = _torus(rng, m) @ haar_orthogonal(rng, 3).T * 1.2 + rng.standard_normal(3)[None, :]
    return PointClouds(_f32(x), _f32(y), np.full(n, 1.0 / n), np.full(m, 1.0 / m))


def c4(seed: int = 0, n: int = 1 << 20, m: int | None = None) -> PointClouds:
    """C4: 8-component GMM in R^3 (means N(0,4I), cov AA^T+0.05I, Dirichlet(1) mix)."""
    m = n if m is None else m
    rng = np.random.default_rng(seed)
    kc = 8
    means = 2.0 * rng.standard_normal((kc, 3))
    amat = 0.5 * rng.standard_normal((kc, 3, 3))
    covs = amat @ np.transpose(amat, (0, 2, 1)) + 0.05 * np.eye(3)[None]
    chol = np.linalg.cholesky(covs)
    mix = rng.dirichlet(np.ones(kc))

    def draw(count):
        lab = rng.choice(kc, size=count, p=mix)
        z = rng.standard_normal((count, 3))
        return means[lab] + np.einsum("nij,nj->ni", chol[lab], z)

    x = draw(n)
    y = draw(m) @ haar_orthogonal(rng, 3).T
    return PointClouds(_f32(x), _f32(y), np.full(n, 1.0 / n), np.full(m, 1.0 / m))


def _c5_side(rng, count: int, dim: int, kc: int = 16):
    means = 2.0 * rng.standard_normal((kc, dim))
    var = rng.uniform(0.05, 0.5, size=(kc, dim))
    mass = rng.dirichlet(np.ones(kc))
    # equal-size clusters (count/kc points each, contiguous); cluster mass is
    # spread uniformly over its points, then renormalised in fp64
    lab = np.minimum(np.arange(count) * kc // count, kc - 1)
    pts = means[lab] + np.sqrt(var[lab]) * rng.standard_normal((count, dim))
    sizes = np.bincount(lab, minlength=kc).astype(np.float64)
    w = mass[lab] / sizes[lab]
    w = w / w.sum()
    return pts, w


def c5(seed: int = 0, n: int = 1 << 18, m: int | None = None) -> PointClouds:
    """C5: 16-cluster GMMs, X in R^64 and Y in R^32, Dirichlet cluster masses."""
    m = n if m is None else m
    rng = np.random.default_rng(seed)
    x, a = _c5_side(rng, n, 64)
    y, b = _c5_side(rng, m, 32)
    return PointClouds(_f32(x), _f32(y), a, b)


GENERATORS = {"C1": c1, "C3": c3, "C4": c4, "C5": c5}
