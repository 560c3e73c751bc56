"""Seeded synthetic inputs for the exact-ddKS hot path (shared by tests, bench.py and smoke()).

This module holds NONE of the method's arithmetic: it only draws samples. It is the one module the
oracle side (tests/, oracle/) and the CUDA side (the binding) may both use.

Recipes follow BASELINE.json ``configs`` and SURVEY.md §8d (the paper's datasets GVM/Skew/DVU/GVS/MM,
P:L319-324, have unstated parameters; these fixed recipes stand in for them — DESIGN.md "Inputs").
NumPy ``default_rng`` (PCG64) draws in float64, then ONE cast to float32 (round-to-nearest-even).
P is drawn before Q. NumPy does not promise cross-version stream stability, so the bytes are the contract:
``sha256(P.tobytes() + Q.tobytes())`` is pinned in SURVEY_SHA256 (NumPy 2.3.5).
"""
from __future__ import annotations

import hashlib

import numpy as np

# SURVEY.md §8d "Input sha256 (P bytes then Q bytes, C-order float32; NumPy 2.3.5)"
SURVEY_SHA256 = {
    "C1": "c15b89ae7163ed64c708a0757fe2bcb5ee5d9cb60a0cd65b9d04bedb29cd6a4d",
    "C2": "8af671a8cdc57817e0db949c9e41416949e3e5c3003e9ab37dc966e170d78f03",
    "C3": "6ca09c94e00a20c2d5e209d18b9d6b0f2543a9cd6b31c530783f540b0229a8d2",
    "C4": "2cd268e7fbf1b45345f6ceb99e6bea86da6de6dea3e605853db004c59626cfe3",
    "C4_perms": "a557fdf25f9ab5c370352e0f4215a4d27868107bb3dde76f9410ca52a69dec46",
    "C5": "0893b0ba96b4565dbacbeba66bc31e38ab2e4ebc25791e6a9ca03cde8962132d",
}

CONFIG_NAMES = {
    "C1": "ddks d=3 n_P=n_Q=200 GVM-like (mean shift 0.1), seed 0",
    "C2": "ddks d=3 n_P=n_Q=10000 uniform vs skewed coordinate 2 (U^1.2), seed 1",
    "C3": "ddks d=8 n_P=n_Q=20000 N(0,I) vs tridiagonal-covariance N(0,Sigma), seed 2",
    "C4": "ddks batch 4096 pairs d=4 n_P=n_Q=512 (half null, half scale 1.15) + 1000-permutation null, seed 3",
    "C5": "ddks d=5 n_P=n_Q=1000000 N(0,I) vs 0.9 N(0,I) + 0.1 N(0.5,0.25 I) mixture, seed 4",
}


def sha256_pq(P: np.ndarray, Q: np.ndarray) -> str:
    h = hashlib.sha256()
    h.update(np.ascontiguousarray(P, dtype=np.float32).tobytes())
    h.update(np.ascontiguousarray(Q, dtype=np.float32).tobytes())
    return h.hexdigest()


def f32(a: np.ndarray) -> np.ndarray:
    return np.ascontiguousarray(a.astype(np.float32))


def config(name: str):
    """Return (P, Q) float32 arrays for C1, C2, C3, C5, or (P[B,n,d], Q[B,n,d]) for C4."""
    if name == "C1":
        rng = np.random.default_rng(0)
        P = rng.standard_normal((200, 3))
        Q = rng.standard_normal((200, 3)) + 0.1
        return f32(P), f32(Q)
    if name == "C2":
        rng = np.random.default_rng(1)
        P = rng.random((10_000, 3))
        Q = rng.random((10_000, 3))
        Q[:, 2] = Q[:, 2] ** 1.2
        return f32(P), f32(Q)
    if name == "C3":
        rng = np.random.default_rng(2)
        P = rng.standard_normal((20_000, 8))
        Z = rng.standard_normal((20_000, 8))
        sigma = np.eye(8) + 0.2 * (np.eye(8, k=1) + np.eye(8, k=-1))
        Q = Z @ np.linalg.cholesky(sigma).T
        return f32(P), f32(Q)
    if name == "C4":
        rng = np.random.default_rng(3)
        B, n, d = 4096, 512, 4
        P = np.empty((B, n, d))
        Q = np.empty((B, n, d))
        for b in range(B):
            P[b] = rng.standard_normal((n, d))
            Q[b] = rng.standard_normal((n, d)) * (1.15 if b >= 2048 else 1.0)
        return f32(P), f32(Q)
    if name == "C5":
        rng = np.random.default_rng(4)
        n, d = 1_000_000, 5
        P = rng.standard_normal((n, d))
        z = rng.random(n) < 0.1
        A = rng.standard_normal((n, d))
        Q = np.where(z[:, None], 0.5 + 0.5 * A, A)
        return f32(P), f32(Q)
    raise KeyError(name)


C4_PERM_PAIR = 2048  # pooled pair for the permutation null = first alternative pair


def c4_perms(n_perm: int = 1000, N: int = 1024) -> np.ndarray:
    """Label-shuffle permutations for C4b: default_rng([3, 1]).permutation(N), n_perm times, int32 [n_perm, N]."""
    rng = np.random.default_rng([3, 1])
    return np.ascontiguousarray(np.stack([rng.permutation(N) for _ in range(n_perm)]).astype(np.int32))


def random_pair(seed: int, n_P: int, n_Q: int, d: int, kind: str = "normal"):
    """Small seeded parity inputs. kind: 'normal' (continuous), 'grid' (integer grid 0..3: tie-heavy),
    'mixed' (half grid, half normal), 'dup' (repeated rows)."""
    rng = np.random.default_rng(seed)
    if kind == "normal":
        P = rng.standard_normal((n_P, d))
        Q = rng.standard_normal((n_Q, d)) + 0.25
    elif kind == "grid":
        P = rng.integers(0, 4, (n_P, d)).astype(np.float64)
        Q = rng.integers(0, 4, (n_Q, d)).astype(np.float64)
    elif kind == "mixed":
        P = rng.standard_normal((n_P, d))
        Q = rng.standard_normal((n_Q, d))
        P[:, 0] = np.round(P[:, 0])
        Q[:, : max(1, d // 2)] = np.round(Q[:, : max(1, d // 2)])
    elif kind == "dup":
        base = rng.standard_normal((max(1, (n_P + n_Q) // 4), d))
        P = base[rng.integers(0, len(base), n_P)]
        Q = base[rng.integers(0, len(base), n_Q)] * 1.5
    else:
        raise KeyError(kind)
    return f32(P), f32(Q)
