"""Seeded synthetic inputs for the five BASELINE.json configurations (BJ:7-11).

Recipes follow SURVEY.md §8(d) ("Exact recipes"); every draw uses NumPy's PCG64
``default_rng(seed)`` in fp64 and is cast to fp32 at the end (BJ:7-11 say fp32
inputs; both the oracle and the CUDA path read the same fp32 bits).

Nothing here is the method: no Gram spectrum, no eigenvalue solve, no
recomposition.  ``eigh`` is used only to *sample* from a known Kronecker-sum
Gaussian N(0, (⊕Ψ)^-1) and ``qr`` only to draw orthonormal factors.

Configurations
--------------
C1  2-axis 200x100 matrix, ER(p=0.05) precisions, k=(100,100), top-5   (BJ:7)
C2  10,000 cells x 2,000 genes log1p(zero-inflated NB counts), k=(50,50), top-10 (BJ:8)
C3  400x300x200 tensor, ER(p=0.02) precisions, full rank, top-10       (BJ:9)
C4  factor-level axis n=200,000, k=64, top-10                           (BJ:10)
C5  factor-level axes n=1,000,000 and n=30,000, k=100, top-10           (BJ:11)
"""
from __future__ import annotations

import numpy as np

__all__ = [
    "er_precision", "ks_sample", "random_factor", "matrix_config", "config",
    "CONFIG_META", "small_tensor", "small_factor",
]

# Per-config metadata: seed, kind, shapes, ranks, top-t per row.
CONFIG_META = {
    "C1": dict(seed=1, kind="data", shape=(200, 100), k=(100, 100), t=5, p=0.05),
    "C2": dict(seed=2, kind="data", shape=(10000, 2000), k=(50, 50), t=10),
    "C3": dict(seed=3, kind="data", shape=(400, 300, 200), k=(400, 300, 200), t=10, p=0.02),
    "C4": dict(seed=4, kind="factor", axes=((200_000, 64),), t=10),
    "C5": dict(seed=5, kind="factor", axes=((1_000_000, 100), (30_000, 100)), t=10),
}


def er_precision(rng: np.random.Generator, d: int, p: float, delta: float = 0.1) -> np.ndarray:
    """Erdos-Renyi sparse precision (SURVEY §8(d) "ER precision per axis").

    Strict-upper mask ~ Bernoulli(p), off-diagonals U[-0.3,-0.1], symmetrized,
    diagonal = row |off-diagonal| sum + delta (diagonal dominance => PD).
    """
    mask = rng.random((d, d)) < p
    w = rng.uniform(-0.3, -0.1, (d, d))
    a = np.triu(mask * w, 1)
    psi = a + a.T
    psi[np.diag_indices(d)] = np.abs(psi).sum(axis=1) + delta
    return psi


def ks_sample(rng: np.random.Generator, psis) -> np.ndarray:
    """One draw of X ~ N(0, (⊕_l Ψ_l)^-1), first axis at the largest stride.

    Ψ_l = U_l D_l U_l^T;  W ~ N(0, 1/(Σ_l D_l[i_l]))  on the grid;
    X = W x_1 U_1 x_2 U_2 (x_3 U_3)   (mode-l product from the left).
    """
    decomp = [np.linalg.eigh(p) for p in psis]
    shape = tuple(p.shape[0] for p in psis)
    grid = np.zeros(shape)
    for ax, (dl, _) in enumerate(decomp):
        sh = [1] * len(shape)
        sh[ax] = shape[ax]
        grid = grid + dl.reshape(sh)
    w = rng.standard_normal(shape) / np.sqrt(grid)
    x = w
    for ax, (_, u) in enumerate(decomp):
        x = np.moveaxis(np.tensordot(u, x, axes=([1], [ax])), 0, ax)
    return np.ascontiguousarray(x)


def random_factor(rng: np.random.Generator, n: int, k: int):
    """Factor-level input (BJ:10-11): V = Q of reduced QR of an n x k N(0,1) matrix
    (fp64 Householder -> fp32), lambda ~ LogNormal(0,1) sorted descending.

    lambda is rounded to fp32 (the configs say fp32) and returned as float64 so
    both paths read the same values.  Draw order: G (n x k), then lambda (k).
    """
    g = rng.standard_normal((n, k))
    q, _ = np.linalg.qr(g, mode="reduced")
    v = np.ascontiguousarray(q, dtype=np.float32)
    lam = np.sort(rng.lognormal(0.0, 1.0, k))[::-1].astype(np.float32).astype(np.float64)
    return v, np.ascontiguousarray(lam)


def matrix_config(name: str) -> np.ndarray:
    meta = CONFIG_META[name]
    rng = np.random.default_rng(meta["seed"])
    if name == "C2":
        mu = rng.lognormal(0.0, 1.0, meta["shape"][1])
        counts = rng.negative_binomial(2, 2.0 / (2.0 + mu), size=meta["shape"])
        keep = rng.random(counts.shape) < 0.181
        return np.log1p(counts * keep).astype(np.float32)
    psis = [er_precision(rng, d, meta["p"]) for d in meta["shape"]]
    return np.ascontiguousarray(ks_sample(rng, psis), dtype=np.float32)


def config(name: str):
    """Return the seeded input of a configuration.

    data configs  -> dict(X=fp32 array, k=tuple, t=int)
    factor configs -> dict(axes=[(V fp32 n x k, lam float64 k), ...], t=int)
    """
    meta = CONFIG_META[name]
    if meta["kind"] == "data":
        return dict(X=matrix_config(name), k=meta["k"], t=meta["t"])
    rng = np.random.default_rng(meta["seed"])
    axes = [random_factor(rng, n, k) for (n, k) in meta["axes"]]
    return dict(axes=axes, t=meta["t"])


def small_tensor(seed: int, shape, p: float = 0.3) -> np.ndarray:
    """Small Kronecker-sum Gaussian tensor for brute-force tests (same ER recipe)."""
    rng = np.random.default_rng(seed)
    psis = [er_precision(rng, d, p) for d in shape]
    return np.ascontiguousarray(ks_sample(rng, psis), dtype=np.float32)


def small_factor(seed: int, n: int, k: int):
    rng = np.random.default_rng(seed)
    return random_factor(rng, n, k)
