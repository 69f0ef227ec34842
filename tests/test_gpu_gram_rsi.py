"""At-scale Gram spectrum (include/ggm.h (1b)): randomized subspace
iteration against the fp64 oracle (SVD of the matricisation, Alg. 1 lines 3-4) on small
inputs, and against a closed form at a size the dense Gram path refuses (both sides of the
unfolding > 32768): X = U diag(s) Wᵀ has S = U diag(s²) Uᵀ exactly."""
import numpy as np
import pytest
import torch

import oracle as O
from synth import gen

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def G():
    import paper_2407_19892_b200 as G
    assert torch.cuda.is_available()
    assert G.device_supported(), "needs an sm_100a (B200) device"
    return G


def _sin_max(A, B):
    """Largest principal angle sine between the column spaces of A and B (orthonormal)."""
    qa, _ = np.linalg.qr(A)
    qb, _ = np.linalg.qr(B)
    s = np.linalg.svd(qa.T @ qb, compute_uv=False)
    return float(np.sqrt(max(0.0, 1.0 - s.min() ** 2)))


def _low_rank_noise(seed, d, m, r0, noise):
    rng = np.random.default_rng(seed)
    U = np.linalg.qr(rng.standard_normal((d, r0)))[0]
    W = np.linalg.qr(rng.standard_normal((m, r0)))[0]
    s = np.geomspace(100.0, 5.0, r0)
    return ((U * s) @ W.T + noise * rng.standard_normal((d, m))).astype(np.float32)


@pytest.mark.parametrize("case", ["c1", "lowrank", "tensor", "tall"])
def test_rsi_vs_oracle(G, case):
    if case == "c1":
        X = gen.config("C1")["X"]
        axis, k = 0, 20
    elif case == "lowrank":
        X = _low_rank_noise(5, 3000, 5000, 60, 0.05)
        axis, k = 1, 25
    elif case == "tensor":
        rng = np.random.default_rng(9)
        X = rng.standard_normal((40, 30, 20)).astype(np.float32)
        X += (5 * np.outer(rng.standard_normal(40 * 30), rng.standard_normal(20))).reshape(40, 30, 20).astype(np.float32)
        axis, k = 1, 10
    else:
        X = _low_rank_noise(6, 20000, 800, 40, 0.01)
        axis, k = 0, 30
    Xd = torch.from_numpy(X).cuda()
    V, E, tr, it, ch = G.ggm_gram_eig_rsi(Xd, axis, k, max_iter=300, tol=1e-14)
    Vo, Eo = O.gram_eig(X.astype(np.float64), axis, k)
    E = E.cpu().numpy()
    np.testing.assert_allclose(E, Eo, rtol=1e-6)
    # top-k subspace (eigengap-limited individual vectors: compare the span)
    assert _sin_max(V.cpu().numpy().astype(np.float64), Vo) < 1e-3
    np.testing.assert_allclose(tr, float(np.sum(X.astype(np.float64) ** 2)), rtol=1e-10)


def test_rsi_closed_form_at_scale(G):
    """d = m = 40,000 (> 32768): ggm_gram_eig dispatches to the randomized path; the
    spectrum of X = U diag(s) Wᵀ is s² (fp32 rounding of X perturbs it at ~1e-7)."""
    d = m = 40_000
    r0, k = 24, 16
    g = torch.Generator(device="cuda").manual_seed(3)
    U = torch.linalg.qr(torch.randn(d, r0, device="cuda", dtype=torch.float64, generator=g))[0]
    W = torch.linalg.qr(torch.randn(m, r0, device="cuda", dtype=torch.float64, generator=g))[0]
    s = torch.logspace(3, 1, r0, device="cuda", dtype=torch.float64)
    X = ((U * s) @ W.T).float()
    del W
    V, E, tr = G.ggm_gram_eig(X, 0, k)
    torch.cuda.synchronize()
    np.testing.assert_allclose(E.cpu().numpy(), (s[:k] ** 2).cpu().numpy(), rtol=1e-5)
    Vn = V.double().cpu().numpy()
    assert _sin_max(Vn, U[:, :k].cpu().numpy()) < 1e-4
    np.testing.assert_allclose(np.linalg.norm(Vn, axis=0), 1.0, rtol=1e-5)
