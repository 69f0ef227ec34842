"""GPU parity of the multi-modal (shared-axis) steps, §8(f) row 4: the concatenated-axis
spectrum (Alg. 1 line 2) and the Σ_γ eigenvalue MLE (Thm 2), through the
C ABI, against oracle.gram_eig_multi / oracle.solve_eigvals_multi."""
import numpy as np
import pytest
import torch

import oracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def G():
    import paper_2407_19892_b200 as G
    assert torch.cuda.is_available()
    assert G.device_supported(), "needs an sm_100a (B200) device"
    return G


def _dataset(seed=0):
    """Three modalities over 5 global axes: X1 (axes 0, 1), X2 stored as (axis 2, axis 1),
    X3 a tensor (axes 3, 4, 1); axis 1 is shared by all three.  Every axis full rank."""
    rng = np.random.default_rng(seed)
    X1 = rng.standard_normal((30, 40)).astype(np.float32)
    X2 = (0.5 * rng.standard_normal((25, 40))).astype(np.float32)
    X3 = rng.standard_normal((10, 12, 40)).astype(np.float32)
    return [X1, X2, X3], [[0, 1], [2, 1], [3, 4, 1]], [30, 40, 25, 10, 12]


def _angles(Va, Vb):
    """Largest per-eigenvector deviation 1 - |<v_gpu, v_oracle>| (distinct eigenvalues on
    random data; signs are arbitrary on the oracle side)."""
    d = np.abs(np.sum(np.asarray(Va, np.float64) * np.asarray(Vb, np.float64), axis=0))
    return float(np.max(1.0 - d))


@pytest.mark.parametrize("axis", [0, 1, 2, 3, 4])
def test_gram_eig_multi_matches_oracle(G, axis):
    T, mods, ks = _dataset()
    k = ks[axis]
    Xd = [torch.from_numpy(x).cuda() for x in T]
    pos = [m.index(axis) if axis in m else -1 for m in mods]
    V, E, tr = G.ggm_gram_eig_multi([x if p >= 0 else None for x, p in zip(Xd, pos)], pos, k)
    Vo, Eo = O.gram_eig_multi(T, mods, axis, k)
    assert np.allclose(E.cpu().numpy(), Eo, rtol=1e-9)
    want_tr = sum(float(np.sum(np.asarray(x, np.float64) ** 2)) for x, m in zip(T, mods) if axis in m)
    assert abs(tr - want_tr) <= 1e-9 * want_tr
    assert _angles(V.cpu().numpy(), Vo) < 1e-5


def test_gram_eig_multi_dual_side(G):
    """Shared axis longer than the concatenated other side (the Σm x Σm Gram path)."""
    rng = np.random.default_rng(4)
    X1 = rng.standard_normal((20, 300)).astype(np.float32)
    X2 = rng.standard_normal((15, 300)).astype(np.float32)
    mods = [[0, 1], [2, 1]]
    V, E, _ = G.ggm_gram_eig_multi([torch.from_numpy(X1).cuda(), torch.from_numpy(X2).cuda()],
                                   [1, 1], 30)
    Vo, Eo = O.gram_eig_multi([X1, X2], mods, 1, 30)
    assert np.allclose(E.cpu().numpy(), Eo, rtol=1e-9)
    assert _angles(V.cpu().numpy(), Vo) < 1e-5


def test_solve_eigvals_multi_matches_oracle(G):
    T, mods, ks = _dataset()
    E = [O.gram_eig_multi(T, mods, a, ks[a])[1] for a in range(len(ks))]
    Ed = torch.from_numpy(np.concatenate(E)).cuda()
    lam, info = G.ggm_solve_eigvals_multi(Ed, ks, mods, tol=1e-9)
    ref, rinfo = O.solve_eigvals_multi(E, mods, tol=1e-12)
    assert info["stationarity"] <= 1e-9
    got = np.split(lam.cpu().numpy(), np.cumsum(ks)[:-1])
    for sg, so in zip(O.grid_sums_multi(got, mods), O.grid_sums_multi(ref, mods)):
        assert np.allclose(sg, so, rtol=1e-6)
    for a in range(len(ks)):                      # gauge 0 on both sides (reading G2)
        assert np.allclose(got[a], ref[a], rtol=1e-6, atol=1e-9 * np.abs(ref[a]).max())
    assert abs(info["nll"] - rinfo["nll"]) <= 1e-6 * abs(rinfo["nll"])
    assert info["trace_inconsistency"] < 1e-9


def test_solve_multi_single_modality_equals_single(G):
    rng = np.random.default_rng(7)
    X = rng.standard_normal((20, 15, 12)).astype(np.float32)
    ks = [20, 15, 12]             # full rank: an interior MLE (reading T)
    Xd = torch.from_numpy(X).cuda()
    E = torch.cat([G.ggm_gram_eig(Xd, a, k)[1] for a, k in enumerate(ks)])
    a, ia = G.ggm_solve_eigvals(E, ks, tol=1e-9)
    b, ib = G.ggm_solve_eigvals_multi(E, ks, [[0, 1, 2]], tol=1e-9)
    assert ia["iterations"] == ib["iterations"]
    assert torch.allclose(a, b, rtol=1e-12, atol=0)


def test_solve_multi_rejects_bad_modalities(G):
    E = torch.ones(6, dtype=torch.float64, device="cuda")
    with pytest.raises(G.GGMError):
        G.ggm_solve_eigvals_multi(E, [3, 3], [[0, 0]])      # repeated axis
    with pytest.raises(G.GGMError):
        G.ggm_solve_eigvals_multi(E, [3, 3], [[0]])         # axis 1 in no modality
