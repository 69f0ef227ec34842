"""GPU parity of ggm_grid_marginals / ggm_solve_eigvals (Thm 2, Alg. 1 lines 5-17) and
ggm_gram_eig (Alg. 1 lines 1-4, Thm 1) against the fp64 oracle, through the C ABI."""
import numpy as np
import pytest
import torch

import oracle as O
from synth import gen

pytestmark = pytest.mark.gpu

EIG_REL = 1e-5   # north_star: eigenvalues within 1e-5 relative


@pytest.fixture(scope="module")
def G():
    import paper_2407_19892_b200 as G
    assert G.device_supported()
    return G


def _cat(xs):
    return torch.from_numpy(np.concatenate([np.asarray(x, np.float64) for x in xs])).cuda()


@pytest.mark.parametrize("ks", [(2, 2), (5,), (7, 3, 4), (40, 30, 20), (130, 3), (1, 600),
                                (3, 2, 2, 3, 2)])
def test_grid_marginals(G, ks):
    rng = np.random.default_rng(len(ks) * 100 + sum(ks))
    lams = [rng.uniform(0.05, 2.0, k) for k in ks]
    g, ls = G.ggm_grid_marginals(_cat(lams), ks, with_logsum=True)
    want = np.concatenate(O.marginals(lams))
    np.testing.assert_allclose(g.cpu().numpy(), want, rtol=2e-6)
    assert ls == pytest.approx(float(np.log(O.grid_sums(lams)).sum()), rel=1e-6)


def test_grid_marginals_golden(G):
    g = G.ggm_grid_marginals(_cat([[1.0, 2.0], [3.0, 4.0]]), (2, 2))
    np.testing.assert_allclose(g.cpu().numpy(), [0.45, 0.36666666666666664] * 2, rtol=1e-6)


def _split(x, ks):
    off = np.cumsum([0] + list(ks))
    return [x[off[i]:off[i + 1]] for i in range(len(ks))]


@pytest.mark.parametrize("shape", [(20, 10), (6, 5, 4), (30, 20, 10)])
def test_solve_matches_oracle(G, shape):
    x = gen.small_tensor(sum(shape), shape)
    ks = []
    Es = []
    for l, d in enumerate(shape):
        k = min(d, int(np.prod(shape)) // d)
        _, E = O.gram_eig(x, l, k)
        ks.append(k)
        Es.append(E)
    lo, _ = O.solve_eigvals(Es, tol=1e-13)
    lam, info = G.ggm_solve_eigvals(_cat(Es), ks, tol=2e-8)
    lg = _split(lam.cpu().numpy(), ks)
    # gauge-free comparison: grid sums, then the canonical (gauge 0) λ
    np.testing.assert_allclose(O.grid_sums(lg), O.grid_sums(lo), rtol=EIG_REL)
    for a, b in zip(lg, lo):
        np.testing.assert_allclose(a, b, rtol=EIG_REL)
    assert O.stationarity(Es, lg) < 1e-6
    assert info["stationarity"] <= 2e-8
    assert info["nll"] == pytest.approx(O.nll(Es, lo), rel=1e-6, abs=1e-6)


def test_solve_isotropic_closed_form_c3_size(G):
    """E_l = (T/k_l)·1 ⇒ every grid sum = Πk/T, at the full C3 grid (24M points)."""
    ks = (400, 300, 200)
    T = 123.0
    E = [np.full(k, T / k) for k in ks]
    lam, info = G.ggm_solve_eigvals(_cat(E), ks, tol=1e-7)
    lg = _split(lam.cpu().numpy(), ks)
    s = O.grid_sums([l.astype(np.float64) for l in lg])
    np.testing.assert_allclose(s, np.prod(ks) / T, rtol=1e-5)
    assert info["iterations"] <= 2


def test_solve_single_axis(G):
    E = np.array([4.0, 2.0, 0.5])
    lam, info = G.ggm_solve_eigvals(_cat([E]), (3,), gauge=1)
    np.testing.assert_allclose(lam.cpu().numpy(), 1.0 / E, rtol=1e-6)


def test_solve_domain_error(G):
    with pytest.raises(G.GGMError) as e:
        G.ggm_solve_eigvals(_cat([[1.0, -2.0], [1.0, 1.0]]), (2, 2))
    assert e.value.status == 3


@pytest.mark.parametrize("shape,axis,k", [((200, 100), 0, 100), ((200, 100), 1, 100),
                                          ((50, 80), 0, 20), ((12, 9, 7), 1, 9),
                                          ((40, 3, 2), 0, 6), ((64, 48, 30), 2, 30)])
def test_gram_eig(G, shape, axis, k):
    x = gen.small_tensor(sum(shape) + axis, shape)
    V, E, tr = G.ggm_gram_eig(torch.from_numpy(x).cuda(), axis, k)
    Vo, Eo = O.gram_eig(x, axis, k)
    np.testing.assert_allclose(E.cpu().numpy(), Eo, rtol=1e-9)
    assert tr == pytest.approx(float(np.sum(x.astype(np.float64) ** 2)), rel=1e-12)
    Vg = V.cpu().numpy().astype(np.float64)
    # subspace agreement (largest principal angle) and orthonormality
    sv = np.linalg.svd(Vg.T @ Vo, compute_uv=False)
    assert sv.min() > 1 - 1e-5
    np.testing.assert_allclose(Vg.T @ Vg, np.eye(k), atol=1e-5)


def test_gram_eig_matrix_axes_share_spectrum(G):
    """Reading T: both axes of a matrix get the bitwise-identical spectrum."""
    x = gen.small_tensor(3, (60, 25))
    xd = torch.from_numpy(x).cuda()
    _, E0, _ = G.ggm_gram_eig(xd, 0, 25)
    _, E1, _ = G.ggm_gram_eig(xd, 1, 25)
    assert torch.equal(E0, E1)


def test_gram_eig_rank_error(G):
    x = gen.small_tensor(3, (6, 3))
    with pytest.raises(G.GGMError) as e:
        G.ggm_gram_eig(torch.from_numpy(x).cuda(), 0, 4)
    assert e.value.status == 2


@pytest.mark.parametrize("shape,k0,k1", [((200, 100), 100, 100), ((10000, 2000), 50, 50),
                                         ((300, 700), 40, 25), ((64, 64), 64, 64)])
def test_gram_eig_matrix_both_axes(G, shape, k0, k1):
    """One Gram + one eigensolve for both axes of a matrix equals the per-axis calls and the
    oracle (Thm 1 / P:125)."""
    import oracle as O
    rng = np.random.default_rng(sum(shape))
    X = rng.standard_normal(shape).astype(np.float32)
    Xd = torch.from_numpy(X).cuda()
    V0, E0, V1, E1, tr = G.ggm_gram_eig_matrix(Xd, k0, k1)
    for V, E, axis, k in ((V0, E0, 0, k0), (V1, E1, 1, k1)):
        Vo, Eo = O.gram_eig(X, axis, k)
        np.testing.assert_allclose(E.cpu().numpy(), Eo, rtol=1e-9)
        d = np.abs(np.sum(V.cpu().numpy().astype(np.float64) * Vo, axis=0))
        assert np.all(1.0 - d[:min(k, 20)] < 1e-5)
        Vs, Es, _ = G.ggm_gram_eig(Xd, axis, k)
        np.testing.assert_allclose(E.cpu().numpy(), Es.cpu().numpy(), rtol=1e-10)
    assert abs(tr - float(np.sum(X.astype(np.float64) ** 2))) < 1e-9 * tr


@pytest.mark.parametrize("cfg_name", ["C1", "C3"])
def test_gram_eig_axes_concurrent(G, cfg_name):
    """Every axis at once on side streams (include/ggm.h (1h)) equals the per-axis calls
    (same kernels; the trace and library reductions may sum in another order) and the
    oracle's spectra."""
    cfg = gen.config(cfg_name)
    X = cfg["X"]
    Xd = torch.from_numpy(X).cuda()
    res, tr = G.ggm_gram_eig_axes(Xd, cfg["k"])
    for a, (V, E) in enumerate(res):
        Vs, Es, trs = G.ggm_gram_eig(Xd, a, cfg["k"][a])
        np.testing.assert_allclose(E.cpu().numpy(), Es.cpu().numpy(), rtol=1e-11)
        assert float((V - Vs).abs().max()) <= 1e-5
        assert abs(tr - trs) <= 1e-12 * trs
        _, Eo = O.gram_eig(X, a, min(cfg["k"][a], 20))
        np.testing.assert_allclose(E.cpu().numpy()[:len(Eo)], Eo, rtol=1e-9)


def test_gram_eig_axes_rank_error(G):
    x = np.random.default_rng(3).standard_normal((6, 5, 4)).astype(np.float32)
    with pytest.raises(G.GGMError) as e:
        G.ggm_gram_eig_axes(torch.from_numpy(x).cuda(), [6, 5, 5])  # k_2 = 5 > d_2 = 4
    assert e.value.status_name == "GGM_ERR_RANK"


def test_solve_methods_same_grid(G):
    """Method 0 (SQUAREM-accelerated majorise-minimise) and method 1 (the plain MM step)
    reach the same grid at C2 (BK4), method 0 in fewer passes; a method-0 run that
    cannot converge within max_iter reports GGM_ERR_NO_CONVERGENCE."""
    cfg = gen.config("C2")
    X = torch.from_numpy(cfg["X"]).cuda()
    Ec = torch.cat([G.ggm_gram_eig(X, a, k)[1] for a, k in enumerate(cfg["k"])])
    lam1, info1 = G.ggm_solve_eigvals(Ec, cfg["k"], method=1)
    lam0, info0 = G.ggm_solve_eigvals(Ec, cfg["k"], method=0)
    assert info0["iterations"] < info1["iterations"]
    s = [O.grid_sums(_split(l.cpu().numpy(), cfg["k"])) for l in (lam1, lam0)]
    np.testing.assert_allclose(s[1], s[0], rtol=1e-5)
    with pytest.raises(G.GGMError) as e:
        G.ggm_solve_eigvals(Ec, cfg["k"], max_iter=3)
    assert e.value.status == 4


def _truncated(seed, shape=(9, 7, 6), ks=(4, 3, 5)):
    x = gen.small_tensor(seed, shape)
    return [O.gram_eig(x, l, k)[1] for l, k in enumerate(ks)], list(ks)


@pytest.mark.parametrize("seed", [1, 2, 3])
@pytest.mark.parametrize("gauge", [0, 1])
def test_solve_barrier_truncated_tensor(G, seed, gauge):
    """Reading T: a truncated 3-axis tensor (unequal traces) has its MLE on the barrier
    λ >= ε (Lemma 6).  GPU λ and floor set equal the oracle's active-set
    Newton; floor_active on both sides."""
    Es, ks = _truncated(seed)
    lo, oinfo = O.solve_eigvals(Es, gauge=gauge)
    assert oinfo["floor_active"]
    lam, info = G.ggm_solve_eigvals(_cat(Es), ks, gauge=gauge, tol=1e-9)
    lg = _split(lam.cpu().numpy(), ks)
    assert info["floor_active"] == 1
    eps = oinfo["eps"]
    for a, b in zip(lg, lo):
        on_o = b <= eps * (1 + 1e-9)
        on_g = a <= eps * (1 + 1e-9)
        assert np.array_equal(on_o, on_g)
        np.testing.assert_allclose(a, b, rtol=EIG_REL, atol=1e-3 * eps)
    np.testing.assert_allclose(O.grid_sums(lg), O.grid_sums(lo), rtol=EIG_REL)
    assert O.kkt_residual(Es, lg, eps * (1 + 1e-9)) <= 1e-6


def test_solve_barrier_matrix_unequal_ranks(G):
    """A matrix with k0 != k1: barrier regime on both sides, same λ."""
    x = gen.small_tensor(41, (30, 20))
    Es = [O.gram_eig(x, 0, 12)[1], O.gram_eig(x, 1, 6)[1]]
    lo, oinfo = O.solve_eigvals(Es)
    lam, info = G.ggm_solve_eigvals(_cat(Es), (12, 6), tol=1e-9)
    lg = _split(lam.cpu().numpy(), (12, 6))
    assert info["floor_active"] == 1 and oinfo["floor_active"]
    for a, b in zip(lg, lo):
        np.testing.assert_allclose(a, b, rtol=EIG_REL, atol=1e-3 * oinfo["eps"])


@pytest.mark.parametrize("shape", [(20, 10), (6, 5, 4), (12, 9, 7)])
def test_solve_gauge1_matches_oracle(G, shape):
    """Gauge 1 = Algorithm 1's gauge, (λ − 1/E) ⊥ G (L >= 2), against the oracle's gauge 1."""
    x = gen.small_tensor(sum(shape) + 5, shape)
    ks = [min(d, int(np.prod(shape)) // d) for d in shape]
    Es = [O.gram_eig(x, l, k)[1] for l, k in enumerate(ks)]
    lo, _ = O.solve_eigvals(Es, tol=1e-13, gauge=1)
    lam, info = G.ggm_solve_eigvals(_cat(Es), ks, gauge=1, tol=1e-9)
    lg = _split(lam.cpu().numpy(), ks)
    for a, b in zip(lg, lo):
        np.testing.assert_allclose(a, b, rtol=EIG_REL, atol=EIG_REL * max(np.abs(b).max(), 1e-30))
    d = [float(np.sum(l - 1.0 / e)) for l, e in zip(lg, Es)]
    np.testing.assert_allclose(d, d[0], rtol=1e-6, atol=1e-9 * max(abs(v) for v in d))
    assert info["floor_active"] == 0


def test_solve_method2_algorithm1_matches_oracle(G):
    """Method 2 = Algorithm 1 as printed (readings Q1-Q3) vs oracle.paper_gd_solve: the same
    deterministic iteration (μ halving on infeasible / non-decreasing steps) reaches the same λ
    (gauge 1 is what gradient descent preserves)."""
    rng = np.random.default_rng(4)
    Es = [rng.uniform(1.0, 2.0, 3), rng.uniform(1.0, 2.0, 2)]
    Es[1] *= Es[0].sum() / Es[1].sum()
    lo, oi = O.paper_gd_solve(Es, tol=1e-8)
    lam, info = G.ggm_solve_eigvals(_cat(Es), (3, 2), method=2, gauge=1, tol=1e-8)
    lg = _split(lam.cpu().numpy(), (3, 2))
    for a, b in zip(lg, lo):
        np.testing.assert_allclose(a, b, rtol=1e-6)
    assert abs(info["iterations"] - oi["iterations"]) <= 2
    assert info["stationarity"] <= 1e-8


def test_solve_method2_trace_inconsistent_does_not_converge(G):
    """Algorithm 1 as printed bounds only the grid minimum (reading Q3), so with unequal
    traces the NLL decreases without bound along the gauge: no convergence (the barrier MLE
    needs method 0/1)."""
    Es, ks = _truncated(2)
    with pytest.raises(G.GGMError) as e:
        G.ggm_solve_eigvals(_cat(Es), ks, method=2, max_iter=2000)
    assert e.value.status == 4


def test_solve_multi_barrier(G):
    """Reading T with the multi-modal gauge space: one modality through the multi-modal entry
    equals the single-modality barrier solve."""
    Es, ks = _truncated(3)
    lam1, _ = G.ggm_solve_eigvals(_cat(Es), ks, tol=1e-9)
    lam2, info = G.ggm_solve_eigvals_multi(_cat(Es), ks, [[0, 1, 2]], tol=1e-9)
    assert info["floor_active"] == 1
    np.testing.assert_allclose(lam2.cpu().numpy(), lam1.cpu().numpy(), rtol=1e-7)


def test_gram_eig_axes_with_rsi_axis(G):
    """(1h) with one axis beyond the dense Gram (33,000 rows, complement 40,000: randomized
    subspace iteration on `stream` after the concurrent dense axes): every axis equals its
    per-axis call.  Rank-4 CP tensor + small noise, k = 4 on every axis."""
    g = torch.Generator(device="cuda").manual_seed(5)
    shape = (33000, 200, 200)
    fs = [torch.randn(d, 4, device="cuda", generator=g) for d in shape]
    w = torch.tensor([8.0, 4.0, 2.0, 1.0], device="cuda")
    X = torch.einsum("ir,jr,lr,r->ijl", fs[0], fs[1], fs[2], w)
    X += 1e-3 * torch.randn(shape, device="cuda", generator=g)
    X = X.contiguous()
    res, tr = G.ggm_gram_eig_axes(X, [4, 4, 4])
    for a, (V, E) in enumerate(res):
        Vs, Es, _ = G.ggm_gram_eig(X, a, 4)
        np.testing.assert_allclose(E.cpu().numpy(), Es.cpu().numpy(), rtol=1e-9)
        d = (V.double() * Vs.double()).sum(0).abs()
        assert float((1 - d).max()) < 1e-5
    del X
    torch.cuda.empty_cache()
