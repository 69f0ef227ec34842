"""Pins of the oracle's eigenvalue MLE on the paper's domain Λ_l >= ε (Lemma 6 P:657-690,
P:1026) when the truncated traces disagree (reading T), and of the gauge-1
option (Algorithm 1's gauge).  CPU only; each pin is a closed form derived by
hand, an independent optimiser, an independent fixed-point algorithm or an invariant."""
import numpy as np
import pytest
from scipy.optimize import minimize

import oracle as O
from synth import gen


def _eps(E, eps_scale=1e-10):
    return eps_scale * max(float(np.max(1.0 / np.asarray(e))) for e in E)


# ------------------------------------------------------- closed forms, k = (2, 1)
# E_1 = (e1, e2), e1 >= e2; E_2 = (f).  Grid s_i = λ_1i + μ.  KKT on the box (hand-derived):
#  (a) f > e1 + e2 (axis 2 has the larger trace): μ = ε, λ_1i = 1/e_i − ε;
#  (b) f < e1 + e2 and f >= 2 e2: λ_11 = ε, μ = 1/(f − e2) − ε, λ_12 = 1/e2 − μ;
#  (c) f < 2 e2 (hence f < e1 + e2): λ_1 = (ε, ε), μ = 2/f − ε.
@pytest.mark.parametrize("e1,e2,f,case", [(3.0, 2.0, 7.0, "a"), (2.0, 1.0, 2.5, "b"),
                                          (5.0, 1.0, 2.0, "b"), (3.0, 2.0, 1.5, "c"),
                                          (1.5, 1.0, 1.0, "c")])
def test_barrier_closed_forms_k21(e1, e2, f, case):
    E = [np.array([e1, e2]), np.array([f])]
    eps = _eps(E)
    lams, info = O.solve_eigvals(E, gauge=0)
    if case == "a":
        want = [1.0 / np.array([e1, e2]) - eps, np.array([eps])]
    elif case == "b":
        mu = 1.0 / (f - e2) - eps
        want = [np.array([eps, 1.0 / e2 - mu]), np.array([mu])]
    else:
        want = [np.array([eps, eps]), np.array([2.0 / f - eps])]
    for a, b in zip(lams, want):
        np.testing.assert_allclose(a, b, rtol=1e-10, atol=1e-3 * eps)
    assert info["floor_active"] and info["regime"] == "barrier"
    assert info["stationarity"] <= 1e-12


def _random_truncated(seed):
    """Top-k spectra of a small tensor's unfoldings with k_l < d_l: traces differ."""
    x = gen.small_tensor(seed, (9, 7, 6))
    ks = (4, 3, 5)
    return [O.gram_eig(x, l, k)[1] for l, k in enumerate(ks)]


def _kkt_ok(E, lams, eps, tol):
    g = O.marginals(lams)
    emax = max(e.max() for e in E)
    for e, gl, l in zip(E, g, lams):
        on = l <= eps * (1 + 1e-9)
        assert np.all(l >= eps * (1 - 1e-12))
        assert np.all(np.abs(e - gl)[~on] <= tol * emax)
        assert np.all((e - gl)[on] >= -tol * emax)     # multipliers ½(E − g) >= 0


@pytest.mark.parametrize("seed", [1, 2, 3])
def test_barrier_kkt_truncated_tensor(seed):
    """KKT conditions of min NLL s.t. λ >= ε (Lemma 6's domain): stationary off the floor,
    non-negative multipliers on it; at least one floor coordinate on every axis but the
    minimum-trace one (the NLL decreases along the gauge otherwise)."""
    E = _random_truncated(seed)
    tr = [e.sum() for e in E]
    assert O.trace_inconsistency(E) > 1e-3
    lams, info = O.solve_eigvals(E)
    eps = info["eps"]
    _kkt_ok(E, lams, eps, 1e-11)
    lo = int(np.argmin(tr))
    for a, l in enumerate(lams):
        if a != lo:
            assert np.min(l) <= eps * (1 + 1e-9)


@pytest.mark.parametrize("seed", [1, 2, 3])
def test_barrier_matches_lbfgsb(seed):
    """An independent route: SciPy's bound-constrained L-BFGS-B on the NLL (analytic
    gradient ½(E − g), Thm 2) reaches the same grid."""
    E = _random_truncated(seed)
    ks = [len(e) for e in E]
    off = np.cumsum([0] + ks)
    eps = _eps(E)
    split = lambda v: [v[off[a]:off[a + 1]] for a in range(len(ks))]
    ev = np.concatenate(E)
    scale = float(ev.max())

    def fg(v):
        lams = split(v)
        return O.nll(E, lams) / scale, np.concatenate(O.gradient(E, lams)) / scale

    x0 = np.concatenate([1.0 / e for e in E])
    r = minimize(fg, x0, jac=True, method="L-BFGS-B", bounds=[(eps, None)] * len(x0),
                 options=dict(maxiter=20000, ftol=1e-16, gtol=1e-12, maxcor=50))
    lams, _ = O.solve_eigvals(E)
    s_o = O.grid_sums(lams)
    s_b = O.grid_sums(split(r.x))
    np.testing.assert_allclose(s_b, s_o, rtol=2e-4)
    assert O.nll(E, lams) <= O.nll(E, split(r.x)) + 1e-12 * abs(O.nll(E, lams))


@pytest.mark.parametrize("seed", [1, 2])
def test_barrier_matches_clamped_fixed_point(seed):
    """A second independent algorithm: the majorise-minimise step λ ← max(ε, λ g/E) (a
    separable majoriser of the NLL, minimised on the box coordinate-wise) converges to the
    same λ (the box MLE is unique here: one minimum-trace axis)."""
    E = _random_truncated(seed)
    eps = _eps(E)
    lams = [1.0 / e for e in E]
    for _ in range(200000):
        g = O.marginals(lams)
        lams = [np.maximum(eps, l * gl / e) for l, gl, e in zip(lams, g, E)]
        if O.kkt_residual(E, lams, eps * (1 + 1e-9)) < 1e-13:
            break
    lo, _ = O.solve_eigvals(E)
    for a, b in zip(lams, lo):
        np.testing.assert_allclose(a, b, rtol=1e-8, atol=1e-6 * eps)


def test_matrix_unequal_ranks():
    """A matrix with k0 != k1 (traces of the two truncated spectra differ): barrier regime,
    the larger-trace axis carries floor coordinates; a consistent matrix stays interior."""
    x = gen.small_tensor(41, (30, 20))
    E0 = O.gram_eig(x, 0, 12)[1]
    E1 = O.gram_eig(x, 1, 6)[1]
    lams, info = O.solve_eigvals([E0, E1])
    assert info["regime"] == "barrier" and info["floor_active"]
    assert np.min(lams[0]) <= info["eps"] * (1 + 1e-9)
    _kkt_ok([E0, E1], lams, info["eps"], 1e-11)
    lams2, info2 = O.solve_eigvals([E0, O.gram_eig(x, 1, 12)[1]])
    assert info2["regime"] == "interior" and not info2["floor_active"]


def test_interior_projection_is_rounding_level():
    """Traces equal up to rounding (full-rank tensor: tr S_l = ||X||^2 for every l):
    the interior regime, E_eff = P_G⊥ E differs from E by rounding only."""
    x = gen.small_tensor(21, (5, 4, 3))
    E = [O.gram_eig(x, l, x.shape[l])[1] for l in range(3)]
    assert O.trace_inconsistency(E) < 1e-12
    Ee = O.project_spectrum(E)
    for a, b in zip(E, Ee):
        np.testing.assert_allclose(a, b, rtol=1e-12)
    lams, info = O.solve_eigvals(E)
    assert info["regime"] == "interior" and not info["floor_active"]


# ------------------------------------------------------- gauge 1 (Algorithm 1's gauge)

def test_gauge1_is_orthogonal_and_matches_algorithm1():
    """Gauge 1: λ − 1/E ⊥ G (Σ_i (λ_li − 1/E_li) equal across axes); Algorithm 1's gradient
    descent (paper_gd_solve, readings Q1-Q3) preserves exactly that, so it reaches the same
    λ, not only the same grid."""
    rng = np.random.default_rng(4)
    E = [rng.uniform(1.0, 2.0, 3), rng.uniform(1.0, 2.0, 2), rng.uniform(1.0, 2.0, 2)]
    E[1] *= E[0].sum() / E[1].sum()
    E[2] *= E[0].sum() / E[2].sum()
    l1, _ = O.solve_eigvals(E, tol=1e-13, gauge=1)
    d = [float(np.sum(l - 1.0 / e)) for l, e in zip(l1, E)]
    np.testing.assert_allclose(d, d[0], atol=1e-12)
    lg, info = O.paper_gd_solve(E, tol=1e-8)
    for a, b in zip(lg, l1):
        np.testing.assert_allclose(a, b, rtol=2e-5)
    l0, _ = O.solve_eigvals(E, tol=1e-13, gauge=0)
    np.testing.assert_allclose(O.grid_sums(l0), O.grid_sums(l1), rtol=1e-12)


def test_gauge1_multi_modal_reduces():
    """One modality through the multi-modal solver gives the same gauge-1 λ."""
    E = _random_truncated(7)
    E = [e * (E[0].sum() / e.sum()) for e in E]        # consistent traces
    a, _ = O.solve_eigvals(E, gauge=1)
    b, _ = O.solve_eigvals_multi(E, [[0, 1, 2]], gauge=1)
    for x, y in zip(a, b):
        np.testing.assert_allclose(x, y, rtol=1e-10)


# ------------------------------------------------------- helpers pinned directly

def test_marginals_sq2d_brute_force_and_hessian():
    """marginals_sq2d (the Newton oracle's Hessian blocks): the 1-D and 2-D marginals of
    1/s² equal explicit loops over the grid, and ½ of them is the finite-difference Jacobian
    of the gradient ½(E − g) (∂g_li/∂λ_mj = −Σ 1/s² over the grid points with j_l=i, j_m=j)."""
    rng = np.random.default_rng(3)
    lams = [rng.uniform(0.3, 2.0, k) for k in (3, 4, 2)]
    diag, pair = O.marginals_sq2d(lams)
    for a in range(3):
        for i in range(len(lams[a])):
            want = 0.0
            for j0 in range(3):
                for j1 in range(4):
                    for j2 in range(2):
                        idx = (j0, j1, j2)
                        if idx[a] != i:
                            continue
                        want += 1.0 / (lams[0][j0] + lams[1][j1] + lams[2][j2]) ** 2
            assert diag[a][i] == pytest.approx(want, rel=1e-13)
    E = [rng.uniform(1, 2, len(l)) for l in lams]
    h = 1e-6
    for (a, b), M in pair.items():
        for i in range(len(lams[a])):
            for j in range(len(lams[b])):
                lp = [l.copy() for l in lams]
                lm = [l.copy() for l in lams]
                lp[b][j] += h
                lm[b][j] -= h
                dg = (O.gradient(E, lp)[a][i] - O.gradient(E, lm)[a][i]) / (2 * h)
                assert dg == pytest.approx(0.5 * M[i, j], rel=1e-6)


def test_trace_inconsistency_closed_forms():
    """trace_inconsistency = max_l |tr E_l − mean| / mean (reading T): equal traces → 0;
    traces (6, 1.5) → mean 3.75, max deviation 2.25 → 0.6; the multi-modal form with one
    modality is the same number."""
    assert O.trace_inconsistency([np.array([1.0, 2.0]), np.array([3.0])]) == 0.0
    E = [np.array([3.0, 2.0, 1.0]), np.array([1.0, 0.5])]
    assert O.trace_inconsistency(E) == pytest.approx(0.6, rel=1e-15)
    assert O.trace_inconsistency_multi(E, [[0, 1]]) == pytest.approx(0.6, rel=1e-12)
