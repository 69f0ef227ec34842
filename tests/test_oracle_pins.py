"""Pins of the fp64 oracle against things other than itself (brute force, closed forms,
worked values, invariants).  CPU only.  Each test names the passage it follows."""
import json
import os

import numpy as np
import pytest

import oracle as O
from synth import gen

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _gold(name):
    with open(os.path.join(GOLD, name)) as f:
        return json.load(f)


# ----------------------------------------------------------------- grid / sb-trace

def test_sbtrace_golden_examples():
    """S:233-235 worked values for the Thm 2 trace term."""
    for case in _gold("sbtrace_two_axis.json")["cases"]:
        g = O.marginals(case["lams"])
        for gl, want in zip(g, case["marginals"]):
            np.testing.assert_allclose(gl, want, rtol=1e-15)


@pytest.mark.parametrize("ks", [(2, 2), (2, 3, 2), (3, 1, 4)])
def test_marginals_equal_dense_sbtrace_of_inverse(ks):
    """Brute force: diag of tr^{k<l}_{k>l}[(⊕Λ)^-1] from a dense Kronecker sum."""
    rng = np.random.default_rng(sum(ks))
    lams = [rng.uniform(0.2, 2.0, k) for k in ks]
    inv = np.linalg.inv(O.kron_sum([np.diag(l) for l in lams]))
    g = O.marginals(lams)
    for l, k in enumerate(ks):
        a = int(np.prod(ks[:l])) if l else 1
        b = int(np.prod(ks[l + 1:])) if l + 1 < len(ks) else 1
        tr = O.sb_trace(inv, a, b, k)
        np.testing.assert_allclose(np.diag(tr), g[l], rtol=1e-12)
        np.testing.assert_allclose(tr - np.diag(np.diag(tr)), 0, atol=1e-13)


def test_sbtrace_extraction_with_eigenvectors():
    """Thm 1 proof: tr^{d<l}_{d>l}[(⊕ V Λ V^T)^-1] = V_l diag(g_l) V_l^T."""
    rng = np.random.default_rng(7)
    ds = (3, 4, 2)
    Vs = [np.linalg.qr(rng.standard_normal((d, d)))[0] for d in ds]
    lams = [rng.uniform(0.3, 1.5, d) for d in ds]
    psis = [V @ np.diag(l) @ V.T for V, l in zip(Vs, lams)]
    inv = np.linalg.inv(O.kron_sum(psis))
    g = O.marginals(lams)
    for l, d in enumerate(ds):
        a = int(np.prod(ds[:l])) if l else 1
        b = int(np.prod(ds[l + 1:])) if l + 1 < len(ds) else 1
        np.testing.assert_allclose(O.sb_trace(inv, a, b, d), Vs[l] @ np.diag(g[l]) @ Vs[l].T,
                                   atol=1e-12)


# ----------------------------------------------------------------- NLL / gradient

def test_nll_closed_form_single():
    c = _gold("closed_forms.json")["nll_single"]
    assert O.nll(c["E"], c["lams"]) == pytest.approx(c["nll"], abs=1e-15)


def test_nll_equals_dense_matrix_form():
    """k-space NLL equals the matrix NLL for full-rank factors."""
    x = gen.small_tensor(11, (4, 3, 3))
    Ss = [O.gram(x, l) for l in range(3)]
    Vs, Es = zip(*[O.gram_eig_eigh(x, l, x.shape[l]) for l in range(3)])
    rng = np.random.default_rng(3)
    lams = [rng.uniform(0.5, 2.0, x.shape[l]) for l in range(3)]
    psis = [V @ np.diag(lm) @ V.T for V, lm in zip(Vs, lams)]
    assert O.nll(Es, lams) == pytest.approx(O.dense_nll(Ss, psis), rel=1e-12)


def test_vec_quadratic_form_matches_gram_traces():
    """Unfolding convention: vec^T(⊕Ψ)vec = Σ_l tr[S_l Ψ_l]."""
    x = gen.small_tensor(5, (3, 4, 2)).astype(np.float64)
    rng = np.random.default_rng(0)
    psis = []
    for d in x.shape:
        a = rng.standard_normal((d, d))
        psis.append(a + a.T)
    vec = x.reshape(-1)
    lhs = vec @ O.kron_sum(psis) @ vec
    rhs = sum(np.trace(O.gram(x, l) @ p) for l, p in enumerate(psis))
    assert lhs == pytest.approx(rhs, rel=1e-12)


def test_gradient_matches_finite_differences():
    """Thm 2 vs central differences of the NLL."""
    rng = np.random.default_rng(1)
    E = [rng.uniform(1, 3, 3), rng.uniform(1, 3, 4)]
    lams = [rng.uniform(0.5, 1.0, 3), rng.uniform(0.5, 1.0, 4)]
    g = O.gradient(E, lams)
    h = 1e-6
    for l in range(2):
        for i in range(len(lams[l])):
            lp = [v.copy() for v in lams]
            lm = [v.copy() for v in lams]
            lp[l][i] += h
            lm[l][i] -= h
            fd = (O.nll(E, lp) - O.nll(E, lm)) / (2 * h)
            assert g[l][i] == pytest.approx(fd, rel=1e-6, abs=1e-9)


def test_nll_convex_along_segments():
    """Lemma 4."""
    rng = np.random.default_rng(2)
    E = [rng.uniform(1, 3, 3), rng.uniform(1, 3, 2), rng.uniform(1, 2, 2)]
    for _ in range(20):
        a = [rng.uniform(0.1, 2, len(e)) for e in E]
        b = [rng.uniform(0.1, 2, len(e)) for e in E]
        mid = [(u + v) / 2 for u, v in zip(a, b)]
        assert O.nll(E, mid) <= 0.5 * O.nll(E, a) + 0.5 * O.nll(E, b) + 1e-12


# ----------------------------------------------------------------- solve

def test_single_axis_closed_form():
    """One axis: λ = 1/E is stationary."""
    E = [np.array([4.0, 2.0, 0.5])]
    lams, info = O.solve_eigvals(E, gauge=1)
    np.testing.assert_allclose(lams[0], 1.0 / E[0], rtol=1e-15)
    assert info["iterations"] == 0
    assert max(abs(v) for v in O.gradient(E, [1.0 / E[0]])[0]) == 0.0


@pytest.mark.parametrize("ks,T", [((4, 3, 5), 7.0), ((40, 30, 20), 123.0), ((6, 9), 2.5)])
def test_isotropic_closed_form(ks, T):
    """E_l = (T/k_l)·1  ⇒  every grid sum equals Πk/T (derived from P:667)."""
    E = [np.full(k, T / k) for k in ks]
    lams, info = O.solve_eigvals(E)
    s = O.grid_sums(lams)
    np.testing.assert_allclose(s, np.prod(ks) / T, rtol=1e-12)


def test_lemma3_stationarity_dense_full_rank():
    """At the MLE, S_l = tr^{d<l}_{d>l}[(⊕Ψ)^-1] (Lemma 3), brute force."""
    x = gen.small_tensor(21, (4, 3, 3))
    Es, Vs = [], []
    for l in range(3):
        V, E = O.gram_eig(x, l, x.shape[l])
        Vs.append(V)
        Es.append(E)
    lams, info = O.solve_eigvals(Es, tol=1e-13)
    assert info["stationarity"] < 1e-12
    psis = [V @ np.diag(lm) @ V.T for V, lm in zip(Vs, lams)]
    inv = np.linalg.inv(O.kron_sum(psis))
    ds = x.shape
    for l in range(3):
        a = int(np.prod(ds[:l])) if l else 1
        b = int(np.prod(ds[l + 1:])) if l + 1 < 3 else 1
        S = O.gram(x, l)
        np.testing.assert_allclose(O.sb_trace(inv, a, b, ds[l]), S, atol=1e-10 * np.abs(S).max())


def test_lemma3_restricted_rank_deficient_matrix():
    """Rank-deficient 8x6 matrix, k=(6,6): on the rank-k subspace the restricted inverse
    (V0⊗V1)(⊕Λ)^-1(V0⊗V1)^T satisfies Lemma 3 (pseudo-inverse form)."""
    x = gen.small_tensor(31, (8, 6)).astype(np.float64)
    Vs, Es = zip(*[O.gram_eig(x, l, 6) for l in range(2)])
    lams, info = O.solve_eigvals(Es, tol=1e-13)
    W = np.kron(Vs[0], Vs[1])
    M = W @ np.diag(1.0 / O.grid_sums(lams).reshape(-1)) @ W.T
    np.testing.assert_allclose(O.sb_trace(M, 1, 6, 8), O.gram(x, 0), atol=1e-10 * np.abs(O.gram(x, 0)).max())
    np.testing.assert_allclose(O.sb_trace(M, 8, 1, 6), O.gram(x, 1), atol=1e-10 * np.abs(O.gram(x, 1)).max())


def test_paper_algorithm1_reaches_same_grid():
    """Algorithm 1 (readings Q1-Q3) converges to the Newton MLE's grid."""
    rng = np.random.default_rng(4)
    E = [rng.uniform(1.0, 2.0, 3), None]
    E[1] = rng.uniform(1.0, 2.0, 2)
    E[1] *= E[0].sum() / E[1].sum()          # equal traces (reading T)
    ln, _ = O.solve_eigvals(E, tol=1e-13)
    lg, info = O.paper_gd_solve(E, tol=1e-8)
    assert info["stationarity"] <= 1e-8
    np.testing.assert_allclose(O.grid_sums(lg), O.grid_sums(ln), rtol=1e-6)


def test_gauge_invariance_and_psd():
    """Gauge 0 leaves the grid unchanged and is min-balanced, PSD."""
    rng = np.random.default_rng(5)
    lams = [rng.uniform(-1, 3, 4), rng.uniform(2, 5, 3), rng.uniform(1, 2, 2)]
    can = O.canonical_gauge(lams)
    np.testing.assert_allclose(O.grid_sums(can), O.grid_sums(lams), rtol=1e-14)
    mins = [c.min() for c in can]
    np.testing.assert_allclose(mins, mins[0], rtol=1e-14)
    shifted = [lams[0] + 0.7, lams[1] - 0.2, lams[2] - 0.5]
    for a, b in zip(O.canonical_gauge(shifted), can):
        np.testing.assert_allclose(a, b, rtol=1e-12, atol=1e-12)
    t1, lt1 = O.identifiable(lams)
    t2, lt2 = O.identifiable(shifted)
    assert t1 == pytest.approx(t2, rel=1e-14)
    for a, b in zip(lt1, lt2):
        np.testing.assert_allclose(a, b, atol=1e-14)


def test_symmetric_matrix_axes_equal_and_bound():
    """E_1 = E_2 ⇒ λ_1 = λ_2; Lemma 6 bound λ_li <= K_{\\l}/E_li (reading Q6)."""
    x = gen.small_tensor(41, (30, 20))
    V0, E0 = O.gram_eig(x, 0, 20)
    V1, E1 = O.gram_eig(x, 1, 20)
    np.testing.assert_allclose(E0, E1, rtol=1e-12)
    lams, info = O.solve_eigvals([E0, E0])
    np.testing.assert_allclose(lams[0], lams[1], rtol=1e-12)
    for l in range(2):
        assert np.all(lams[l] <= 20.0 / E0 * (1 + 1e-9))
        assert np.all(lams[l] > 0)


# ----------------------------------------------------------------- Gram spectrum

@pytest.mark.parametrize("shape", [(7, 5), (5, 7), (4, 3, 5)])
def test_gram_eig_two_routes(shape):
    """SVD route (Alg. 1 lines 3-4) vs eigh of the explicit S_l; tr S_l = ||X||^2."""
    x = gen.small_tensor(sum(shape), shape)
    fro = float(np.sum(x.astype(np.float64) ** 2))
    for l in range(len(shape)):
        k = min(shape[l], int(np.prod(shape)) // shape[l])
        V1, E1 = O.gram_eig(x, l, k)
        V2, E2 = O.gram_eig_eigh(x, l, k)
        np.testing.assert_allclose(E1, E2, rtol=1e-10)
        sv = np.linalg.svd(V1.T @ V2, compute_uv=False)
        assert sv.min() > 1 - 1e-10
        assert np.trace(O.gram(x, l)) == pytest.approx(fro, rel=1e-12)
        np.testing.assert_allclose(V1.T @ V1, np.eye(k), atol=1e-12)


def test_gram_eig_rank_error():
    x = gen.small_tensor(3, (6, 3))
    with pytest.raises(O.RankError):
        O.gram_eig(x, 0, 4)     # rank S_0 <= 3


# ----------------------------------------------------------------- sparsification

def _brute_topt(P, t):
    n = P.shape[0]
    out = []
    for i in range(n):
        cand = sorted([(-abs(P[i, j]), j) for j in range(n) if j != i])
        sel = sorted(j for _, j in cand[:min(t, n - 1)])
        out.append(sel)
    return out


@pytest.mark.parametrize("n,k,t", [(37, 5, 4), (50, 50, 10), (9, 3, 20), (2, 1, 5)])
def test_top_t_vs_dense_bruteforce(n, k, t):
    """Dense V diag(λ) V^T + exhaustive sort by (−|ψ|, j) (Q8, Q9)."""
    V, lam = gen.small_factor(n * 7 + k, n, k)
    P = V.astype(np.float64) @ np.diag(lam) @ V.astype(np.float64).T
    ptr, col, val = O.sparse_precision(V, lam, 0, n, mode=0, t=t)
    want = _brute_topt(P, t)
    for i in range(n):
        c = col[ptr[i]:ptr[i + 1]]
        assert list(c) == want[i]
        np.testing.assert_allclose(val[ptr[i]:ptr[i + 1]], P[i, c], rtol=1e-13)


def test_threshold_vs_dense():
    V, lam = gen.small_factor(99, 40, 6)
    P = V.astype(np.float64) @ np.diag(lam) @ V.astype(np.float64).T
    tau = float(np.quantile(np.abs(P[~np.eye(40, dtype=bool)]), 0.9))
    ptr, col, val = O.sparse_precision(V, lam, 0, 40, mode=1, tau=tau)
    for i in range(40):
        want = [j for j in range(40) if j != i and abs(P[i, j]) > tau]
        assert list(col[ptr[i]:ptr[i + 1]]) == want


def test_rank1_closed_form_and_ties():
    """v=(1,1,0)/√2, λ=2 ⇒ ψ_01 = 1; identity factors ⇒ all-tie case picks the
    t smallest j ≠ i (Q9)."""
    c = _gold("closed_forms.json")["rank1"]
    V = np.array(c["v"]).reshape(3, 1)
    ptr, col, val = O.sparse_precision(V, np.array([c["lam"]]), 0, 3, mode=0, t=1)
    assert col[0] == 1 and val[0] == pytest.approx(c["psi_01"], rel=1e-15)
    V = np.eye(10)[:, :3]
    ptr, col, val = O.sparse_precision(V, np.ones(3), 0, 10, mode=0, t=4)
    for i in range(10):
        want = [j for j in range(10) if j != i][:4]
        assert list(col[ptr[i]:ptr[i + 1]]) == want
        assert np.all(val[ptr[i]:ptr[i + 1]] == 0)


def test_rank1_large_n_topt_is_top_of_v():
    """Rank 1 at any n: row i's set = top-t of |v_j|, j ≠ i (closed form)."""
    rng = np.random.default_rng(8)
    n = 5000
    v = rng.standard_normal(n)
    v /= np.linalg.norm(v)
    rows = [0, 17, 4999]
    ptr, col, val = O.sparse_precision(v.reshape(n, 1), np.array([3.0]), 0, 0, rows=rows, t=10)
    for r, i in enumerate(rows):
        a = np.abs(v).copy()
        a[i] = -1
        want = sorted(np.argsort(-a, kind="stable")[:10])
        assert list(col[ptr[r]:ptr[r + 1]]) == want


# ------------------------------------------------------------------ whole-graph edge rules
def test_overall_edges_brute_force_and_closed_forms():
    """overall_edges against brute force over all pairs, and closed forms:
    rank 1 (psi_ij = lam v_i v_j): the overall top-N pairs are the pairs of the largest |v|;
    with down-weighting w_i = |v_i| (sum_k|v_k| - |v_i|) ... checked by brute force."""
    import itertools
    rng = np.random.default_rng(4)
    n, k = 23, 4
    V = np.linalg.qr(rng.standard_normal((n, k)))[0]
    lam = rng.lognormal(0, 1, k)
    P = (V * lam) @ V.T
    for dw in (False, True):
        A = np.abs(P)
        np.fill_diagonal(A, 0)
        w = A.sum(1)
        pairs = []
        for i, j in itertools.combinations(range(n), 2):
            s = A[i, j] / np.sqrt(w[i] * w[j]) if dw else A[i, j]
            pairs.append((-s, i, j))
        pairs.sort()
        for N in (1, 7, 40):
            want = sorted((i, j) for _, i, j in pairs[:N])
            ii, jj, vv = O.overall_edges(V, lam, N, downweight=dw)
            assert list(zip(ii.tolist(), jj.tolist())) == want
            np.testing.assert_allclose(vv, P[ii, jj])
    # rank 1 closed form (psi_ij = lam v_i v_j): with a1, a2, a3 the indices of the three
    # largest |v|, the two largest pairs are {a1, a2} and {a1, a3}
    v = rng.standard_normal(30)
    v /= np.linalg.norm(v)
    ii, jj, _ = O.overall_edges(v.reshape(-1, 1), [2.0], 2)
    a1, a2, a3 = np.argsort(-np.abs(v))[:3].tolist()
    assert set(zip(ii.tolist(), jj.tolist())) == {tuple(sorted((a1, a2))), tuple(sorted((a1, a3)))}


def test_overall_min_edges_and_symmetric_csr():
    rng = np.random.default_rng(5)
    n, k = 40, 5
    V = np.linalg.qr(rng.standard_normal((n, k)))[0]
    lam = rng.lognormal(0, 1, k)
    ii, jj, vv = O.overall_edges(V, lam, 5, downweight=True, min_edges=2)
    deg = np.bincount(np.concatenate([ii, jj]), minlength=n)
    assert deg.min() >= 2                         # every vertex keeps >= 2 edges
    rp, c, v = O.edges_to_symmetric_csr(n, ii, jj, vv)
    assert rp[-1] == 2 * len(ii)
    P = (V * lam) @ V.T
    for r in range(n):
        cc = c[rp[r]:rp[r + 1]]
        assert np.all(np.diff(cc) > 0) and r not in cc
        np.testing.assert_allclose(v[rp[r]:rp[r + 1]], P[r, cc])


def test_overall_zero_psi_is_no_edge():
    """Q17: exactly-zero psi_ij (block-diagonal Psi) never becomes an edge, even when fewer
    than N nonzero pairs exist; min-edges skip zero entries too."""
    V = np.zeros((6, 2))
    V[:3, 0] = [1.0, 2.0, 3.0]     # block {0,1,2}
    V[3:, 1] = [1.0, -1.0, 0.0]    # block {3,4,5}; vertex 5 isolated
    ii, jj, vv = O.overall_edges(V, [1.0, 1.0], 15, min_edges=3)
    got = set(zip(ii.tolist(), jj.tolist()))
    assert got == {(0, 1), (0, 2), (1, 2), (3, 4)}
    assert np.allclose(vv, [2.0, 3.0, 6.0, -1.0])


# ---------------------------------------------------------------- multi-modal (shared axes)

def _two_matrices(seed=3):
    """Modality 0 = X1 (axes 0, 1), modality 1 = X2 stored as (axis 2, axis 1): axis 1 is
    shared.  Full rank on every axis."""
    rng = np.random.default_rng(seed)
    X1 = rng.standard_normal((3, 4))
    X2 = rng.standard_normal((3, 4))
    return [X1, X2], [[0, 1], [2, 1]]


def test_gram_eig_multi_concatenation_vs_summed_grams():
    """Alg. 1 line 2: SVD of [mat(D^1) mat(D^2)] = eigh of Σ_γ S^γ_l."""
    T, mods = _two_matrices()
    V, E = O.gram_eig_multi(T, mods, 1, 4)
    S = O.gram(T[0], 1) + O.gram(T[1], 1)
    ev = np.sort(np.linalg.eigvalsh(S))[::-1]
    assert np.allclose(E, ev, rtol=1e-12)
    assert np.allclose(V @ np.diag(E) @ V.T, S, atol=1e-10)
    with pytest.raises(ValueError):
        O.gram_eig_multi(T, mods, 5, 1)


def test_multi_single_modality_reduces_to_single():
    rng = np.random.default_rng(5)
    E = [np.sort(rng.uniform(1, 4, k))[::-1] for k in (4, 3, 5)]
    E = [e * 12.0 / e.sum() for e in E]          # equal traces: interior MLE (reading T)
    a, ia = O.solve_eigvals(E)
    b, ib = O.solve_eigvals_multi(E, [[0, 1, 2]])
    assert ib["stationarity"] < 1e-10
    for x, y in zip(a, b):
        assert np.allclose(x, y, rtol=1e-9, atol=1e-12)
    assert np.allclose(O.grid_sums(a), O.grid_sums_multi(b, [[0, 1, 2]])[0], rtol=1e-10)


def test_multi_disjoint_modalities_are_independent():
    rng = np.random.default_rng(6)
    E = [np.sort(rng.uniform(1, 3, k))[::-1] for k in (3, 4, 2, 5)]
    E[0] *= E[1].sum() / E[0].sum()
    E[2] *= E[3].sum() / E[2].sum()
    m, _ = O.solve_eigvals_multi(E, [[0, 1], [2, 3]])
    a, _ = O.solve_eigvals(E[:2])
    b, _ = O.solve_eigvals(E[2:])
    assert np.allclose(O.grid_sums(m[:2]), O.grid_sums(a), rtol=1e-10)
    assert np.allclose(O.grid_sums(m[2:]), O.grid_sums(b), rtol=1e-10)


def test_multi_dense_nll_and_stationarity():
    """Shared axis: nll_multi = Σ_γ of the dense matrix-form NLL of each modality,
    and at the solution the dense full-rank stationarity Σ_{γ∋l} sb-trace[(⊕_γ Ψ)^-1] = S_l
    (Thm 2 with Σ_γ) holds."""
    T, mods = _two_matrices()
    d = {0: 3, 1: 4, 2: 3}
    Sg = [[O.gram(T[g], p) for p in range(2)] for g in range(2)]
    S = {0: Sg[0][0], 1: Sg[0][1] + Sg[1][1], 2: Sg[1][0]}
    VE = {a: np.linalg.eigh(S[a]) for a in range(3)}
    V = {a: VE[a][1][:, ::-1] for a in range(3)}
    E = [VE[a][0][::-1].copy() for a in range(3)]
    rng = np.random.default_rng(9)
    lam = [rng.uniform(0.5, 2.0, d[a]) for a in range(3)]
    psi = {a: V[a] @ np.diag(lam[a]) @ V[a].T for a in range(3)}
    dense = sum(O.dense_nll([Sg[g][p] for p in range(2)], [psi[a] for a in mods[g]])
                for g in range(2))
    assert abs(O.nll_multi(E, lam, mods) - dense) < 1e-9 * max(1.0, abs(dense))
    sol, info = O.solve_eigvals_multi(E, mods, tol=1e-13)
    assert info["stationarity"] < 1e-11
    psi = {a: V[a] @ np.diag(sol[a]) @ V[a].T for a in range(3)}
    acc = {a: np.zeros((d[a], d[a])) for a in range(3)}
    for g, mod in enumerate(mods):
        inv = np.linalg.inv(O.kron_sum([psi[a] for a in mod]))
        dims = [d[a] for a in mod]
        for p, a in enumerate(mod):
            pre = int(np.prod(dims[:p])) if p else 1
            post = int(np.prod(dims[p + 1:])) if p + 1 < len(dims) else 1
            acc[a] += O.sb_trace(inv, pre, post, d[a])
    for a in range(3):
        assert np.allclose(acc[a], S[a], atol=1e-8 * np.abs(S[a]).max())


def test_multi_gauge_space_and_canonical_invariance():
    mods = [[0, 1], [2, 1]]
    N = O.gauge_space_multi(3, mods)
    assert N.shape == (3, 1)
    assert np.allclose(N[:, 0] / N[0, 0], [1.0, -1.0, 1.0])
    rng = np.random.default_rng(2)
    lam = [rng.uniform(1, 2, k) for k in (3, 4, 3)]
    c = 0.37 * N[:, 0]
    sh = [l + c[a] for a, l in enumerate(lam)]
    for s1, s2 in zip(O.grid_sums_multi(lam, mods), O.grid_sums_multi(sh, mods)):
        assert np.allclose(s1, s2, rtol=1e-13)
    for x, y in zip(O.canonical_gauge_multi(lam, mods), O.canonical_gauge_multi(sh, mods)):
        assert np.allclose(x, y, rtol=1e-12)
    single = O.canonical_gauge_multi(lam, [[0, 1, 2]])
    for x, y in zip(single, O.canonical_gauge(lam)):
        assert np.allclose(x, y, rtol=1e-12)


# ---------------------------------------------------------------- nonparanormal (COCA)

def test_nonparanormal_paper_example():
    """ranks, Φ^-1(r/6) values and the sparse part + z 1^T, to the paper's
    printed 2 decimals."""
    with open(os.path.join(GOLD, "nonparanormal.json")) as f:
        g = json.load(f)
    X = np.array(g["data"], dtype=np.float64)
    from scipy.stats import rankdata
    assert np.array_equal(rankdata(X, method="min", axis=1), np.array(g["ranks"]))
    T = O.nonparanormal(X, 0)
    assert np.allclose(np.round(T, 2), g["normal"], atol=1e-12)
    S, z = O.nonparanormal_sparse_split(X, 0)
    assert np.allclose(np.round(S, 2), g["sparse_part"], atol=0.011)
    assert np.allclose(np.round(z, 2), g["z"], atol=1e-12)
    assert np.array_equal(S == 0, X == 0)
    assert np.allclose(S + z[:, None], T, atol=1e-15)


def test_nonparanormal_invariances():
    """Copula invariance: strictly increasing maps of the data leave the transform unchanged;
    with no ties every row holds exactly the values Φ^-1(r/(n+1)), r = 1..n."""
    from scipy.special import ndtri
    rng = np.random.default_rng(4)
    X = rng.standard_normal((7, 5, 6))
    for ax in range(3):
        a = O.nonparanormal(X, ax)
        b = O.nonparanormal(np.exp(3.0 * X) + 2.0, ax)
        assert np.allclose(a, b, atol=1e-14)
        n = a.shape[1]
        want = ndtri(np.arange(1, n + 1) / (n + 1.0))
        assert np.allclose(np.sort(a, axis=1), np.broadcast_to(want, a.shape), atol=1e-14)
    V, E = O.gram_eig_nonparanormal(X, 1, 5)
    T = O.nonparanormal(X, 1)
    assert np.allclose(np.sort(np.linalg.eigvalsh(T @ T.T))[::-1][:5], E, rtol=1e-12)


def test_overall_spec_worked_examples():
    """SPEC S:316-318 (recompose_threshold examples): Λ = 0 gives the empty graph; the rank-1
    spectrum v = (1, 1, 0)/√2, λ = 2 on d = 3 has the single off-diagonal ψ_12 = 1 and
    top_overall(1) yields the edge (1, 2, 1.0) (0-based (0, 1))."""
    v = np.array([[1.0], [1.0], [0.0]]) / np.sqrt(2.0)
    ii, jj, vv = O.overall_edges(v, [2.0], 1)
    assert (ii.tolist(), jj.tolist()) == ([0], [1]) and np.allclose(vv, [1.0], atol=1e-15)
    V = np.random.default_rng(1).standard_normal((6, 3))
    ii, jj, vv = O.overall_edges(V, [0.0, 0.0, 0.0], 5, min_edges=2)
    assert len(ii) == 0
