"""Plain, slow, fp64 NumPy oracle of the GmGM hot path (arXiv 2407.19892).

TEST INFRASTRUCTURE — not product code.  Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import or run anything in ``oracle/``.

Citations: ``P:n`` = PAPER.md line n (LaTeX source of arXiv 2407.19892),
``S:n`` = SPEC.md line n, readings Q1..Q15 / G / T / TOL = DESIGN.md §"Readings".

Pinning (tests/test_oracle_pins.py, ``-m "not gpu"``):
  matricize / gram_eig      eigh(S) vs SVD route; tr S_l = ||X||_F^2; E_1 = E_2 for
                            matrices; vec^T(⊕Ψ)vec = Σ tr[S_l Ψ_l] (brute force)
  grid_sums / marginals     dense Kronecker-sum inverse + stridewise-blockwise trace
                            (brute force); golden example S:234
  nll                       dense log-pseudodeterminant NLL on tiny inputs;
                            convexity (Lemma 4)
  gradient                  finite differences of nll; single axis closed form
  solve_eigvals             Lemma 3 on dense ⊕Ψ; isotropic closed form;
                            Alg. 1 gradient descent (paper_gd_solve) reaches the same grid
                            and, in gauge 1, the same λ
  barrier regime (reading T) hand-derived closed forms for k = (2, 1) (all three active
                            sets); KKT conditions on truncated tensors; SciPy L-BFGS-B on
                            the box and the clamped majorise-minimise iteration reach the
                            same grid / λ (tests/test_oracle_barrier.py)
  marginals_sq2d            explicit grid loops; ½ of it = finite-difference Jacobian of the
                            gradient (the Newton Hessian blocks)
  trace_inconsistency       closed forms (equal traces → 0; (6, 1.5) → 0.6), = the
                            multi-modal form for one modality
  canonical gauge          grid invariance; PSD; closed form on shifted inputs
  psi_rows / top_t / thr    dense V diag(λ) V^T + brute-force sort on tiny inputs;
                            rank-1 closed form; identity-factor all-tie case
  nonparanormal (COCA)      the paper's worked example (ranks, Φ^-1 values, sparse part
                            and z; tests/golden/nonparanormal.json);
                            invariance under strictly increasing maps; row values are
                            the Φ^-1(r/(n+1)) of a rank multiset
  *_multi (shared axes)     one modality = the single-modality functions; disjoint
                            modalities = independent solves; dense multi-modal NLL and
                            the dense stationarity Σ_γ sb-trace[(⊕_γΨ)^-1] = S_l
                            at the solution; gauge-class invariance; SVD of the
                            concatenation vs eigh of Σ_γ S^γ_l
No function here is "parity unpinned".
"""
from __future__ import annotations

import numpy as np

__all__ = [
    "RankError", "matricize", "gram", "gram_eig", "gram_eig_eigh",
    "grid_sums", "marginals", "marginals_sq2d", "nll", "gradient", "stationarity",
    "solve_eigvals", "paper_gd_solve", "canonical_gauge", "identifiable",
    "trace_inconsistency",
    "kron_sum", "sb_trace", "dense_nll",
    "psi_rows", "top_t_row", "threshold_row", "sparse_precision",
    "wald_edge", "wald_threshold", "overall_edges", "edges_to_symmetric_csr",
    "gram_eig_multi", "grid_sums_multi", "marginals_multi", "nll_multi", "gradient_multi",
    "stationarity_multi", "gauge_space_multi", "canonical_gauge_multi", "solve_eigvals_multi",
    "project_spectrum", "kkt_residual", "trace_inconsistency_multi", "gauge_space_free",
    "gauge_lift",
    "nonparanormal", "nonparanormal_sparse_split", "gram_eig_nonparanormal",
]


class RankError(ValueError):
    """k_l exceeds the attainable rank (Cor. 3)."""


# ---------------------------------------------------------------------------
# Gram spectrum — Algorithm 1 lines 1-4, Theorem 1
# ---------------------------------------------------------------------------

def matricize(x: np.ndarray, axis: int) -> np.ndarray:
    """l-matricization mat_l[D]: a d_l x d_{\\l} matrix whose row i holds every
    entry with l-index i.  First axis has the largest stride; the column order
    does not affect S_l = mat_l mat_l^T."""
    x = np.asarray(x, dtype=np.float64)
    return np.moveaxis(x, axis, 0).reshape(x.shape[axis], -1)


def gram(x: np.ndarray, axis: int) -> np.ndarray:
    """Empirical Gram matrix S_l = mat_l[D] mat_l[D]^T, fp64."""
    m = matricize(x, axis)
    return m @ m.T


def _check_rank(e: np.ndarray, k: int):
    if not (e[k - 1] > 1e-12 * e[0]):
        raise RankError(f"E_k={e[k-1]:.3e} <= 1e-12*E_1 ({e[0]:.3e}); k exceeds rank (S:140)")


def gram_eig(x: np.ndarray, axis: int, k: int):
    """Top-k left singular vectors of D_l = mat_l[D] and E = sigma^2 (Alg. 1 lines 3-4,
    P:910-911: "top k_l left singular vectors of D_l", "(top k_l singular values)^2").

    Returns V (d_l x k, fp64) and E (k, descending).  Single modality: D_l = mat_l.
    """
    m = matricize(x, axis)
    if not 1 <= k <= min(m.shape):
        raise RankError(f"k={k} not in [1, min(d_l, d_\\l)={min(m.shape)}] (S:116)")
    u, sig, _ = np.linalg.svd(m, full_matrices=False)
    e = sig ** 2
    _check_rank(e, k)
    return u[:, :k].copy(), e[:k].copy()


def gram_eig_eigh(x: np.ndarray, axis: int, k: int):
    """Independent route (pin only): eigh of the explicitly formed S_l."""
    s = gram(x, axis)
    e, v = np.linalg.eigh(s)
    order = np.argsort(-e, kind="stable")
    e, v = e[order], v[:, order]
    _check_rank(e, k)
    return v[:, :k].copy(), e[:k].copy()


# ---------------------------------------------------------------------------
# Eigenvalue grid — Theorem 2, elementwise form (Lemma 6 proof P:662-668)
# ---------------------------------------------------------------------------

def grid_sums(lams) -> np.ndarray:
    """s_j = Σ_l λ_l[j_l] on the full k-grid (the diagonal of ⊕Λ), shape (k_1..k_L);
    axis 1 outermost, matching ⊕ = Σ I_{<l} ⊗ Λ_l ⊗ I_{>l}."""
    s = np.zeros(())
    for lam in lams:
        s = np.add.outer(s, np.asarray(lam, dtype=np.float64))
    return s


def marginals(lams):
    """g_l[i] = Σ_{grid points j with j_l = i} 1/s_j — the diagonal of
    tr^{k<l}_{k>l}[(⊕Λ)^†] in Thm 2, elementwise as in P:667."""
    s = grid_sums(lams)
    if s.min() <= 0:
        raise ValueError("grid sum <= 0: outside the domain (Lemma 4, P:650)")
    r = 1.0 / s
    out = []
    for ax in range(s.ndim):
        other = tuple(a for a in range(s.ndim) if a != ax)
        out.append(r.sum(axis=other) if other else r.copy())
    return out


def marginals_sq2d(lams):
    """Second-order marginals of 1/s^2 used by the Newton oracle: returns
    (diag list: Σ_{j_l=i} 1/s^2, pair dict {(l,m): Σ_{j_l=i, j_m=j} 1/s^2})."""
    s = grid_sums(lams)
    r2 = 1.0 / (s * s)
    L = s.ndim
    diag, pair = [], {}
    for a in range(L):
        other = tuple(x for x in range(L) if x != a)
        diag.append(r2.sum(axis=other) if other else r2.copy())
    for a in range(L):
        for b in range(a + 1, L):
            other = tuple(x for x in range(L) if x not in (a, b))
            pair[(a, b)] = r2.sum(axis=other) if other else r2.copy()
    return diag, pair


def nll(E, lams) -> float:
    """NLL(λ) = ½ Σ_l e_l^T λ_l − ½ Σ_{grid} log s_j  (constants of P:262
    dropped, reading Q11)."""
    s = grid_sums(lams)
    if s.min() <= 0:
        return np.inf
    lin = sum(float(np.dot(np.asarray(e, np.float64), np.asarray(l, np.float64)))
              for e, l in zip(E, lams))
    return 0.5 * lin - 0.5 * float(np.log(s).sum())


def gradient(E, lams):
    """∂NLL/∂Λ_l = ½ (E_l − g_l)  (Theorem 2)."""
    g = marginals(lams)
    return [0.5 * (np.asarray(e, np.float64) - gl) for e, gl in zip(E, g)]


def stationarity(E, lams) -> float:
    """max_l max_i |E_li − g_li| / max E  (reading Q4)."""
    g = marginals(lams)
    emax = max(float(np.max(e)) for e in E)
    return max(float(np.max(np.abs(np.asarray(e) - gl))) for e, gl in zip(E, g)) / emax


def trace_inconsistency(E) -> float:
    """|P_G(tr E)|: the gradient component along the gauge directions G (reading T).
    Stationarity in G⊥ needs tr E_l equal across axes for a single modality."""
    tr = np.array([float(np.sum(e)) for e in E])
    return float(np.max(np.abs(tr - tr.mean())) / max(abs(tr.mean()), 1e-300))


def _gauge_projector(ks):
    """Orthogonal projector onto G⊥, G = span{(c_l 1_{k_l})_l : Σ c_l = 0} (reading G)."""
    L = len(ks)
    n = int(sum(ks))
    if L == 1:
        return np.eye(n)
    cols = []
    off = np.cumsum([0] + list(ks))
    for l in range(L - 1):
        c = np.zeros(n)
        c[off[l]:off[l + 1]] = 1.0
        c[off[L - 1]:off[L]] = -1.0
        cols.append(c)
    B = np.stack(cols, axis=1)
    Q, _ = np.linalg.qr(B)
    return np.eye(n) - Q @ Q.T


def _split(vec, ks):
    off = np.cumsum([0] + list(ks))
    return [vec[off[i]:off[i + 1]].copy() for i in range(len(ks))]


def canonical_gauge(lams):
    """Gauge 0 (reading G): λ_l ← λ_l − min λ_l + s_min / L, s_min = Σ_l min λ_l.
    Leaves every grid sum unchanged (shifts sum to 0) and makes each axis'
    minimum equal, so Ψ_l = V diag(λ_l) V^T is PSD whenever s_min > 0."""
    L = len(lams)
    smin = sum(float(np.min(l)) for l in lams)
    return [np.asarray(l, np.float64) - float(np.min(l)) + smin / L for l in lams]


def identifiable(lams):
    """Gauge-free coordinates (t, λ̃): t = Σ_l mean(λ_l), λ̃_l = λ_l − mean(λ_l)
    (k-space form of the Greenewald reparameterization; reading G)."""
    t = sum(float(np.mean(l)) for l in lams)
    return t, [np.asarray(l, np.float64) - float(np.mean(l)) for l in lams]


def solve_eigvals(E, tol: float = 1e-12, max_iter: int = 200, gauge: int = 0,
                  eps_scale: float = 1e-10, trace_tol: float = 1e-8):
    """Eigenvalue MLE: the minimizer of the convex NLL (Lemma 4) over the paper's
    domain Λ_l >= ε (Lemma 6), uniqueness of the grid (Thm 4).
    Reading T:
      * traces consistent (trace_inconsistency(E) <= trace_tol): the interior stationary
        point of the NLL with E replaced by its G⊥ projection (the gauge component of the
        linear term, non-zero only through rounding, is dropped) — projected Newton on G⊥
        (Hessian from the 1/s^2 marginals, a library least-squares solve as the primitive),
        backtracking on NLL with grid feasibility, start λ = 1/E (Alg. 1 line 5);
      * otherwise the NLL is linear and decreasing along a gauge direction and the minimum
        lies on the barrier λ >= ε = eps_scale·max(1/E): active-set Newton on the box
        (_box_mle), floor_active = True ("consistently running into this barrier ... pick a
        smaller k_l").
    gauge 0 → canonical_gauge (min-balanced), gauge 1 → (λ − 1/E) ⊥ G, the gauge Algorithm 1's
    gradient steps preserve; in the barrier regime both act only among the axes with no
    coordinate on the floor (the others have no gauge freedom left).
    Returns (lams, info dict)."""
    return _solve_mle(E, None, tol, max_iter, gauge, eps_scale, trace_tol)


def gauge_lift(ks, N: np.ndarray) -> np.ndarray:
    """Orthonormal basis, in the Σk coordinate space, of the per-axis constant shifts
    {(c_l 1_{k_l})_l : c ∈ span N} (N: axis-space basis, nax x r)."""
    off = np.cumsum([0] + list(ks))
    n = int(off[-1])
    if N.size == 0:
        return np.zeros((n, 0))
    B = np.zeros((n, N.shape[1]))
    for a in range(len(ks)):
        B[off[a]:off[a + 1], :] = N[a][None, :]
    Q, _ = np.linalg.qr(B)
    return Q


def gauge_space_free(nax: int, modalities, free_axes) -> np.ndarray:
    """Axis-space basis of G_F = {c ∈ G : c_l = 0 for l not in free_axes} (the gauge freedom
    left when the axes outside free_axes have a coordinate pinned at the floor)."""
    rows = []
    for mod in modalities:
        r = np.zeros(nax)
        r[list(mod)] = 1.0
        rows.append(r)
    for a in range(nax):
        if a not in free_axes:
            r = np.zeros(nax)
            r[a] = 1.0
            rows.append(r)
    M = np.array(rows)
    _, sv, vt = np.linalg.svd(M)
    rank = int(np.sum(sv > 1e-12 * max(sv.max(), 1.0)))
    return vt[rank:].T.copy()


def project_spectrum(E, modalities=None):
    """E_eff = P_{G⊥}(E) (reading T): the grid marginals g are always ⊥ G (every modality's
    marginals have the same sum on each of its axes), so E_eff is the part of E that an
    interior stationary point g = E_eff can match.  Equal to E when the traces agree."""
    E = [np.asarray(e, np.float64) for e in E]
    ks = [len(e) for e in E]
    if modalities is None:
        modalities = [list(range(len(E)))]
    Q = gauge_lift(ks, gauge_space_multi(len(E), modalities))
    v = np.concatenate(E)
    return _split(v - Q @ (Q.T @ v), ks)


def _hessian_multi(lams, modalities, ks):
    """∂²NLL/∂λ∂λ = ½ Σ_γ (1D marginals of 1/s² on the diagonal blocks, 2D marginals off it)."""
    off = np.cumsum([0] + list(ks))
    n = int(off[-1])
    H = np.zeros((n, n))
    for mod in modalities:
        diag, pair = marginals_sq2d([lams[a] for a in mod])
        for pa, a in enumerate(mod):
            H[off[a]:off[a + 1], off[a]:off[a + 1]] += np.diag(0.5 * diag[pa])
        for (pa, pb), m in pair.items():
            a, b = mod[pa], mod[pb]
            H[off[a]:off[a + 1], off[b]:off[b + 1]] += 0.5 * m
            H[off[b]:off[b + 1], off[a]:off[a + 1]] += 0.5 * m.T
    return H


def _interior_newton(E, modalities, tol, max_iter):
    """Projected Newton on G⊥ from λ = 1/E (every step ⊥ G, so λ − 1/E stays ⊥ G)."""
    ks = [len(e) for e in E]
    n = int(sum(ks))
    Q = gauge_lift(ks, gauge_space_multi(len(E), modalities))
    P = np.eye(n) - Q @ Q.T
    lam = np.concatenate([1.0 / e for e in E])
    f = nll_multi(E, _split(lam, ks), modalities)
    it = 0
    res = stationarity_multi(E, _split(lam, ks), modalities)
    while res > tol and it < max_iter:
        lams = _split(lam, ks)
        grad = np.concatenate(gradient_multi(E, lams, modalities))
        H = _hessian_multi(lams, modalities, ks)
        step = P @ (-np.linalg.lstsq(P @ H @ P, P @ grad, rcond=None)[0])
        alpha = 1.0
        while True:
            cand = lam + alpha * step
            fc = nll_multi(E, _split(cand, ks), modalities)
            if np.isfinite(fc) and fc <= f + 1e-4 * alpha * float(grad @ step):
                break
            alpha *= 0.5
            if alpha < 1e-12:
                cand, fc = lam, f
                break
        if np.array_equal(cand, lam):
            break
        lam, f = cand, fc
        it += 1
        res = stationarity_multi(E, _split(lam, ks), modalities)
    return _split(lam, ks), it


def kkt_residual(E, lams, eps: float, modalities=None) -> float:
    """Stationarity on the box λ >= ε: max over coordinates of |E − g| off the floor and of
    max(0, g − E) on it (a floor coordinate needs ∂NLL/∂λ = ½(E − g) >= 0), / max E."""
    if modalities is None:
        modalities = [list(range(len(E)))]
    g = marginals_multi(lams, modalities)
    emax = max(float(np.max(e)) for e in E)
    r = 0.0
    for e, gl, l in zip(E, g, lams):
        e = np.asarray(e, np.float64)
        on = np.asarray(l) <= eps
        r = max(r, float(np.max(np.abs(e - gl)[~on], initial=0.0)),
                float(np.max(np.maximum(0.0, gl - e)[on], initial=0.0)))
    return r / emax


def _box_mle(E, modalities, eps, tol, max_iter):
    """argmin NLL over the box λ >= ε (Lemma 6's domain) by a primal active-set method:
      * gauge directions left free (axes with no floor coordinate) along which the NLL is
        linear and decreasing are followed to the first coordinate that reaches ε, which
        joins the active set (the NLL is unbounded below along them otherwise);
      * else a Newton step on the free coordinates (projected off the remaining gauge
        directions), cut at the first bound reached, Armijo backtracking on the NLL;
      * when the free coordinates are stationary, an active coordinate whose multiplier
        ½(E − g) is negative is released (the most negative first); none left → KKT point.
    Returns (lams, iterations, active mask)."""
    ks = [len(e) for e in E]
    nax = len(E)
    off = np.cumsum([0] + ks)
    ev = np.concatenate(E)
    emax = float(ev.max())
    lam = np.maximum(eps, np.concatenate([1.0 / e for e in E]))
    active = lam <= eps
    f = nll_multi(E, _split(lam, ks), modalities)
    gtol = 1e-12 * float(np.abs(ev).sum())
    it = 0
    for it in range(max_iter):
        lams = _split(lam, ks)
        g = np.concatenate(marginals_multi(lams, modalities))
        grad = 0.5 * (ev - g)
        free_axes = [a for a in range(nax) if not active[off[a]:off[a + 1]].any()]
        Q = gauge_lift(ks, gauge_space_free(nax, modalities, free_axes))
        q = Q @ (Q.T @ grad)
        if np.linalg.norm(q) > gtol:
            d = -q
            d[active] = 0.0          # q lives on the free axes (rounding elsewhere)
            ratio = np.where(d < 0, (lam - eps) / np.where(d < 0, -d, 1.0), np.inf)
            i = int(np.argmin(ratio))
            lam = np.maximum(eps, lam + ratio[i] * d)
            lam[i] = eps
            active[i] = True
            f = nll_multi(E, _split(lam, ks), modalities)
            continue
        F = ~active
        r_free = float(np.max(np.abs(ev - g)[F], initial=0.0)) / emax
        if r_free <= tol:
            mult = (ev - g) / emax
            if active.any() and float(mult[active].min()) < -tol:
                idx = np.nonzero(active)[0]
                active[idx[int(np.argmin(mult[active]))]] = False
                continue
            break
        idx = np.nonzero(F)[0]
        H = _hessian_multi(lams, modalities, ks)
        QF = Q[idx, :]
        P = np.eye(len(idx)) - QF @ QF.T
        dF = -P @ np.linalg.lstsq(P @ H[np.ix_(idx, idx)] @ P, P @ grad[idx], rcond=None)[0]
        d = np.zeros_like(lam)
        d[idx] = dF
        ratio = np.where(d < 0, (lam - eps) / np.where(d < 0, -d, 1.0), np.inf)
        amax = float(ratio.min())
        alpha = min(1.0, amax)
        hit = alpha == amax
        while True:
            cand = np.maximum(eps, lam + alpha * d)
            fc = nll_multi(E, _split(cand, ks), modalities)
            if fc <= f + 1e-4 * alpha * float(grad @ d):
                break
            alpha *= 0.5
            hit = False
            if alpha < 1e-14:
                cand, fc = lam, f
                break
        if hit:
            i = int(np.argmin(ratio))
            cand[i] = eps
            active[i] = True
        lam, f = cand, fc
    return _split(lam, ks), it, active


def _apply_gauge(lams, E, modalities, gauge, free_axes):
    """Gauge 0 (reading G / G2): λ_l ← λ_l − (P_{G_F} μ)_l, μ_l = min λ_l; gauge 1: remove the
    G_F component of λ − 1/E in the Σk coordinates (Algorithm 1's gradient steps keep
    λ − λ⁰ ⊥ G).  G_F: the gauge directions over free_axes (all axes in the interior)."""
    nax = len(lams)
    N = gauge_space_free(nax, modalities, free_axes)
    if N.size == 0:
        return [np.asarray(l, np.float64).copy() for l in lams]
    if gauge == 0:
        mu = np.array([float(np.min(l)) for l in lams])
        sh = N @ (N.T @ mu)
        return [np.asarray(l, np.float64) - float(sh[a]) for a, l in enumerate(lams)]
    ks = [len(l) for l in lams]
    Q = gauge_lift(ks, N)
    v = np.concatenate([np.asarray(l, np.float64) - 1.0 / np.asarray(e, np.float64)
                        for l, e in zip(lams, E)])
    return _split(np.concatenate(lams) - Q @ (Q.T @ v), ks)


def trace_inconsistency_multi(E, modalities) -> float:
    """|P_G(tr E)|_max / mean tr E: the gauge component of the per-axis traces (reading T)."""
    tr = np.array([float(np.sum(e)) for e in E])
    N = gauge_space_multi(len(E), modalities)
    ptr = N @ (N.T @ tr) if N.size else np.zeros_like(tr)
    return float(np.max(np.abs(ptr)) / max(abs(tr.mean()), 1e-300))


def _solve_mle(E, modalities, tol, max_iter, gauge, eps_scale, trace_tol):
    E = [np.asarray(e, np.float64) for e in E]
    if any(np.any(~np.isfinite(e)) or np.any(e <= 0) for e in E):
        raise ValueError("E must be finite and > 0 (Thm 4 hypothesis, P:742)")
    single = modalities is None
    if single:
        modalities = [list(range(len(E)))]
    _check_modalities(len(E), modalities)
    eps = eps_scale * max(float(np.max(1.0 / e)) for e in E)
    ti = trace_inconsistency(E) if single else trace_inconsistency_multi(E, modalities)
    if ti <= trace_tol:
        Ee = project_spectrum(E, modalities)
        lams, it = _interior_newton(Ee, modalities, tol, max_iter)
        lams = _apply_gauge(lams, E, modalities, gauge, list(range(len(E))))
        active = np.zeros(sum(len(e) for e in E), bool)
        stat = stationarity_multi(Ee, lams, modalities)
        regime = "interior"
    else:
        lams, it, active = _box_mle(E, modalities, eps, tol, max_iter)
        ks = [len(e) for e in E]
        off = np.cumsum([0] + ks)
        free_axes = [a for a in range(len(E)) if not active[off[a]:off[a + 1]].any()]
        lams = _apply_gauge(lams, E, modalities, gauge, free_axes)
        stat = kkt_residual(E, lams, eps * (1 + 1e-9), modalities)
        regime = "barrier"
    info = dict(iterations=it, stationarity=stat, nll=nll_multi(E, lams, modalities),
                grid_min=min(float(s.min()) for s in grid_sums_multi(lams, modalities)),
                trace_inconsistency=ti, floor_active=bool(active.any()), eps=eps,
                regime=regime, active=active)
    return lams, info


def paper_gd_solve(E, max_iter: int = 200000, tol: float = 1e-9, eps_scale: float = 1e-10):
    """Algorithm 1 step by step, in its order and notation, for tiny problems.

    Λ ← 1/E (line 5); μ ← 1 (line 6); while not converged (line 7; Q4 criterion):
      Λ' ← Λ − μ·½(E − g(Λ))   (lines 8-9, reading Q1: the printed update omits Λ − μ·)
      while Σ_l min Λ'_l < ε  (lines 11-12, reading Q3: grid-minimum feasibility) or the
      NLL does not decrease (reading Q2): μ ← μ/2, recompute Λ' (lines 13-14)
      Λ ← Λ' (lines 16-17).
    """
    E = [np.asarray(e, np.float64) for e in E]
    lams = [1.0 / e for e in E]
    eps = eps_scale * max(float(np.max(1.0 / e)) for e in E)
    mu = 1.0
    f = nll(E, lams)
    it = 0
    while stationarity(E, lams) > tol and it < max_iter:
        grad = gradient(E, lams)
        while True:
            cand = [l - mu * g for l, g in zip(lams, grad)]
            smin = sum(float(np.min(c)) for c in cand)
            if smin >= eps:
                fc = nll(E, cand)
                if fc <= f:
                    break
            mu *= 0.5
            if mu < 1e-300:
                return lams, dict(iterations=it, stationarity=stationarity(E, lams))
        lams, f = cand, fc
        it += 1
    return lams, dict(iterations=it, stationarity=stationarity(E, lams))


# ---------------------------------------------------------------------------
# Nonparanormal skeptic via COCA and the sparse rank-one form
# ---------------------------------------------------------------------------

def nonparanormal(x: np.ndarray, axis: int) -> np.ndarray:
    """COCA transform of mat_l[D] ("replacing D_l with its ranks, mapping them to a
    normal distribution"): each row i (all entries with l-index i) is ranked, ties sharing
    the smallest rank (reading Q19, as in the worked example P:983-996), and r -> Φ^-1(r /
    (n + 1)) with n = d_rest (the product of the other axes).  Returns the transformed
    d_l x d_rest matrix (fp64)."""
    from scipy.special import ndtri
    from scipy.stats import rankdata
    m = matricize(x, axis)
    r = rankdata(m, method="min", axis=1)
    return ndtri(r / (m.shape[1] + 1.0))


def nonparanormal_sparse_split(x: np.ndarray, axis: int):
    """The sparse rank-one form: nonparanormal(x) = S + z 1^T, where z_i is the
    value the zeros of row i map to and S is zero wherever mat_l[D] is ("the same
    sparsity structure as our original data").  Returns (S, z); rows without zeros get
    z_i = 0."""
    m = matricize(x, axis)
    t = nonparanormal(x, axis)
    zero = m == 0
    z = np.array([t[i, zero[i]][0] if zero[i].any() else 0.0 for i in range(m.shape[0])])
    S = np.where(zero, 0.0, t - z[:, None])
    return S, z


def gram_eig_nonparanormal(x: np.ndarray, axis: int, k: int):
    """Top-k left singular vectors / σ² of the COCA-transformed mat_l."""
    t = nonparanormal(x, axis)
    if not 1 <= k <= min(t.shape):
        raise RankError(f"k={k} not in [1, {min(t.shape)}] (S:116)")
    u, sig, _ = np.linalg.svd(t, full_matrices=False)
    e = sig ** 2
    _check_rank(e, k)
    return u[:, :k].copy(), e[:k].copy()


# ---------------------------------------------------------------------------
# Multi-modal datasets — shared axes (Thm 2 Σ_γ P:356, Alg. 1 line 2 P:909)
# ---------------------------------------------------------------------------
# A modality γ is a tensor D^γ whose axes are a subset of the global axes (no repeated axis
# within one modality); `modalities` lists, per modality, its global axis ids in the
# tensor's own axis order.

def gram_eig_multi(tensors, modalities, axis: int, k: int):
    """Alg. 1 lines 2-4 for global axis `axis`: D_l = [mat_l(D^γ1) ... mat_l(D^γΓ)] over the
    modalities containing l, top-k left singular vectors and E = σ²."""
    blocks = [matricize(x, list(mod).index(axis)) for x, mod in zip(tensors, modalities)
              if axis in mod]
    if not blocks:
        raise ValueError(f"axis {axis} occurs in no modality")
    m = np.concatenate(blocks, axis=1)
    if not 1 <= k <= min(m.shape):
        raise RankError(f"k={k} not in [1, {min(m.shape)}] (S:116)")
    u, sig, _ = np.linalg.svd(m, full_matrices=False)
    e = sig ** 2
    _check_rank(e, k)
    return u[:, :k].copy(), e[:k].copy()


def _check_modalities(nax: int, modalities):
    for mod in modalities:
        if len(set(mod)) != len(mod):
            raise ValueError("repeated axis within a modality (P:181)")
        if any(a < 0 or a >= nax for a in mod):
            raise ValueError("axis id out of range")
    if set(a for mod in modalities for a in mod) != set(range(nax)):
        raise ValueError("every axis must occur in some modality")


def grid_sums_multi(lams, modalities):
    """Per modality γ: s^γ_j = Σ_{l∈γ} λ_l[j_l] on γ's k-grid (diagonal of ⊕_{l∈γ}Λ_l)."""
    return [grid_sums([lams[a] for a in mod]) for mod in modalities]


def marginals_multi(lams, modalities):
    """Σ_{γ∋l} tr^{k^γ_<l}_{k^γ_>l}[(⊕_{l'∈γ}Λ_l')^†] diagonals (Thm 2): per axis l,
    the sum over the modalities containing l of the single-modality marginals."""
    g = [np.zeros(len(l)) for l in lams]
    for mod in modalities:
        mg = marginals([lams[a] for a in mod])
        for pos, a in enumerate(mod):
            g[a] = g[a] + mg[pos]
    return g


def nll_multi(E, lams, modalities) -> float:
    """NLL = ½ Σ_l E_l·λ_l − ½ Σ_γ Σ_{j∈grid γ} log s^γ_j: the product of the per-modality
    densities in the eigenbasis of S_l = Σ_γ S^γ_l (constants dropped, Q11)."""
    lin = sum(float(np.dot(np.asarray(e, np.float64), np.asarray(l, np.float64)))
              for e, l in zip(E, lams))
    tot = 0.0
    for s in grid_sums_multi(lams, modalities):
        if s.min() <= 0:
            return np.inf
        tot += float(np.log(s).sum())
    return 0.5 * lin - 0.5 * tot


def gradient_multi(E, lams, modalities):
    """∂NLL/∂Λ_l = ½ (E_l − Σ_{γ∋l} g^γ_l)  (Theorem 2)."""
    g = marginals_multi(lams, modalities)
    return [0.5 * (np.asarray(e, np.float64) - gl) for e, gl in zip(E, g)]


def stationarity_multi(E, lams, modalities) -> float:
    g = marginals_multi(lams, modalities)
    emax = max(float(np.max(e)) for e in E)
    return max(float(np.max(np.abs(np.asarray(e) - gl))) for e, gl in zip(E, g)) / emax


def gauge_space_multi(nax: int, modalities) -> np.ndarray:
    """Orthonormal basis (nax x r) of G = {c : Σ_{l∈γ} c_l = 0 for every γ}: the per-axis
    shifts λ_l + c_l that leave every grid sum unchanged (reading G)."""
    M = np.zeros((len(modalities), nax))
    for r, mod in enumerate(modalities):
        M[r, list(mod)] = 1.0
    _, sv, vt = np.linalg.svd(M)
    rank = int(np.sum(sv > 1e-12 * max(sv.max(), 1.0)))
    return vt[rank:].T.copy()


def canonical_gauge_multi(lams, modalities):
    """Gauge 0 for shared axes (reading G2): with μ_l = min λ_l, subtract the G-component
    of μ: λ_l ← λ_l − (P_G μ)_l.  A function of the gauge class only (P_G c = c on G);
    for one modality P_G μ = μ − mean(μ), i.e. canonical_gauge."""
    N = gauge_space_multi(len(lams), modalities)
    mu = np.array([float(np.min(l)) for l in lams])
    sh = N @ (N.T @ mu) if N.size else np.zeros(len(lams))
    return [np.asarray(l, np.float64) - float(sh[a]) for a, l in enumerate(lams)]


def solve_eigvals_multi(E, modalities, tol: float = 1e-12, max_iter: int = 200,
                        gauge: int = 0, eps_scale: float = 1e-10, trace_tol: float = 1e-8):
    """Multi-modal eigenvalue MLE (Thm 2 with Σ_γ): argmin of nll_multi on the domain
    Λ_l >= ε, computed as in solve_eigvals (reading T with the multi-modal gauge space G,
    reading G2): interior projected Newton on G⊥ when |P_G(tr E)| <= trace_tol, else the
    active-set method on the box."""
    return _solve_mle(E, [list(m) for m in modalities], tol, max_iter, gauge, eps_scale,
                      trace_tol)


# ---------------------------------------------------------------------------
# Brute-force dense algebra (pins only): Kronecker sum, sb-trace, dense NLL
# ---------------------------------------------------------------------------

def kron_sum(mats) -> np.ndarray:
    """⊕_l Ψ_l = Σ_l I_{d_<l} ⊗ Ψ_l ⊗ I_{d_>l}  (definition)."""
    ds = [m.shape[0] for m in mats]
    total = int(np.prod(ds))
    out = np.zeros((total, total))
    for l, m in enumerate(mats):
        a = int(np.prod(ds[:l])) if l else 1
        b = int(np.prod(ds[l + 1:])) if l + 1 < len(ds) else 1
        out += np.kron(np.kron(np.eye(a), m), np.eye(b))
    return out


def sb_trace(M: np.ndarray, a: int, b: int, d: int) -> np.ndarray:
    """Stridewise-blockwise trace: tr^a_b[M]_{ij} = tr[M (I_a ⊗ J^{ij} ⊗ I_b)]."""
    out = np.zeros((d, d))
    for i in range(d):
        for j in range(d):
            J = np.zeros((d, d))
            J[i, j] = 1.0
            out[i, j] = np.trace(M @ np.kron(np.kron(np.eye(a), J), np.eye(b)))
    return out


def dense_nll(S_list, psis, rtol: float = 1e-10) -> float:
    """Matrix-form NLL ½ Σ tr[S_l Ψ_l] − ½ logdet†(⊕Ψ) (constants dropped)."""
    om = kron_sum(psis)
    ev = np.linalg.eigvalsh(om)
    keep = np.abs(ev) > rtol * np.max(np.abs(ev))
    return 0.5 * sum(float(np.trace(S @ P)) for S, P in zip(S_list, psis)) \
        - 0.5 * float(np.log(ev[keep]).sum())


# ---------------------------------------------------------------------------
# Recomposition + sparsification — Alg. 1 lines 18-20
# ---------------------------------------------------------------------------

def psi_rows(V: np.ndarray, lam: np.ndarray, rows) -> np.ndarray:
    """Rows of Ψ = V diag(λ) V^T (Cor. of Thm 2), fp64: ψ_i· = (V_i ⊙ λ) V^T."""
    V = np.asarray(V, np.float64)
    lam = np.asarray(lam, np.float64)
    rows = np.asarray(rows, dtype=np.int64)
    return (V[rows] * lam) @ V.T


def top_t_row(psi_row: np.ndarray, i: int, t: int):
    """Per-vertex top-t (reading Q8/Q9): the t_eff = min(t, n−1) entries j ≠ i with the
    largest |ψ_ij|, ties → smaller j; returned in ascending-j order (cols, vals)."""
    n = psi_row.shape[0]
    te = min(t, n - 1)
    a = np.abs(psi_row).astype(np.float64)
    a[i] = -np.inf
    if te <= 0:
        return np.zeros(0, np.int64), np.zeros(0)
    thr = np.partition(a, n - te)[n - te]          # te-th largest magnitude
    cand = np.nonzero(a >= thr)[0]                 # every entry tied at the boundary too
    order = np.lexsort((cand, -a[cand]))[:te]      # rank by (−|ψ|, j)
    sel = np.sort(cand[order])
    return sel.astype(np.int64), psi_row[sel].astype(np.float64)


def threshold_row(psi_row: np.ndarray, i: int, tau: float):
    """Mode 1: all j ≠ i with |ψ_ij| > τ, ascending j (reading Q15)."""
    a = np.abs(psi_row)
    a[i] = -np.inf
    sel = np.nonzero(a > tau)[0]
    return sel.astype(np.int64), psi_row[sel].astype(np.float64)


def sparse_precision(V, lam, row_begin: int, row_end: int, mode: int = 0, t: int = 10,
                     tau: float = 0.0, rows=None, block: int = 256):
    """thresh_{n_l}[V Λ V^T] for rows [row_begin,row_end) (or an explicit ``rows`` list)
    against all n columns; directed per-row CSR (row_ptr, col, val), ascending columns."""
    if rows is None:
        rows = np.arange(row_begin, row_end, dtype=np.int64)
    rows = np.asarray(rows, np.int64)
    cols, vals, ptr = [], [], [0]
    for b0 in range(0, len(rows), block):
        rb = rows[b0:b0 + block]
        P = psi_rows(V, lam, rb)
        for r, i in enumerate(rb):
            if mode == 0:
                c, v = top_t_row(P[r], int(i), t)
            else:
                c, v = threshold_row(P[r], int(i), tau)
            cols.append(c)
            vals.append(v)
            ptr.append(ptr[-1] + len(c))
    col = np.concatenate(cols) if cols else np.zeros(0, np.int64)
    val = np.concatenate(vals) if vals else np.zeros(0)
    return np.asarray(ptr, np.int64), col, val


# ---------------------------------------------------------------------------
# Edge significance — Theorem 5 (P:768-), Corollary 10, Bonferroni (P:1033,
# P:1097).  Single modality: sqrt(d_\l) sigma^2 psi / 2 ~ N(0, 1) under the empty-graph null.
# ---------------------------------------------------------------------------

def wald_edge(psi: float, d_rest: int, sigma2: float, n_tests: int):
    """(z, p_raw, p_bonferroni) for one edge (Cor. 10; two-sided; Bonferroni over n_tests)."""
    from scipy.stats import norm
    z = np.sqrt(float(d_rest)) * sigma2 * psi / 2.0
    p_raw = min(1.0, 2.0 * norm.sf(abs(z)))
    return z, p_raw, min(1.0, n_tests * p_raw)


def wald_threshold(d_rest: int, sigma2: float, alpha: float, n_tests: int) -> float:
    """|psi| above which p_bonferroni < alpha: 2 z_{1 - alpha/(2 n_tests)} / (sqrt(d_\\l) sigma^2)."""
    from scipy.stats import norm
    return 2.0 * norm.isf(alpha / (2.0 * n_tests)) / (np.sqrt(float(d_rest)) * sigma2)


# ---------------------------------------------------------------------------
# Whole-graph edge rules (SPEC S:312 readings, Q16):
# overall thresholding ("the n_l largest edges overall"), optionally down-weighting edges of
# high-degree vertices ("dividing by the total outgoing edge weight of the vertex": score
# |psi_ij| / sqrt(w_i w_j), w_i = sum_{k != i} |psi_ik|) and keeping a minimum number of
# edges per vertex (each vertex's m best edges by the same score).
# ---------------------------------------------------------------------------

def overall_edges(V, lam, n_edges: int, downweight: bool = False, min_edges: int = 0):
    """Undirected edges (i < j) kept by the overall rule, sorted by (i, j); returns
    (i, j, psi_ij) arrays.  Dense n x n fp64 (small n only).  Ranking: score descending,
    ties -> smaller (i, j) lexicographically; min-edges ties -> smaller j."""
    V = np.asarray(V, np.float64)
    n = V.shape[0]
    P = (V * np.asarray(lam, np.float64)) @ V.T
    A = np.abs(P)
    np.fill_diagonal(A, 0.0)
    if downweight:
        w = A.sum(axis=1)
        inv = np.where(w > 0, 1.0 / np.sqrt(np.where(w > 0, w, 1.0)), 0.0)
        S = A * inv[:, None] * inv[None, :]
    else:
        S = A
    iu, ju = np.triu_indices(n, 1)
    sc = S[iu, ju]
    order = np.lexsort((ju, iu, -sc))          # score desc, then i, then j
    order = order[sc[order] > 0][:n_edges]     # an exactly-zero psi_ij is no edge (Q17)
    keep = set(zip(iu[order].tolist(), ju[order].tolist()))
    if min_edges > 0:
        for i in range(n):
            row = S[i].copy()
            row[i] = -np.inf
            js = np.lexsort((np.arange(n), -row))[:min(min_edges, n - 1)]
            for j in js.tolist():
                if row[j] > 0:
                    keep.add((min(i, j), max(i, j)))
    e = np.array(sorted(keep), dtype=np.int64).reshape(-1, 2)
    return e[:, 0], e[:, 1], P[e[:, 0], e[:, 1]]


def edges_to_symmetric_csr(n: int, i, j, v):
    """Both directions of every undirected edge, rows ascending, columns ascending."""
    r = np.concatenate([i, j])
    c = np.concatenate([j, i])
    vv = np.concatenate([v, v])
    o = np.lexsort((c, r))
    r, c, vv = r[o], c[o], vv[o]
    rp = np.zeros(n + 1, np.int64)
    np.add.at(rp, r + 1, 1)
    return np.cumsum(rp), c, vv
