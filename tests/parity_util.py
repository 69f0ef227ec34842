"""Parity helpers shared by the GPU tests: compare a CUDA-path CSR against the fp64 oracle.

Tolerances (BASELINE.json north_star): values within 1e-4 relative with a 1e-6 absolute
floor; identical per-row top-t index sets except where the t-th and (t+1)-th oracle
magnitudes differ by less than that tolerance (then the GPU set must still be valid:
every chosen entry within tolerance of the oracle's t-th magnitude).  The strict gate
(strict=True: relative tolerance only, reading TOL in DESIGN.md) and the exact-match
fraction (assert_exact_fraction) are asserted where the inputs are shared by both sides.
"""
import numpy as np

import oracle as O

REL = 1e-4
ABS = 1e-6


def tol(x, strict=False):
    return REL * np.abs(x) if strict else np.maximum(REL * np.abs(x), ABS)


def check_topk(row_ptr, col, val, V, lam, rows, t, strict=False, chunk=64):
    """rows: global row ids corresponding to CSR rows 0..len(rows)-1 of the GPU output
    (row_ptr/col/val already restricted to those rows).  Returns stats dict; asserts.
    strict=True: the relative-only gate (reading TOL).  The oracle rows are formed `chunk`
    at a time (n up to 10^6 columns)."""
    V = np.asarray(V)
    n = V.shape[0]
    te = min(t, n - 1)
    rows = np.asarray(rows, dtype=np.int64)
    stats = dict(rows=len(rows), excused=0, exact=0, max_rel_err=0.0, max_abs_err=0.0)
    for c0 in range(0, len(rows), chunk):
        P = O.psi_rows(V, lam, rows[c0:c0 + chunk])
        for rr, i in enumerate(rows[c0:c0 + chunk]):
            r = c0 + rr
            c = np.asarray(col[row_ptr[r]:row_ptr[r + 1]], dtype=np.int64)
            v = np.asarray(val[row_ptr[r]:row_ptr[r + 1]], dtype=np.float64)
            assert len(c) == te, f"row {i}: {len(c)} entries != {te}"
            assert np.all(np.diff(c) > 0), f"row {i}: columns not strictly ascending"
            assert np.all((c >= 0) & (c < n) & (c != i)), f"row {i}: invalid column"
            want = P[rr, c]
            err = np.abs(v - want)
            assert np.all(err <= tol(want, strict)), (
                f"row {i}: value error {err.max():.3e} (|psi| {np.abs(want).max():.3e})")
            rel = err / np.maximum(np.abs(want), 1e-300)
            rel[err == 0] = 0.0
            stats["max_rel_err"] = max(stats["max_rel_err"], float(rel.max()))
            stats["max_abs_err"] = max(stats["max_abs_err"], float(err.max()))
            oc, _ = O.top_t_row(P[rr], int(i), t)
            if np.array_equal(oc, c):
                stats["exact"] += 1
                continue
            a = np.abs(P[rr]).copy()
            a[i] = -np.inf
            part = -np.partition(-a, min(te, n - 2))[:te + 1] if te < n - 1 else -np.sort(-a)
            srt = np.sort(part)[::-1]
            at, at1 = srt[te - 1], (srt[te] if te < n - 1 else -np.inf)
            gap_small = (at - at1) <= tol(at, strict)
            assert gap_small, f"row {i}: top-{t} set differs with a clear gap {at - at1:.3e}"
            # excused: the GPU set must still be a valid top set within tolerance
            assert np.all(np.abs(P[rr, c]) >= at - tol(at, strict)), f"row {i}: invalid near-tie set"
            stats["excused"] += 1
    return stats


def assert_exact_fraction(stats, min_frac, what=""):
    """The exact-match count (reading TOL): set parity on at least min_frac of the rows."""
    frac = stats["exact"] / max(stats["rows"], 1)
    assert frac >= min_frac, f"{what}: exact rows {stats['exact']}/{stats['rows']} < {min_frac}"


def check_threshold(row_ptr, col, val, V, lam, rows, tau):
    """Mode 1: every j != i with |psi| > tau; entries within tolerance of tau may differ."""
    P = O.psi_rows(V, lam, rows)
    for r, i in enumerate(rows):
        c = set(np.asarray(col[row_ptr[r]:row_ptr[r + 1]]).tolist())
        a = np.abs(P[r])
        a[i] = -np.inf
        sure_in = set(np.nonzero(a > tau + tol(tau))[0].tolist())
        maybe = set(np.nonzero(a > tau - tol(tau))[0].tolist())
        assert sure_in <= c <= maybe, f"row {i}: threshold set mismatch"
        cc = np.asarray(col[row_ptr[r]:row_ptr[r + 1]], dtype=np.int64)
        vv = np.asarray(val[row_ptr[r]:row_ptr[r + 1]], dtype=np.float64)
        assert np.all(np.diff(cc) > 0)
        assert np.all(np.abs(vv - P[r, cc]) <= tol(P[r, cc]))


def check_overall(row_ptr, col, val, V, lam, n_edges, downweight=False, min_edges=0):
    """Whole-graph rules: the GPU edge set equals oracle.overall_edges except
    near ties (score within tolerance of the global N-th score or of a vertex's m-th score);
    the CSR is symmetric with ascending columns and values within tolerance of psi_ij."""
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
    row_ptr, col, val = (np.asarray(x) for x in (row_ptr, col, val))
    assert row_ptr[0] == 0 and np.all(np.diff(row_ptr) >= 0) and row_ptr[-1] == len(col)
    rows = np.repeat(np.arange(n), np.diff(row_ptr))
    for r in range(n):
        c = col[row_ptr[r]:row_ptr[r + 1]]
        assert np.all(np.diff(c) > 0), f"row {r}: columns not strictly ascending"
    assert np.all((col >= 0) & (col < n) & (col != rows))
    d = {(int(a), int(b)): float(v) for a, b, v in zip(rows, col, val)}
    for (a, b), v in d.items():
        assert (b, a) in d and d[(b, a)] == v, f"asymmetric entry ({a},{b})"
    want = P[rows, col]
    assert np.all(np.abs(val - want) <= tol(want)), "value mismatch"
    G = {(a, b) for (a, b) in d if a < b}
    oi, oj, _ = O.overall_edges(V, lam, n_edges, downweight=downweight, min_edges=min_edges)
    Oset = set(zip(oi.tolist(), oj.tolist()))
    iu, ju = np.triu_indices(n, 1)
    sc = np.sort(S[iu, ju])[::-1]
    sN = sc[min(n_edges, len(sc)) - 1]
    m = min(min_edges, n - 1)
    rowthr = np.full(n, np.inf)
    if m > 0:
        Sr = S.copy()
        np.fill_diagonal(Sr, -np.inf)
        rowthr = -np.sort(-Sr, axis=1)[:, m - 1]
    diff = G ^ Oset
    for (a, b) in diff:
        s = S[a, b]
        near = [abs(s - sN) <= tol(sN)]
        if m > 0:
            near += [abs(s - rowthr[a]) <= tol(rowthr[a]), abs(s - rowthr[b]) <= tol(rowthr[b])]
        assert any(near), f"edge ({a},{b}) score {s:.6e} differs with a clear gap (sN {sN:.6e})"
    return dict(edges=len(G), oracle_edges=len(Oset), excused=len(diff))
