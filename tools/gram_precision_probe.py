"""Why the spectrum (a1 / f1) runs its Gram products in fp64 (BK5): on the C2
workload (10,000 x 2,000 log1p counts, k = 50, t = 10; BJ:8) compute the top-k spectrum from
an fp64 Gram and from an fp32-accumulated Gram of the same fp32 data (what an fp32-accurate
tensor-core GEMM -- 3xTF32 / 3xFP16 splits -- delivers at best), then the eigenvalue MLE and
the per-row top-10 graphs of both axes, and report the eigenvector subspace angles, the
relative error of the selected ψ values and the fraction of rows whose top-10 set changes.
CPU only (NumPy), run: python tools/gram_precision_probe.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import oracle as O  # noqa: E402
from synth import gen  # noqa: E402


def spectrum(X, axis, k, dtype):
    M = X if axis == 0 else X.T
    if M.shape[0] <= M.shape[1]:
        Gm = (M.astype(dtype) @ M.T.astype(dtype)).astype(np.float64)
        e, W = np.linalg.eigh(Gm)
        o = np.argsort(-e)[:k]
        return W[:, o], e[o]
    Gm = (M.T.astype(dtype) @ M.astype(dtype)).astype(np.float64)   # dual Gram
    e, W = np.linalg.eigh(Gm)
    o = np.argsort(-e)[:k]
    V = (M.astype(np.float64) @ W[:, o]) / np.sqrt(e[o])
    return V, e[o]


def main():
    cfg = gen.config("C2")
    X, ks, t = cfg["X"], cfg["k"], cfg["t"]
    res = {}
    for dt in (np.float64, np.float32):
        Vs, Es = zip(*[spectrum(X, a, k, dt) for a, k in enumerate(ks)])
        lams, _ = O.solve_eigvals(list(Es), tol=1e-12)
        res[np.dtype(dt).name] = (Vs, Es, lams)
    V64, E64, L64 = res["float64"]
    V32, E32, L32 = res["float32"]
    rng = np.random.default_rng(0)
    for a in range(2):
        n = X.shape[a]
        sv = np.linalg.svd(V64[a].T @ V32[a], compute_uv=False)
        sin_max = float(np.sqrt(max(0.0, 1.0 - sv.min() ** 2)))
        rows = np.sort(rng.choice(n, size=min(1000, n), replace=False))
        P64 = O.psi_rows(V64[a], L64[a], rows)
        P32 = O.psi_rows(V32[a], L32[a], rows)
        rel, changed = [], 0
        for r, i in enumerate(rows):
            c64, v64 = O.top_t_row(P64[r], int(i), t)
            c32, _ = O.top_t_row(P32[r], int(i), t)
            rel.append(np.max(np.abs(P32[r, c64] - v64) / np.abs(v64)))
            changed += int(not np.array_equal(c64, c32))
        print(f"axis {a} (n={n}): max rel eigenvalue err {np.max(np.abs(E32[a]-E64[a])/E64[a]):.2e}, "
              f"subspace sin(theta_max) {sin_max:.2e}, selected-psi rel err median "
              f"{np.median(rel):.2e} max {np.max(rel):.2e} (gate 1e-4), rows with a changed "
              f"top-{t} set {changed}/{len(rows)}", flush=True)


if __name__ == "__main__":
    main()
