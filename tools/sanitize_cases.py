"""Small invocations of every kernel family for compute-sanitizer (memcheck / racecheck /
synccheck; tools/sanitize.sh): C1 spectrum + solve (MM, SQUAREM, barrier, Alg. 1 GD), the
grid pass, BK2 in every kind (plain list epilogue, 1-CTA and CTA-pair, streamed A at
k > 128, threshold mode, seed + symmetric screening scheme, 3-term symmetric), the overall
rules and the CSR / COCA spectrum.  Prints one line per case; exits non-zero on any error."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2407_19892_b200 as G  # noqa: E402
from synth import gen  # noqa: E402


def dev(x, dt=None):
    t = torch.from_numpy(np.ascontiguousarray(x)).cuda()
    return t if dt is None else t.to(dt)


def case(name, fn):
    fn()
    torch.cuda.synchronize()
    print(f"case {name}: ok", flush=True)


def main():
    only = set(sys.argv[1:])
    cfg = gen.config("C1")
    X = dev(cfg["X"])
    ks = cfg["k"]

    def spectrum_solve():
        Es = [G.ggm_gram_eig(X, a, k)[1] for a, k in enumerate(ks)]
        G.ggm_gram_eig_matrix(X, ks[0], ks[1])
        Ec = torch.cat(Es)
        G.ggm_solve_eigvals(Ec, ks)
        G.ggm_solve_eigvals(Ec, ks, method=1, gauge=1)
        G.ggm_solve_eigvals(Ec, ks, method=2, max_iter=50, tol=1e-3)
        E3 = dev(np.concatenate([np.array([5., 3, 2, 1]), np.array([4., 2]), np.array([3., 1, .5])]))
        G.ggm_solve_eigvals(E3, (4, 2, 3))                       # barrier regime
        lam = dev(np.random.default_rng(1).uniform(0.1, 2, 60 + 45 + 30))
        G.ggm_grid_marginals(lam, (60, 45, 30), with_logsum=True)
        x3 = dev(gen.small_tensor(3, (12, 9, 7)))
        G.ggm_gram_eig_axes(x3, [12, 9, 7])
    V, lam = gen.small_factor(5, 3000, 100)
    Vd, ld = dev(V), dev(np.asarray(lam, np.float64))
    V2, lam2 = gen.small_factor(6, 600, 300)
    tests = {
        "spectrum_solve": spectrum_solve,
        "bk2_plain_pair": lambda: G.ggm_sparse_precision(Vd, ld, 0, 3000, topk=10, symmetric=2),
        "bk2_plain_rows_chunks": lambda: G.ggm_sparse_precision(Vd, ld, 130, 901, topk=5, col_chunks=3),
        "bk2_streamed_k300": lambda: G.ggm_sparse_precision(dev(V2), dev(np.asarray(lam2, np.float64)), 0, 600, topk=10),
        "bk2_threshold": lambda: G.ggm_sparse_precision(Vd, ld, 0, 3000, mode=1, tau=1e-3),
        "bk2_symmetric_screen": lambda: G.ggm_sparse_precision(Vd, ld, 0, 3000, topk=10, symmetric=1),
        "bk2_symmetric_t32": lambda: G.ggm_sparse_precision(Vd, ld, 0, 3000, topk=32, symmetric=1),
        "overall_rules": lambda: G.ggm_sparse_precision_overall(Vd, ld, 30000, downweight=True, min_edges=1),
    }
    for name, fn in tests.items():
        if not only or name in only:
            case(name, fn)


if __name__ == "__main__":
    main()
