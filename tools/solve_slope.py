"""Per-iteration cost of ggm_solve_eigvals: slope of wall time vs max_iter (tol unreachable)."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2407_19892_b200 as G
for ks in [(400, 300, 200), (100, 100), (50, 50), (200, 150, 100)]:
    rng = np.random.default_rng(0)
    E = np.concatenate([np.sort(rng.uniform(0.5, 1.5, k))[::-1] * 1000.0 / k for k in ks])
    Ed = torch.from_numpy(E).cuda()
    res = []
    for it in (50, 50, 550):
        torch.cuda.synchronize(); t0 = time.perf_counter()
        try:
            G.ggm_solve_eigvals(Ed, ks, tol=1e-300, max_iter=it)
        except G.GGMError:
            pass
        res.append(time.perf_counter() - t0)
    slope = (res[2] - res[1]) / 500
    print(f"ks={ks}: per-iteration {slope*1e6:.1f} us, fixed {(res[1]-50*slope)*1e3:.2f} ms, "
          f"{np.prod(ks)/slope:.3e} grid pts/s", flush=True)
