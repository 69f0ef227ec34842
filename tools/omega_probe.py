"""Iterations / time of ggm_solve_eigvals vs the update exponent GGM_MM_OMEGA (C1-C3)."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2407_19892_b200 as G
from synth import gen
om = os.environ.get("GGM_MM_OMEGA", "default")
for name in ("C1", "C2", "C3"):
    cfg = gen.config(name)
    X = torch.from_numpy(cfg["X"]).cuda()
    Es = [G.ggm_gram_eig(X, a, k)[1] for a, k in enumerate(cfg["k"])]
    Ec = torch.cat(Es)
    try:
        lam, info = G.ggm_solve_eigvals(Ec, cfg["k"]); torch.cuda.synchronize()
        ms = 1e9
        for _ in range(5):
            t0 = time.perf_counter(); lam, info = G.ggm_solve_eigvals(Ec, cfg["k"]); torch.cuda.synchronize()
            ms = min(ms, (time.perf_counter() - t0) * 1e3)
        print(f"omega={om} {name}: it={info['iterations']} ms={ms:.2f} stat={info['stationarity']:.2e}", flush=True)
    except Exception as e:
        print(f"omega={om} {name}: FAIL {e}", flush=True)
