"""C2 / C3 per-axis gram_eig time with DSYEVD vs DSYEVDX (env GGM_NO_SYEVDX)."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2407_19892_b200 as G
from synth import gen
for name in ("C2", "C3"):
    cfg = gen.config(name)
    X = torch.from_numpy(cfg["X"]).cuda()
    for a, k in enumerate(cfg["k"]):
        G.ggm_gram_eig(X, a, k); torch.cuda.synchronize()
        t0 = time.perf_counter(); V, E, _ = G.ggm_gram_eig(X, a, k); torch.cuda.synchronize()
        print(name, a, k, f"{(time.perf_counter()-t0)*1e3:.2f} ms", f"E0 {E[0].item():.6e} Ek {E[-1].item():.6e}")
