"""One C3-size solve with a fixed iteration count (for ncu)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2407_19892_b200 as G
ks = (400, 300, 200)
rng = np.random.default_rng(0)
E = np.concatenate([np.sort(rng.uniform(0.5, 1.5, k))[::-1] * 1000.0 / k for k in ks])
Ed = torch.from_numpy(E).cuda()
for _ in range(2):
    try:
        G.ggm_solve_eigvals(Ed, ks, tol=1e-300, max_iter=50)
    except G.GGMError:
        pass
torch.cuda.synchronize()
print("ok")
