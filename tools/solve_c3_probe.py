"""C3 eigenvalue solve alone (for ncu captures of solve_kernel)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2407_19892_b200 as G
from synth import gen
cfg = gen.config("C3")
X = torch.from_numpy(cfg["X"]).cuda()
res, _ = G.ggm_gram_eig_axes(X, cfg["k"])
Ec = torch.cat([E for _, E in res])
lam, info = G.ggm_solve_eigvals(Ec, cfg["k"], max_iter=int(os.environ.get("ITERS", "20000")))
print(info)
