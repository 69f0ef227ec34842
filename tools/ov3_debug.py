import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_2407_19892_b200 as G
from synth import gen
n, k = 70000, 64
V, lam = gen.small_factor(2024, n, k)
Vd = torch.from_numpy(V).cuda(); ld = torch.from_numpy(np.asarray(lam, np.float64)).cuda()
rp, c, v = G.ggm_sparse_precision_overall(Vd, ld, 10 * n, min_edges=1)
print("path", G.overall_last_path())
