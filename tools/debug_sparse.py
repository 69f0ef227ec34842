"""Quick GPU sanity run of the three C-ABI calls on tiny inputs (prints diagnostics)."""
import sys
import time
import os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2407_19892_b200 as G
import oracle as O
from synth import gen

print("device:", torch.cuda.get_device_name(0), "supported:", G.device_supported(), flush=True)
for (n, k) in [(256, 16), (300, 64), (1000, 100), (600, 300)]:
    V, lam = gen.small_factor(1, n, k)
    Vd = torch.from_numpy(V).cuda(); ld = torch.from_numpy(lam).cuda()
    t0 = time.time()
    rp, c, v = G.ggm_sparse_precision(Vd, ld, 0, n, mode=1, tau=0.0)
    torch.cuda.synchronize()
    rp, c, v = rp.cpu().numpy(), c.cpu().numpy(), v.cpu().numpy()
    P = (V.astype(np.float64) * lam) @ V.astype(np.float64).T
    D = np.zeros((n, n))
    for i in range(n):
        D[i, c[rp[i]:rp[i + 1]]] = v[rp[i]:rp[i + 1]]
    off = ~np.eye(n, dtype=bool)
    err = np.abs(D - P)[off]
    print(f"n={n} k={k} nnz={len(c)} (full {n*(n-1)}) max|err|={err.max():.3e} "
          f"max|P|={np.abs(P[off]).max():.3e} rel={err.max()/np.abs(P[off]).max():.3e} "
          f"t={time.time()-t0:.2f}s", flush=True)
    if err.max() > 1e-4 * np.abs(P[off]).max():
        bad = np.argwhere((np.abs(D - P) > 1e-4 * np.abs(P).max()) & off)
        print("  first bad", bad[:10].tolist())
        print("  D[0,:8]", D[0, :8]); print("  P[0,:8]", P[0, :8])
    rp, c, v = G.ggm_sparse_precision(Vd, ld, 0, n, mode=0, topk=10)
    rp, c, v = rp.cpu().numpy(), c.cpu().numpy(), v.cpu().numpy()
    ok = 0
    for i in range(n):
        oc, ov = O.top_t_row(P[i], i, 10)
        ok += int(np.array_equal(oc, c[rp[i]:rp[i + 1]]))
    print(f"   top10 exact rows {ok}/{n}", flush=True)
g = G.ggm_grid_marginals(torch.tensor([1.0, 2.0, 3.0, 4.0], dtype=torch.float64).cuda(), (2, 2))
print("marginals", g.cpu().numpy(), "want [0.45 0.3667 0.45 0.3667]", flush=True)
lam, info = G.ggm_solve_eigvals(torch.tensor([3.0, 1.0, 2.0, 2.0], dtype=torch.float64).cuda(), (2, 2))
print("solve", lam.cpu().numpy(), info, flush=True)
x = gen.small_tensor(3, (60, 25))
Vg, E, tr = G.ggm_gram_eig(torch.from_numpy(x).cuda(), 0, 10)
Vo, Eo = O.gram_eig(x, 0, 10)
print("gram E rel err", np.max(np.abs(E.cpu().numpy() - Eo) / Eo), flush=True)
