"""One ggm_sparse_precision call on random orthonormal factors (for ncu).  Env: N, K, SYM
(0 auto / 1 sym / 2 plain), T."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2407_19892_b200 as G
n, k = int(os.environ.get("N", "200000")), int(os.environ.get("K", "100"))
g = torch.Generator(device="cuda").manual_seed(0)
V = torch.linalg.qr(torch.randn(n, k, device="cuda", generator=g, dtype=torch.float64))[0].float().contiguous()
lam = torch.exp(torch.randn(k, device="cuda", dtype=torch.float64, generator=g)).sort(descending=True).values
plan = G.SparsePlan(n, k, 0, n, mode=0, topk=int(os.environ.get("T", "10")), symmetric=int(os.environ.get("SYM", "2")))
plan.run(V, lam)
torch.cuda.synchronize()
print(G.last_stats(), G.last_timing())
