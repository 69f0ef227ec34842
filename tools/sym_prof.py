"""One symmetric-scheme call at n=1e6, k=100 (for ncu)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2407_19892_b200 as G
n, k = int(os.environ.get("N", "1000000")), 100
g = torch.Generator(device="cuda").manual_seed(0)
V = torch.linalg.qr(torch.randn(n, k, device="cuda", generator=g, dtype=torch.float64))[0].float().contiguous()
lam = torch.exp(torch.randn(k, device="cuda", dtype=torch.float64, generator=g)).sort(descending=True).values
plan = G.SparsePlan(n, k, 0, n, mode=0, topk=10, symmetric=1)
plan.run(V, lam)
torch.cuda.synchronize()
print(G.last_stats())
