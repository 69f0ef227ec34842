"""Threshold mode (mode 1) at n = 1e6: symmetric (screening) vs plain scheme."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2407_19892_b200 as G
n, k = 1_000_000, 100
g = torch.Generator(device="cuda").manual_seed(5)
V = torch.linalg.qr(torch.randn(n, k, device="cuda", dtype=torch.float64, generator=g))[0].float().contiguous()
lam = torch.exp(torch.randn(k, device="cuda", dtype=torch.float64, generator=g)).sort(descending=True)[0]
rp, c, v = G.ggm_sparse_precision(V, lam, mode=0, topk=10)
tau = float(v.abs().view(n, 10).min(dim=1).values.max())   # at most 10 edges per row
G.set_timing(True)
for sym in (1, 2):
    plan = G.SparsePlan(n, k, 0, n, mode=1, tau=tau, capacity=40 * n, symmetric=sym)
    plan.run(V, lam)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); nnz = plan.run(V, lam); e1.record(); torch.cuda.synchronize()
    print(f"sym={sym}: {e0.elapsed_time(e1):.1f} ms nnz={nnz} ({nnz/n:.1f}/row) {G.last_stats()['scheme']} timing={G.last_timing()}")
