"""Plain vs symmetric (screening) scheme time for mid-size axes (where the auto switch is)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2407_19892_b200 as G
G.set_timing(True)
for n in (2048, 4096, 8192):
    g = torch.Generator(device="cuda").manual_seed(1)
    V = torch.linalg.qr(torch.randn(n, 100, device="cuda", generator=g, dtype=torch.float64))[0].float().contiguous()
    lam = torch.exp(torch.randn(100, device="cuda", dtype=torch.float64, generator=g)).sort(descending=True).values
    for sym in (2, 1):
        plan = G.SparsePlan(n, 100, 0, n, mode=0, topk=10, symmetric=sym)
        for _ in range(3):
            plan.run(V, lam)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(10):
            plan.run(V, lam)
        e1.record()
        torch.cuda.synchronize()
        print(f"n={n} sym={sym}: {e0.elapsed_time(e1)/10:.3f} ms  {G.last_stats()['scheme']}")
