"""Phase estimate of ggm_sparse_precision_overall at C5 axis-A size (GPU probe)."""
import sys, time
import numpy as np
import torch
sys.path.insert(0, ".")
import paper_2407_19892_b200 as G

n, k = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000, 100
g = torch.Generator(device="cuda").manual_seed(5)
V = torch.linalg.qr(torch.randn(n, k, device="cuda", dtype=torch.float64, generator=g))[0].float().contiguous()
lam = torch.exp(torch.randn(k, device="cuda", dtype=torch.float64, generator=g)).sort(descending=True)[0]


def tm(f, reps=2):
    f(); torch.cuda.synchronize()
    best = 1e30
    for _ in range(reps):
        t0 = time.perf_counter(); r = f(); torch.cuda.synchronize()
        best = min(best, (time.perf_counter() - t0) * 1e3)
    return best, r


G.set_timing(True)
for dw in (True, False):
    _, _, _, caps = G.ggm_sparse_precision_overall(V, lam, 10 * n, downweight=dw, min_edges=1, return_caps=True)
    ms, r = tm(lambda: G.ggm_sparse_precision_overall(V, lam, 10 * n, downweight=dw, min_edges=1,
                                                      cand_capacity=caps[0], capacity=caps[1]))
    print(f"overall dw={dw}: {ms:.1f} ms caps={caps} edges={r[1].numel()//2} path={G.overall_last_path()} {G.overall_last_timing()}")
ms, r = tm(lambda: G.ggm_sparse_precision(V, lam, mode=0, topk=32))
print(f"top-32 auto: {ms:.1f} ms stats={G.last_stats()}")
v = r[2].abs()
tau = float(torch.sort(v, descending=True)[0][2 * 10 * n - 1])
ms, r = tm(lambda: G.ggm_sparse_precision(V, lam, mode=1, tau=tau * 0.99999, capacity=25 * n))
print(f"threshold plain: {ms:.1f} ms nnz={r[1].numel()}")
ms, r = tm(lambda: G.ggm_sparse_precision(V, lam, mode=0, topk=10))
print(f"top-10 auto: {ms:.1f} ms")
# saturation: rows whose 32nd listed value >= tau
rp, c, val = G.ggm_sparse_precision(V, lam, mode=0, topk=32)
m32 = val.abs().view(n, 32).min(dim=1)[0]
print("rows saturated at the 2N-th listed value:", int((m32 >= tau).sum()))
