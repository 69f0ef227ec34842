"""Symmetric scheme main-kernel timing at C4 / C5 sizes (QR factors), best of 3; for A/B of
library variants (GGM_LIB_PATH) in one session."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2407_19892_b200 as G  # noqa: E402

tag = os.environ.get("TAG", os.path.basename(os.environ.get("GGM_LIB_PATH", "base")))
for n, k in [(200_000, 64), (1_000_000, 100)]:
    g = torch.Generator(device="cuda").manual_seed(0)
    V = torch.linalg.qr(torch.randn(n, k, device="cuda", generator=g, dtype=torch.float64))[0].float().contiguous()
    lam = torch.exp(torch.randn(k, device="cuda", dtype=torch.float64, generator=g)).sort(descending=True).values
    plan = G.SparsePlan(n, k, 0, n, mode=0, topk=10, symmetric=1)
    G.set_timing(True)
    best = None
    for _ in range(3):
        plan.run(V, lam)
        torch.cuda.synchronize()
        ms = G.last_timing()
        best = ms if best is None or sum(ms) < sum(best) else best
    print(f"[{tag}] n={n}: prep {best[0]:.2f} main {best[1]:.2f} merge {best[2]:.2f} total {sum(best):.2f}", flush=True)
