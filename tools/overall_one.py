"""One down-weighted overall-rules call at C5 axis-A size (for launch lists / A/B)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2407_19892_b200 as G  # noqa: E402

n, k = 1_000_000, 100
g = torch.Generator(device="cuda").manual_seed(5)
V = torch.linalg.qr(torch.randn(n, k, device="cuda", dtype=torch.float64, generator=g))[0].float().contiguous()
lam = torch.exp(torch.randn(k, device="cuda", dtype=torch.float64, generator=g)).sort(descending=True)[0]
G.set_timing(True)
_, _, _, caps = G.ggm_sparse_precision_overall(V, lam, 10 * n, downweight=True, min_edges=1, return_caps=True)
for _ in range(int(os.environ.get("REPS", "2"))):
    r = G.ggm_sparse_precision_overall(V, lam, 10 * n, downweight=True, min_edges=1,
                                       cand_capacity=caps[0], capacity=caps[1])
    torch.cuda.synchronize()
    print("overall", G.overall_last_timing(), flush=True)
