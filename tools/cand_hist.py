"""Candidates per target row of the symmetric scheme (single rank of the sharded form):
distribution and the rows with the most candidates.  Usage: python tools/cand_hist.py C4|C5"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2407_19892_b200 as G  # noqa: E402
from synth import gen  # noqa: E402

cfg = gen.config(sys.argv[1] if len(sys.argv) > 1 else "C4")
V, lam = [torch.from_numpy(x).cuda() for x in cfg["axes"][0]]
n, k = V.shape
plan = G.SymShardPlan(n, k, cfg["t"], 0, 1)
key, val, counts, perm = plan.run(V, lam)
c = torch.bincount(key.long(), minlength=n).double()
q = torch.tensor([0.5, 0.9, 0.99, 0.999, 0.9999, 1.0], dtype=torch.float64, device=c.device)
print(f"n={n} k={k} total={int(c.sum())} per row mean {c.mean():.2f} quantiles",
      [round(float(x), 1) for x in torch.quantile(c, q)])
top = torch.topk(c, 10)
print("largest rows (bound order index, count):", list(zip(top.indices.tolist(), top.values.long().tolist())))
edges = [0, 10, 20, 50, 100, 256, 1000, 10**9]
for a, b in zip(edges[:-1], edges[1:]):
    m = (c >= a) & (c < b)
    print(f"  [{a},{b}): rows {int(m.sum())} candidates {int(c[m].sum())}")
