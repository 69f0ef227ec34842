"""Seeded shard call with and without the seed-call reuse (same workspace), C5 axis A, N = 8
shares: prep stage (CUDA events in libggm) of the first run after a seed call vs a repeat."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2407_19892_b200 as G  # noqa: E402
from synth import gen  # noqa: E402

cfg = gen.config("C5")
(V, lam), _ = [(torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda()) for a, b in cfg["axes"]]
n, k = V.shape
N = 8
plans = [G.SymShardPlan(n, k, cfg["t"], r, N) for r in range(N)]
parts = [p.seed(V, lam).clone() for p in plans]
thr = torch.stack(parts).min(dim=0).values
G.set_timing(True)
for rep in range(2):
    for r in (0, 7):
        if rep == 0:
            plans[r].seed(V, lam)  # fresh stamp for this rank's workspace
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        plans[r].run(V, lam, thr_all=thr)
        e1.record()
        torch.cuda.synchronize()
        print(f"rank {r} {'after seed (reuse)' if rep == 0 else 'repeat (no stamp)'}: call "
              f"{e0.elapsed_time(e1):.2f} ms, stages {[round(x, 3) for x in G.last_timing()]}",
              flush=True)
