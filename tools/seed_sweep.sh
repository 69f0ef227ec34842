# C4 / C5 symmetric scheme vs the seed sample fraction (GGM_SEED_FRAC tuning hook)
cat > /tmp/ss.py <<'PY'
import sys, os
sys.path.insert(0, os.getcwd())
import torch, paper_2407_19892_b200 as G
for n, k in [(200_000, 64), (1_000_000, 100)]:
    g = torch.Generator(device="cuda").manual_seed(0)
    V = torch.linalg.qr(torch.randn(n, k, device="cuda", generator=g, dtype=torch.float64))[0].float().contiguous()
    lam = torch.exp(torch.randn(k, device="cuda", dtype=torch.float64, generator=g)).sort(descending=True).values
    plan = G.SparsePlan(n, k, 0, n, mode=0, topk=10, symmetric=1)
    G.set_timing(True)
    best = None
    for r in range(3):
        plan.run(V, lam); torch.cuda.synchronize()
        ms = G.last_timing()
        best = ms if best is None or ms[1] < best[1] else best
    st = G.last_stats()
    print(f"frac={os.environ.get('GGM_SEED_FRAC','default')} n={n}: prep {best[0]:.2f} main {best[1]:.2f} merge {best[2]:.2f} cand/row {st['candidates']/n:.1f}", flush=True)
PY
timeout 300 python /tmp/ss.py
for f in ${FRACS:-64 32 16 8 4 2}; do GGM_SEED_FRAC=$f timeout 300 python /tmp/ss.py; done
