"""Symmetric-scheme diagnostics: timing split and candidate statistics (random factors)."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2407_19892_b200 as G

def run(n, k, sym, t=10, ortho=False):
    g = torch.Generator(device="cuda").manual_seed(0)
    V = torch.randn(n, k, device="cuda", generator=g, dtype=torch.float64)
    if ortho:
        V = torch.linalg.qr(V)[0]
    else:
        V = V / n ** 0.5
    V = V.float().contiguous()
    lam = torch.exp(torch.randn(k, device="cuda", dtype=torch.float64, generator=g)).sort(descending=True).values
    plan = G.SparsePlan(n, k, 0, n, mode=0, topk=t, symmetric=sym)
    G.set_timing(True)
    plan.run(V, lam)
    plan.run(V, lam)
    ms = G.last_timing()
    st = G.last_stats()
    print(f"n={n} k={k} sym={sym} ortho={ortho} dbg={os.environ.get('GGM_DEBUG_EPI','0')}: prep {ms[0]:.2f} main {ms[1]:.2f} merge {ms[2]:.2f} ms | "
          f"{st} cand/row={st['candidates']/n:.1f}", flush=True)

for args in [(200_000, 64), (1_000_000, 100)]:
    for sym in (2, 1):
        run(*args, sym=sym, ortho=True)
