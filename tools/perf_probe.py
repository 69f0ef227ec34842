"""Timing probe of ggm_sparse_precision on C4/C5-shaped random factors (device-generated)."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2407_19892_b200 as G

def probe(n, k, t=10, reps=3, chunks=0):
    g = torch.Generator(device="cuda").manual_seed(0)
    V = (torch.randn(n, k, device="cuda", generator=g) / n ** 0.5).float().contiguous()
    lam = torch.exp(torch.randn(k, device="cuda", dtype=torch.float64, generator=g)).sort(descending=True).values
    plan = G.SparsePlan(n, k, 0, n, mode=0, topk=t, col_chunks=chunks)
    G.set_timing(True)
    plan.run(V, lam)
    best = None
    for _ in range(reps):
        torch.cuda.synchronize(); t0 = time.time()
        plan.run(V, lam)
        wall = time.time() - t0
        ms = G.last_timing()
        if best is None or ms[1] < best[1][1]:
            best = (wall, ms)
    wall, ms = best
    ent = n * n
    kpad = (k + 15) // 16 * 16
    tflops_alg = 2 * k * ent / (ms[1] * 1e-3) / 1e12
    tflops_hw = 3 * 2 * kpad * ent / (ms[1] * 1e-3) / 1e12
    print(f"n={n} k={k} t={t} chunks={chunks}: prep {ms[0]:.3f} ms fused {ms[1]:.3f} ms merge {ms[2]:.3f} ms "
          f"wall {wall*1e3:.1f} ms | {ent/(ms[1]*1e-3):.3e} entries/s | alg {tflops_alg:.1f} TF/s "
          f"(frac of 1623.7/3={tflops_alg/(1623.7/3):.3f}) | TC {tflops_hw:.1f} TF/s", flush=True)

for args in ([] if "--solve-only" in sys.argv else [(200_000, 64), (30_000, 100), (1_000_000, 100)]):
    probe(*args)

def probe_solve(ks, seed=0):
    import numpy as np
    rng = np.random.default_rng(seed)
    T = 1000.0
    E = np.concatenate([np.sort(T / k * rng.uniform(0.5, 1.5, k))[::-1] for k in ks])
    # equalise traces (reading T)
    off = np.cumsum([0] + list(ks))
    for a in range(len(ks)):
        E[off[a]:off[a+1]] *= T / E[off[a]:off[a+1]].sum()
    Ed = torch.from_numpy(E).cuda()
    G.ggm_solve_eigvals(Ed, ks, tol=1e-7)
    torch.cuda.synchronize(); t0 = time.time()
    lam, info = G.ggm_solve_eigvals(Ed, ks, tol=1e-7)
    dt = time.time() - t0
    pts = float(np.prod(ks))
    print(f"solve ks={ks}: {dt*1e3:.2f} ms, {info['iterations']} it, {dt/max(info['iterations'],1)*1e6:.1f} us/it, "
          f"{pts*max(info['iterations'],1)/dt:.3e} grid pts/s, res {info['stationarity']:.2e}", flush=True)
    g = torch.cat([torch.full((k,), 0.5, dtype=torch.float64) for k in ks]).cuda()
    G.ggm_grid_marginals(g, ks); torch.cuda.synchronize(); t0 = time.time()
    for _ in range(10): G.ggm_grid_marginals(g, ks)
    torch.cuda.synchronize(); dt = (time.time() - t0) / 10
    print(f"   single marginal pass (incl. alloc+reduce): {dt*1e6:.1f} us = {pts/dt:.3e} pts/s", flush=True)

for ks in ([] if "--sparse-only" in sys.argv else [(400, 300, 200), (100, 100), (50, 50)]):
    probe_solve(ks)
