"""Passes / time of ggm_solve_eigvals per method on C1-C3 (BK4), plus one
isolated C3 solve for an ncu capture (--ncu: run the C3 solve once after a warm-up)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2407_19892_b200 as G  # noqa: E402
from synth import gen  # noqa: E402

names = () if "--pass" in sys.argv else ("C3",) if "--ncu" in sys.argv else ("C1", "C2", "C3")
for name in names:
    cfg = gen.config(name)
    X = torch.from_numpy(cfg["X"]).cuda()
    Ec = torch.cat([G.ggm_gram_eig(X, a, k)[1] for a, k in enumerate(cfg["k"])])
    for method in ((0,) if "--ncu" in sys.argv else (0, 1)):
        lam, info = G.ggm_solve_eigvals(Ec, cfg["k"], method=method)
        torch.cuda.synchronize()
        if "--ncu" in sys.argv:
            break
        ms = 1e9
        for _ in range(5):
            t0 = time.perf_counter()
            lam, info = G.ggm_solve_eigvals(Ec, cfg["k"], method=method)
            torch.cuda.synchronize()
            ms = min(ms, (time.perf_counter() - t0) * 1e3)
        pts = 1.0
        for k in cfg["k"]:
            pts *= k
        print(f"{name} method={method}: passes/it={info['iterations']} ms={ms:.3f} "
              f"stat={info['stationarity']:.2e} us/pass={ms * 1e3 / max(info['iterations'], 1):.2f} "
              f"points/s/pass={pts * max(info['iterations'], 1) / (ms * 1e-3):.3e}", flush=True)

if "--pass" in sys.argv:
    # one stand-alone grid pass (ggm_grid_marginals: pass kernel + partial reduction, no grid
    # barrier, no update) at the C3 solution, CUDA events, best of 20: the per-pass cost of
    # the in-solve pass minus this is the barrier / reduction / update overhead
    cfg = gen.config("C3")
    X = torch.from_numpy(cfg["X"]).cuda()
    Ec = torch.cat([G.ggm_gram_eig(X, a, k)[1] for a, k in enumerate(cfg["k"])])
    lam, info = G.ggm_solve_eigvals(Ec, cfg["k"])
    best = 1e9
    for _ in range(20):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        G.ggm_grid_marginals(lam, cfg["k"])
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    print(f"C3 stand-alone pass: {best * 1e3:.1f} us; in-solve kernel: {info['kernel_ms']:.3f} ms "
          f"over {info['passes']} passes = {info['kernel_ms'] * 1e3 / info['passes']:.1f} us/pass",
          flush=True)
