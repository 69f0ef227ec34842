"""Gram-spectrum timings on C2 / C3 (for GGM_GRAM_SYRK A/B)."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2407_19892_b200 as G
from synth import gen
tag = os.environ.get("GGM_GRAM_SYRK") and "syrk" or "default"
for name in ("C2", "C3"):
    cfg = gen.config(name)
    X = torch.from_numpy(cfg["X"]).cuda()
    out = []
    for a, k in enumerate(cfg["k"]):
        G.ggm_gram_eig(X, a, k); torch.cuda.synchronize()
        best = 1e9
        for _ in range(3):
            t0 = time.perf_counter(); G.ggm_gram_eig(X, a, k); torch.cuda.synchronize()
            best = min(best, (time.perf_counter() - t0) * 1e3)
        out.append(round(best, 2))
    if name == "C2":
        G.ggm_gram_eig_matrix(X, *cfg["k"]); torch.cuda.synchronize()
        t0 = time.perf_counter(); G.ggm_gram_eig_matrix(X, *cfg["k"]); torch.cuda.synchronize()
        out.append(("matrix", round((time.perf_counter() - t0) * 1e3, 2)))
    print(tag, name, out, flush=True)
