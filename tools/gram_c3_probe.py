"""Launch-list probe of ggm_gram_eig on C3 (400 x 300 x 200): which kernels take the time."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2407_19892_b200 as G
from synth import gen
cfg = gen.config("C3")
X = torch.from_numpy(cfg["X"]).cuda()
for rep in range(3):
    for a, k in enumerate(cfg["k"]):
        torch.cuda.synchronize(); t0 = time.perf_counter()
        G.ggm_gram_eig(X, a, k)
        torch.cuda.synchronize()
        print(f"rep {rep} axis {a}: {(time.perf_counter() - t0) * 1e3:.2f} ms", flush=True)
