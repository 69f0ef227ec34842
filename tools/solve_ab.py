"""C3 eigenvalue-MLE kernel time (ggm_solve_info.kernel_ms, CUDA events in libggm), best of
10 calls, for A/B of library variants (GGM_LIB_PATH) in one session."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2407_19892_b200 as G  # noqa: E402
from synth import gen  # noqa: E402

tag = os.environ.get("TAG", os.path.basename(os.environ.get("GGM_LIB_PATH", "base")))
cfg = gen.config("C3")
X = torch.from_numpy(cfg["X"]).cuda()
Ec = torch.cat([G.ggm_gram_eig(X, a, k)[1] for a, k in enumerate(cfg["k"])])
best, info = 1e9, None
if not os.environ.get("FIXED_PASSES"):
    for _ in range(10):
        lam, info = G.ggm_solve_eigvals(Ec, cfg["k"])
        best = min(best, info["kernel_ms"])
    print(f"[{tag}] C3 solve kernel {best:.4f} ms, {info['passes']} passes, "
          f"{best * 1e3 / info['passes']:.2f} us/pass", flush=True)

if os.environ.get("FIXED_PASSES"):
    # fixed pass count (tol 1e-300, plain MM step, max_iter passes): time per pass from CUDA events
    # around the call (the call raises GGM_ERR_NO_CONVERGENCE at the end)
    npass = int(os.environ["FIXED_PASSES"])
    best = 1e9
    for _ in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        try:
            G.ggm_solve_eigvals(Ec, cfg["k"], tol=1e-300, max_iter=npass, method=1)
        except G.GGMError:
            pass
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    print(f"[{tag}] C3 {npass} fixed passes: {best:.3f} ms call, {best * 1e3 / npass:.2f} us/pass",
          flush=True)
