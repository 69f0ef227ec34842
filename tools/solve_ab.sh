# same-session A/B of solve-kernel variants: C3 method-0 kernel time (ggm_solve_info.kernel_ms)
cat > /tmp/sab.py <<'PY'
import os, sys
sys.path.insert(0, os.getcwd())
import torch, paper_2407_19892_b200 as G
from synth import gen
cfg = gen.config("C3")
X = torch.from_numpy(cfg["X"]).cuda()
Ec = torch.cat([G.ggm_gram_eig(X, a, k)[1] for a, k in enumerate(cfg["k"])])
best = 1e9
for _ in range(6):
    lam, info = G.ggm_solve_eigvals(Ec, cfg["k"], method=0)
    best = min(best, info["kernel_ms"])
print(f"[{os.path.basename(os.environ.get('GGM_LIB_PATH','base'))}] C3 kernel {best:.3f} ms passes {info['passes']}", flush=True)
PY
for i in 1 2; do
  timeout 120 python /tmp/sab.py
  for v in $VARS; do GGM_LIB_PATH=tools/variants/$v.so timeout 120 python /tmp/sab.py; done
done
