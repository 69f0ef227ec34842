#!/bin/bash
# Per-role wait-time breakdown of the BK2 main kernel (variant built with -DGGM_MMA_PROF).
cat > /tmp/mp.py <<'PY'
# MP_N / MP_K select the axis (default C5 axis A; C4: MP_N=200000 MP_K=64)
import sys, os
sys.path.insert(0, os.getcwd())
import torch, paper_2407_19892_b200 as G
n, k = int(os.environ.get('MP_N', 1_000_000)), int(os.environ.get('MP_K', 100))
g = torch.Generator(device="cuda").manual_seed(0)
V = torch.linalg.qr(torch.randn(n, k, device="cuda", generator=g, dtype=torch.float64))[0].float().contiguous()
lam = torch.exp(torch.randn(k, device="cuda", dtype=torch.float64, generator=g)).sort(descending=True).values
plan = G.SparsePlan(n, k, 0, n, mode=0, topk=10, symmetric=1)
G.set_timing(True)
plan.run(V, lam); torch.cuda.synchronize()
print("TIMING", G.last_timing(), flush=True)
PY
for v in ${VARIANTS:-mmaprof mmaprof_dbg}; do
  for d in ${DBGS:-0 1 2}; do
    [ $v = mmaprof ] && [ $d != 0 ] && continue
    echo "== $v dbg=$d"
    GGM_DEBUG_EPI=$d GGM_LIB_PATH=tools/variants/$v.so timeout 120 python /tmp/mp.py 2>&1 | grep -v "^$" | sort | awk '/MMAPROF/ && /cta 0 / || /EPIPROF/ && /cta 0 / || /TIMING/ || /cta 64 /' | head -12
  done
done
