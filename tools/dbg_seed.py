import os, sys, numpy as np, torch
sys.path.insert(0, os.getcwd())
import paper_2407_19892_b200 as G
from synth import gen
n, k, t = 3000, 64, int(os.environ.get("T", "3"))
V, lam = gen.small_factor(n + 3 * k + 3, n, k)
Vd = torch.from_numpy(V).cuda(); ld = torch.from_numpy(np.asarray(lam, np.float64)).cuda()
os.environ["GGM_DEBUG_RAW"] = "gpurun_out/raw.bin"
G.ggm_sparse_precision(Vd, ld, 0, n, mode=0, topk=t, symmetric=1); torch.cuda.synchronize()
raw = np.fromfile("gpurun_out/raw.bin", dtype=np.float32)
U = V.astype(np.float64) * np.sqrt(lam); P = np.abs(U @ U.T); np.fill_diagonal(P, 0)
mx = np.abs(U).max(); e = 14 - np.frexp(mx)[1]; raw = raw / 2.0 ** (2 * e)
SS = 8; NT = 12; rk = []; bad = []
for i in range(n):
    cols = np.concatenate([np.arange(256 * j, min(256 * j + 256, n)) for j in range((i // 128) % SS, NT, SS)])
    a = P[i, cols]; cmu = np.array([a[q:q + 32].max() for q in range(0, len(a), 32)]); cm = np.sort(cmu)[::-1]
    r = int(np.argmin(np.abs(cm - raw[i]))); rk.append(r + 1)
    if r + 1 != t and len(bad) < 4:
        # where is that value: which chunk (tile, half)?
        ch = int(np.argmin(np.abs(cmu - raw[i])))
        bad.append((i, r + 1, abs(cm[r] - raw[i]) / raw[i], ch, np.round(cm[:t + 2], 6), np.argsort(-cmu)[:t + 2]))
rk = np.array(rk)
print(f"dbg={os.environ.get('GGM_DEBUG_EPI','0')} t={t}: rank of GPU seed among chunk maxima:", np.bincount(rk)[:12])
for b in bad: print("  ", b)
