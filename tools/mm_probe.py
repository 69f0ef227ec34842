import ctypes as C, numpy as np, torch, sys
sys.path.insert(0, ".")
import oracle as O
import paper_2407_19892_b200 as G
from paper_2407_19892_b200._ggm import lib, SolveOpts, SolveInfo, _ptr, _stream
rng = np.random.default_rng(0)
X1 = rng.standard_normal((30, 40)).astype(np.float32)
X2 = (0.5 * rng.standard_normal((25, 40))).astype(np.float32)
X3 = rng.standard_normal((10, 12, 40)).astype(np.float32)
T, mods, ks = [X1,X2,X3], [[0, 1], [2, 1], [3, 4, 1]], [30, 40, 25, 10, 12]
E = [O.gram_eig_multi(T, mods, a, ks[a])[1] for a in range(5)]
Ed = torch.from_numpy(np.concatenate(E)).cuda()
for mlist in ([[0,1]], [[0,1],[2,1]], [[0,1],[2,1],[3,4,1]]):
    axes_used = sorted(set(a for m in mlist for a in m))
    if axes_used != list(range(len(axes_used))): 
        # restrict to used axes prefix
        pass
    A = max(axes_used)+1
    kk = ks[:A]; Ee = [e for e in E[:A]]
    Edd = torch.from_numpy(np.concatenate(Ee)).cuda()
    for iters in (0, 1, 3):
        ptr=[0]; axes=[]
        for m in mlist: axes += m; ptr.append(len(axes))
        o = SolveOpts(); lib().ggm_solve_opts_default(C.byref(o)); o.max_iter=iters; o.gauge=1; o.tol=1e-30
        lam = torch.empty_like(Edd); info = SolveInfo()
        st = lib().ggm_solve_eigvals_multi(A, (C.c_int*A)(*kk), _ptr(Edd), len(mlist), (C.c_int*len(ptr))(*ptr), (C.c_int*len(axes))(*axes), C.byref(o), _ptr(lam), C.byref(info), _stream())
        torch.cuda.synchronize()
        lam_np = [1/e for e in Ee]
        for _ in range(iters):
            g = O.marginals_multi(lam_np, mlist); lam_np = [l*gg/e for l,gg,e in zip(lam_np,g,Ee)]
        got = np.split(lam.cpu().numpy(), np.cumsum(kk)[:-1])
        err = max(float(np.max(np.abs(a-b)/np.abs(b))) for a,b in zip(got, lam_np))
        print(mlist, "iters", iters, "status", st, "res", info.stationarity, "np res", O.stationarity_multi(Ee, lam_np, mlist), "relerr", err)
