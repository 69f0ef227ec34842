"""GPU parity at the full BASELINE.json configurations (BJ:7-11), through the C ABI, in the
launch configuration bench.py times.  Large configs compare sampled rows one by one
against the oracle (rows are independent, so sampled-row parity is exact parity for those
rows); row-shard invariance is checked bitwise by simulated ranks (disjoint row-range calls
concatenated == one call), as SURVEY §4 prescribes for the multi-GPU path."""
import numpy as np
import pytest
import torch

import oracle as O
from synth import gen
from parity_util import assert_exact_fraction, check_topk

pytestmark = pytest.mark.gpu

EIG_REL = 1e-5


@pytest.fixture(scope="module")
def G():
    import paper_2407_19892_b200 as G
    assert G.device_supported()
    return G


def _sample_rows(n, m, seed, extra=()):
    rng = np.random.default_rng(seed)
    rows = set(rng.choice(n, size=min(m, n), replace=False).tolist())
    rows.update(r for r in extra if 0 <= r < n)
    return np.array(sorted(rows), dtype=np.int64)


def _csr_rows(rp, col, val, rows):
    prp = [0]
    pc, pv = [], []
    for i in rows:
        pc.append(col[rp[i]:rp[i + 1]])
        pv.append(val[rp[i]:rp[i + 1]])
        prp.append(prp[-1] + rp[i + 1] - rp[i])
    return np.array(prp), np.concatenate(pc), np.concatenate(pv)


def _pipeline_gpu(G, X, ks):
    Xd = torch.from_numpy(X).cuda()
    Vs, Es = [], []
    for a, k in enumerate(ks):
        V, E, _ = G.ggm_gram_eig(Xd, a, k)
        Vs.append(V)
        Es.append(E)
    lam, info = G.ggm_solve_eigvals(torch.cat(Es), ks)
    return Vs, Es, list(torch.split(lam, list(ks))), info


def _pipeline_oracle(X, ks):
    Vo, Eo = zip(*[O.gram_eig(X, a, k) for a, k in enumerate(ks)])
    lo, info = O.solve_eigvals(list(Eo), tol=1e-12)
    return list(Vo), list(Eo), lo, info


@pytest.mark.parametrize("name,rows_per_axis", [("C1", None), ("C2", 1500), ("C3", None)])
def test_data_config_pipeline(G, name, rows_per_axis):
    """C1-C3: gram_eig -> solve_eigvals -> sparse_precision per axis vs the oracle pipeline."""
    cfg = gen.config(name)
    X, ks, t = cfg["X"], cfg["k"], cfg["t"]
    Vs, Es, lams, info = _pipeline_gpu(G, X, ks)
    Vo, Eo, lo, oinfo = _pipeline_oracle(X, ks)
    assert info["stationarity"] <= 1e-7
    for a in range(len(ks)):
        np.testing.assert_allclose(Es[a].cpu().numpy(), Eo[a], rtol=1e-9)
    # eigenvalues: gauge-free grid sums and the canonical gauge-0 λ, 1e-5 relative
    lg = [l.cpu().numpy() for l in lams]
    np.testing.assert_allclose(O.grid_sums(lg), O.grid_sums(lo), rtol=EIG_REL)
    for a in range(len(ks)):
        np.testing.assert_allclose(lg[a], lo[a], rtol=EIG_REL)
    # sparse graphs: the GPU path's own V, λ; the oracle recomposes from its fp64 spectrum
    for a in range(len(ks)):
        n = X.shape[a]
        rp, col, val = G.ggm_sparse_precision(Vs[a], lams[a].contiguous(), 0, n, topk=t)
        rp, col, val = rp.cpu().numpy(), col.cpu().numpy(), val.cpu().numpy()
        rows = np.arange(n) if rows_per_axis is None else _sample_rows(n, rows_per_axis, a,
                                                                       (0, n - 1))
        prp, pc, pv = _csr_rows(rp, col, val, rows)
        # C1/C3 (values O(1e-2..0.6)): the strict relative-only gate; C2's 3e-4 eigengaps
        # carry the fp32 spectrum's rounding into ψ at ~1e-5 relative (the GPU pipeline's own
        # V vs the oracle's fp64 V), so C2 keeps the literal gate here and is held to the
        # strict gate kernel-level in test_c2_kernel_strict
        st = check_topk(prp, pc, pv, Vo[a], lo[a], rows, t, strict=name != "C2")
        assert st["exact"] + st["excused"] == len(rows)
        assert_exact_fraction(st, 0.99 if name != "C2" else 0.9, f"{name} axis {a}")


def _shard_sample(n, P, per_shard, seed):
    """Rows of every P-way shard: per_shard random rows plus each shard's first and last row,
    and the 256-row tile boundaries (b·256 - 1, b·256) that fall in the sample's shards."""
    from paper_2407_19892_b200.parallel import shard_rows
    rng = np.random.default_rng(seed)
    rows = set()
    for r in range(P):
        b, e = shard_rows(n, P, r)
        rows.update(rng.choice(np.arange(b, e), size=min(per_shard, e - b), replace=False).tolist())
        rows.update((b, e - 1))
        for tb in range((b + 255) // 256 * 256, e, 256 * 37):   # every 37th tile boundary
            rows.update((tb - 1, tb))
    return np.array(sorted(x for x in rows if 0 <= x < n), dtype=np.int64)


@pytest.mark.parametrize("name", ["C4", "C5"])
def test_factor_config_sampled_rows_and_shards(G, name):
    """C4/C5 at full size in the bench's launch configuration (automatic scheme: the
    symmetric screening scheme for the large axes): sampled rows vs the oracle with the
    strict relative-only gate and the exact-match fraction (reading TOL; §8(c) c3: C5 axis A
    8,192 rows = 1,024 per 8-way shard incl. shard and tile boundaries, axis B all 30,000
    rows), and simulated ranks (P disjoint row ranges, plain scheme) bitwise equal to the
    single plain call."""
    cfg = gen.config(name)
    t = cfg["t"]
    from paper_2407_19892_b200.parallel import shard_rows
    for ax, (V, lam) in enumerate(cfg["axes"]):
        n, k = V.shape
        Vd = torch.from_numpy(V).cuda()
        ld = torch.from_numpy(lam).cuda()
        plan = G.SparsePlan(n, k, 0, n, topk=t)
        plan.run(Vd, ld)
        rp = plan.row_ptr.cpu().numpy()
        col = plan.col.cpu().numpy()
        val = plan.val.cpu().numpy()
        if n <= 30_000:
            rows = np.arange(n)
        else:
            rows = _shard_sample(n, 8, 1024 if name == "C5" else 512, 7 + ax)
        prp, pc, pv = _csr_rows(rp, col, val, rows)
        st = check_topk(prp, pc, pv, V, lam, rows, t, strict=True)
        assert st["exact"] + st["excused"] == len(rows)
        assert_exact_fraction(st, 0.999, f"{name} axis {ax}")
        assert st["max_rel_err"] <= 1e-5, st
        # simulated ranks: concatenated row shards (plain scheme) == one plain full-axis call,
        # bitwise (the automatic full-axis call above may use the symmetric scheme, whose
        # transposed-direction entries accumulate the two cross-term MMAs in swapped order)
        ref = G.SparsePlan(n, k, 0, n, topk=t, symmetric=2)
        ref.run(Vd, ld)
        col, val = ref.col.cpu().numpy(), ref.val.cpu().numpy()
        for P in (2, 8):
            cols, vals = [], []
            for r in range(P):
                b, e = shard_rows(n, P, r)
                sp = G.SparsePlan(n, k, b, e, topk=t)
                sp.run(Vd, ld)
                cols.append(sp.col.cpu().numpy())
                vals.append(sp.val.cpu().numpy())
            assert np.array_equal(np.concatenate(cols), col)
            assert np.array_equal(np.concatenate(vals), val)


@pytest.mark.parametrize("axis", [0, 1])
def test_c2_kernel_strict(G, axis):
    """C2 (10,000 cells x 2,000 genes, k = 50, t = 10; BJ:8): the sparse kernel on the
    oracle's spectrum (fp32 V, the same bits on both sides) over ALL rows of the axis, strict
    relative-only gate and exact-match fraction (reading TOL: the literal 1e-6 floor excuses
    every cell-axis row at C2 magnitudes, so it is not the gate here)."""
    cfg = gen.config("C2")
    X, ks, t = cfg["X"], cfg["k"], cfg["t"]
    Vo, Eo = O.gram_eig(X, axis, ks[axis])
    _, Eother = O.gram_eig(X, 1 - axis, ks[1 - axis])
    lo, _ = O.solve_eigvals([Eo, Eother] if axis == 0 else [Eother, Eo], tol=1e-12)
    V = Vo.astype(np.float32)
    lam = lo[axis]
    n = V.shape[0]
    rp, col, val = G.ggm_sparse_precision(torch.from_numpy(V).cuda(), torch.from_numpy(lam).cuda(),
                                          0, n, topk=t)
    st = check_topk(rp.cpu().numpy(), col.cpu().numpy(), val.cpu().numpy(), V, lam,
                    np.arange(n), t, strict=True)
    assert st["exact"] + st["excused"] == n
    assert_exact_fraction(st, 0.999, f"C2 axis {axis}")
