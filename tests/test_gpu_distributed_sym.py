"""Distributed symmetric scheme (include/ggm.h (3b)) on one GPU with simulated ranks: every
rank's share (ggm_sparse_precision_sym_shard), the all-to-all done in-process (bucket d of
every rank -> rank d), each rank's merge (ggm_sym_merge) and the final scatter must equal the
single-call symmetric result bitwise (the same block-pair tiles with the same operand roles,
so identical MMA values; the merge order is the total order (|ψ| desc, j asc)), and the
oracle's top-t."""
import numpy as np
import pytest
import torch

from synth import gen
from parity_util import check_topk

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def G():
    import paper_2407_19892_b200 as G
    assert torch.cuda.is_available()
    assert G.device_supported(), "needs an sm_100a (B200) device"
    return G


def _simulate(G, V, lam, t, P, seeded=False, same_plans=False):
    """same_plans: every rank seeds and runs on ONE workspace (as bench.py and parallel.py
    do), so the seeded call reuses the seed call's scale, norms and norm order."""
    n, k = V.shape
    thr_all = None
    plans = [G.SymShardPlan(n, k, t, r, P) for r in range(P)] if same_plans else None
    if seeded:  # sharded seed pass: every rank's share, combined by an element-wise minimum
        parts = [(plans[r] if same_plans else G.SymShardPlan(n, k, t, r, P)).seed(V, lam).clone()
                 for r in range(P)]
        thr_all = torch.stack(parts).min(dim=0).values
        for r, part in enumerate(parts):
            assert torch.isinf(part).any() or P == 1
    shards = []
    for r in range(P):
        plan = plans[r] if same_plans else G.SymShardPlan(n, k, t, r, P)
        key, val, counts, perm = plan.run(V, lam, thr_all=thr_all)
        torch.cuda.synchronize()
        shards.append((key.clone(), val.clone(), counts, perm.clone()))
    perm = shards[0][3]
    for _, _, _, p in shards[1:]:
        assert torch.equal(p, perm), "replicated phases must give the same permutation"
    rows = []
    for d in range(P):
        ks, vs = [], []
        for key, val, counts, _ in shards:
            off = sum(counts[:d])
            ks.append(key[off:off + counts[d]])
            vs.append(val[off:off + counts[d]])
        rk, rv = torch.cat(ks), torch.cat(vs)
        b, e = G.sym_rows_begin(n, k, t, d, P), G.sym_rows_begin(n, k, t, d + 1, P)
        assert torch.all((rk >= b) & (rk < e)), "bucket holds rows of another rank"
        rows.append(G.sym_merge(n, t, rk, rv, perm, b, e))
    te = min(t, n - 1)
    row_id = torch.cat([r[0] for r in rows])
    col = torch.cat([r[1] for r in rows]).view(-1, te)
    val = torch.cat([r[2] for r in rows]).view(-1, te)
    assert torch.equal(torch.sort(row_id).values, torch.arange(n, device=row_id.device))
    fc = torch.empty_like(col)
    fv = torch.empty_like(val)
    fc[row_id] = col
    fv[row_id] = val
    return fc.view(-1).cpu().numpy(), fv.view(-1).cpu().numpy()


@pytest.mark.parametrize("n,k,t,P", [(3000, 64, 10, 2), (5000, 100, 10, 3), (2600, 48, 5, 5),
                                     (20000, 100, 16, 8), (700, 32, 10, 1)])
@pytest.mark.parametrize("seeded", [False, True])
def test_simulated_ranks_equal_single_call(G, n, k, t, P, seeded):
    V, lam = gen.small_factor(4000 + n + P, n, k)
    Vd = torch.from_numpy(V).cuda()
    ld = torch.from_numpy(np.asarray(lam, np.float64)).cuda()
    rp, c, v = G.ggm_sparse_precision(Vd, ld, 0, n, mode=0, topk=t, symmetric=1)
    torch.cuda.synchronize()
    assert G.last_stats()["scheme"] == "symmetric"
    c, v = c.cpu().numpy(), v.cpu().numpy()
    c2, v2 = _simulate(G, Vd, ld, t, P, seeded)
    assert np.array_equal(c, c2)
    np.testing.assert_array_equal(v, v2)
    te = min(t, n - 1)
    rows = np.arange(n) if n <= 5000 else np.arange(0, n, 17)
    prp = np.arange(0, (len(rows) + 1) * te, te)
    pc = np.concatenate([c2[i * te:(i + 1) * te] for i in rows])
    pv = np.concatenate([v2[i * te:(i + 1) * te] for i in rows])
    res = check_topk(prp, pc, pv, V, lam, rows, t)
    assert res["exact"] + res["excused"] == len(rows)


def test_rows_begin_partition(G):
    n, k, t = 1_000_000, 100, 10
    for P in (1, 2, 4, 8):
        b = [G.sym_rows_begin(n, k, t, r, P) for r in range(P + 1)]
        assert b[0] == 0 and b[-1] == n and all(x <= y for x, y in zip(b, b[1:]))
        assert all(x % 256 == 0 for x in b[:-1])


@pytest.mark.parametrize("assign", ["part", "strided"])
@pytest.mark.parametrize("P", [2, 4, 8])
def test_unit_assignments_equal_single_call(G, monkeypatch, assign, P):
    """Both shares of the block-pair units (folded part-major: sub-windows j and 7 - j of every
    row block for the pairs j owned by the rank, the default when P divides the sub-window
    count; rank-strided units r, r + P, ..., GGM_SYM_ASSIGN=strided) cover every unit exactly
    once: bitwise the single call (P = 8 is in test_simulated_ranks_equal_single_call)."""
    n, k, t = 6000, 64, 10
    if assign == "strided":
        monkeypatch.setenv("GGM_SYM_ASSIGN", "strided")
    V, lam = gen.small_factor(77 + P, n, k)
    Vd = torch.from_numpy(V).cuda()
    ld = torch.from_numpy(np.asarray(lam, np.float64)).cuda()
    rp, c, v = G.ggm_sparse_precision(Vd, ld, 0, n, mode=0, topk=t, symmetric=1)
    torch.cuda.synchronize()
    c2, v2 = _simulate(G, Vd, ld, t, P, seeded=True)
    assert np.array_equal(c.cpu().numpy(), c2)
    np.testing.assert_array_equal(v.cpu().numpy(), v2)


@pytest.mark.parametrize("P", [2, 8])
def test_seeded_call_reusing_the_seed_workspace(G, P):
    """The seeded shard call on the workspace of the same rank's seed call (same V, λ) reuses
    its scale, row norms and norm order: bitwise the single call."""
    n, k, t = 20000, 100, 10
    V, lam = gen.small_factor(555 + P, n, k)
    Vd = torch.from_numpy(V).cuda()
    ld = torch.from_numpy(np.asarray(lam, np.float64)).cuda()
    rp, c, v = G.ggm_sparse_precision(Vd, ld, 0, n, mode=0, topk=t, symmetric=1)
    torch.cuda.synchronize()
    c2, v2 = _simulate(G, Vd, ld, t, P, seeded=True, same_plans=True)
    assert np.array_equal(c.cpu().numpy(), c2)
    np.testing.assert_array_equal(v.cpu().numpy(), v2)
