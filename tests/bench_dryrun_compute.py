"""Per-shard compute injected into `bench.py --dry-run` (tests/test_bench_launcher.py): the
plain definition of a row block of thresh_t[V diag(λ) V^T] with torch CPU ops (dense rows,
diagonal excluded, top-t by |ψ| with ties to the smaller column, ascending columns).  Test
infrastructure: the launcher test checks the gathered result against the oracle."""
import torch


def compute(V, lam, begin, end, t):
    n = V.shape[0]
    te = min(t, n - 1)
    P = (V[begin:end].double() * lam.double()) @ V.double().T
    rows = torch.arange(begin, end)
    a = P.abs()
    a[torch.arange(end - begin), rows] = -1.0
    # stable order by (-|ψ|, j): sort columns descending by magnitude, stable on ties
    order = torch.sort(-a, dim=1, stable=True).indices[:, :te]
    cols = torch.sort(order, dim=1).values
    vals = torch.gather(P, 1, cols)
    rp = torch.arange(0, (end - begin + 1) * te, te, dtype=torch.int64)
    return rp, cols.reshape(-1).to(torch.int32), vals.reshape(-1).to(torch.float32)
