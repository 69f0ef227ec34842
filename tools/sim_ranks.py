"""Per-rank work of the multi-GPU C5 step, measured on ONE GPU by running every rank's share
in turn (no rank waits on another): axis A (n = 10^6) distributed symmetric scheme = sharded
seed pass + this rank's block pairs + merge of its rows; axis B (n = 30,000) plain row shards.
Prints, per N, the max-over-ranks compute time and a projected step time = that + the
collectives' bytes at an assumed NVLink/NCCL bus bandwidth (a projection, not a measurement of
N GPUs: DESIGN.md §5).  Usage: python tools/sim_ranks.py [N ...] [--symB]  (--symB: axis B by the distributed
symmetric scheme too at N > 1)"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2407_19892_b200 as G  # noqa: E402
from paper_2407_19892_b200.parallel import shard_rows  # noqa: E402
from synth import gen  # noqa: E402

BUS_GBS = 600.0      # assumed effective NCCL bus bandwidth per GPU over NVLink 5 (GB/s)
LAT_MS = 0.03        # assumed per-collective latency


def ev_ms(fn, reps=3):
    best = 1e30
    out = None
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        out = fn()
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    return best, out


def main():
    Ns = [int(x) for x in sys.argv[1:] if x.isdigit()] or [1, 2, 4, 8]
    cfg = gen.config("C5")
    t = cfg["t"]
    (VA, lA), (VB, lB) = [(torch.from_numpy(V).cuda(), torch.from_numpy(l).cuda())
                          for V, l in cfg["axes"]]
    nA, k = VA.shape
    nB = VB.shape[0]
    res = {}
    symB = "--symB" in sys.argv   # axis B by the distributed symmetric scheme as well

    def sym_axis(V, lam, N):
        """Per-rank seed / units / merge times (ms) of the distributed symmetric scheme."""
        n = V.shape[0]
        seeds, runs, merges, plans, shards = [], [], [], [], []
        for r in range(N):
            plans.append(G.SymShardPlan(n, k, t, r, N))
        parts = []
        for r in range(N):
            ms, thr = ev_ms(lambda: plans[r].seed(V, lam).clone())
            seeds.append(ms)
            parts.append(thr)
        thr_all = torch.stack(parts).min(dim=0).values
        del parts
        ncand, stages = [], []
        G.set_timing(True)
        for r in range(N):
            best, out, st_best = 1e30, None, None
            for _ in range(3):
                # as in bench.py: this rank's seed call precedes its seeded call on the same
                # workspace (the seeded call then reuses the seed call's norm pass)
                plans[r].seed(V, lam)
                ms, o = ev_ms(lambda: plans[r].run(V, lam, thr_all=thr_all), reps=1)
                if ms < best:
                    best, out, st_best = ms, o, [round(x, 3) for x in G.last_timing()]
            runs.append(best)
            stages.append(st_best)
            key, val, counts, perm = out
            shards.append((key.clone(), val.clone(), list(counts), perm))
            ncand.append(int(sum(counts)))
        for d in range(N):
            ks, vs = [], []
            for key, val, counts, _ in shards:
                off = sum(counts[:d])
                ks.append(key[off:off + counts[d]])
                vs.append(val[off:off + counts[d]])
            rk, rv = torch.cat(ks), torch.cat(vs)
            b, e = G.sym_rows_begin(n, k, t, d, N), G.sym_rows_begin(n, k, t, d + 1, N)
            ms, _ = ev_ms(lambda: G.sym_merge(n, t, rk, rv, shards[0][3], b, e))
            merges.append(ms)
        del shards
        torch.cuda.empty_cache()
        return seeds, runs, merges, ncand, stages

    for N in Ns:
        seeds, runs, merges, ncand, stages = sym_axis(VA, lA, N)
        rowsB, ncB = [], [0]
        if symB and N > 1:
            sB, rB, mB, ncB, _ = sym_axis(VB, lB, N)
            rowsB = [a + b + c for a, b, c in zip(sB, rB, mB)]
        else:
            for r in range(N):
                b, e = shard_rows(nB, N, r)
                p = G.SparsePlan(nB, k, b, e, topk=t)
                ms, _ = ev_ms(lambda: p.run(VB, lB))
                rowsB.append(ms)
        perA = [a + b + c for a, b, c in zip(seeds, runs, merges)]
        comp = max(perA) + max(rowsB)
        # collectives per step at N > 1: all-reduce(MIN) of nA floats, all-to-all of the
        # candidates (12 B each, (N-1)/N of them leave the rank), all-gather of both CSRs
        if N > 1:
            byt = [4.0 * nA * 2 * (N - 1) / N,
                   12.0 * max(ncand) * (N - 1) / N,
                   (8.0 * nA * t + 8.0 * nA) * (N - 1) / N,
                   8.0 * nB * t * (N - 1) / N]
            if symB:  # axis B's seed all-reduce and candidate all-to-all
                byt += [4.0 * nB * 2 * (N - 1) / N, 12.0 * max(ncB) * (N - 1) / N]
            comm = sum(b / (BUS_GBS * 1e9) * 1e3 + LAT_MS for b in byt)
        else:
            comm = 0.0
        res[N] = {"axisA_seed_ms": seeds, "axisA_units_ms": runs, "axisA_merge_ms": merges,
                  "axisB_rows_ms": rowsB, "max_rank_compute_ms": comp,
                  "projected_comm_ms": comm, "projected_step_ms": comp + comm,
                  "candidates_per_rank": ncand, "axisA_stages_prep_main_tail_ms": stages}
        print(json.dumps({"N": N, **res[N]}), flush=True)
    if 1 in res:
        t1 = res[1]["projected_step_ms"]
        for N in res:
            print(json.dumps({"N": N, "projected_efficiency_vs_N1":
                              t1 / (N * res[N]["projected_step_ms"])}), flush=True)


if __name__ == "__main__":
    main()
