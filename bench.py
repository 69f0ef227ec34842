#!/usr/bin/env python
"""Benchmark of the GmGM hot path (arXiv 2407.19892) on B200: precision entries evaluated +
sparsified per second (n^2 per axis) for the BASELINE.json workload C5 (factor-level axes
n = 1,000,000 and n = 30,000, rank 100, top-10 per row; BJ:11), row-sharded over N GPUs.

    python bench.py [--gpus N --steps K --warmup W] [--impl ours|reference] [--config C5|C4]

--gpus N > 1 without WORLD_SIZE in the environment re-launches this script under
`torch.distributed.run --nnodes=1 --nproc-per-node N --master-addr 127.0.0.1` (one rank per GPU,
NCCL; NCCL_DEBUG=INFO for the communicator lines, on stderr); under torchrun WORLD_SIZE must
equal N.  --dry-run exercises the same launcher and multi-rank plumbing on CPU (gloo) with an
injected per-shard compute function (tests/test_bench_launcher.py); it measures nothing.

A step = one pass of the hot path over the workload: for every axis, ggm_sparse_precision
(BK1 prep/split -> BK2 fused tcgen05 recomposition + top-t -> CSR) on this rank's rows; at
N > 1 also the NCCL all-gather of the CSR shards.  Inputs (V, λ) are resident in HBM when the
timed region starts (replicated by one NCCL broadcast at setup).  The inputs (V 400 MB, the
split operand 512 MB) are larger than L2, so no explicit flush is used.  The e2e arm repeats
the step through the same public API from pinned HOST buffers with H2D/D2H inside the timed
region.  The reference arm (--impl reference) times the fp64 CPU oracle on a bounded row
sample of the same workload (the reference of this tier).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "precision entries evaluated+sparsified/sec (n^2 per axis), % of TC roofline"
UNIT = "entries/s"
DTYPE = ("f16 hi*hi screening (f32 accumulate, thresholds lowered by its error bound) + "
         "f64-accumulated exact re-evaluation of the candidates from the f32 inputs")
WORKLOADS = {
    "C5": "C5: factor-level axes n=1,000,000 and n=30,000 (cell / gene axis of a million-cell "
          "dataset), rank 100, V = QR of N(0,1), lambda ~ LogNormal(0,1), top-10 per row",
    "C4": "C4: factor-level axis n=200,000, rank 64, top-10 per row",
}


def _peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            d = json.load(f)
        return d, "MEASURED_PEAKS.json"
    except Exception:
        return {"bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0, "hbm_gbs": 6650.0}, \
            "fallback (B200_PROFILING.md)"


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled every 200 ms during the timed region."""
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return None
        self.proc.terminate()
        try:
            out, _ = self.proc.communicate(timeout=5)
        except Exception:
            self.proc.kill()
            out = ""
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in out.strip().splitlines():
            f = [x.strip() for x in line.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                mx.append(float(f[2]))
            except ValueError:
                continue
            for nm, v in zip(names, f[5:9]):
                if v.lower() == "active":
                    reasons.add(nm)
        if not sm:
            return None
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


def _free_port():
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _maybe_launch(args):
    """--gpus N > 1 outside torchrun: re-exec under torch.distributed.run (one process per GPU)
    and return its exit code; None when this process is already the (or a) rank."""
    world_env = os.environ.get("WORLD_SIZE")
    if world_env is not None:
        if int(world_env) != args.gpus:
            raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world_env}")
        return None
    if args.gpus <= 1:
        return None
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")
    env.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    env.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")
    env.setdefault("OMP_NUM_THREADS", "1")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr", "127.0.0.1",
           f"--master-port={_free_port()}", os.path.abspath(__file__)] + sys.argv[1:]
    print(f"bench.py: launching {args.gpus} ranks: {' '.join(cmd)}", file=sys.stderr, flush=True)
    return subprocess.call(cmd, env=env)


def _dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def _load_workload(name):
    from synth import gen
    c = gen.config(name)
    return c["axes"], c["t"]


def _load_injected():
    spec = os.environ.get("BENCH_DRYRUN_COMPUTE", "")
    if ":" not in spec:
        raise SystemExit("--dry-run needs BENCH_DRYRUN_COMPUTE=module:function (a CPU per-shard "
                         "compute (V, lam, begin, end, t) -> (row_ptr, col, val))")
    import importlib
    mod, fn = spec.split(":", 1)
    return getattr(importlib.import_module(mod), fn)


def run_dry(args):
    """The launcher and the multi-rank plumbing of a step on CPU (gloo): row shards of two
    synthetic axes through an injected compute function, the CSR gather of parallel.py, the
    barrier + max-over-ranks timing and rank 0's single JSON line.  No number it prints is a
    measurement of this repository's kernels."""
    import torch
    import torch.distributed as dist
    from paper_2407_19892_b200.parallel import gather_topk_csr, shard_rows
    from synth import gen
    world, rank, _ = _dist_env()
    if world > 1:
        dist.init_process_group("gloo")
    compute = _load_injected()
    t = 10
    axes = []
    for seed, n in ((5, args.dry_n), (6, max(args.dry_n // 10, 16))):
        V, lam = gen.small_factor(seed, n, 16)
        axes.append((torch.from_numpy(V), torch.from_numpy(lam)))

    def step():
        out = []
        for V, lam in axes:
            n = V.shape[0]
            b, e = shard_rows(n, world, rank)
            _, col, val = compute(V, lam, b, e, t)
            out.append(gather_topk_csr(col, val, min(t, n - 1), n))
        return out

    for _ in range(args.warmup):
        step()
    if world > 1:
        dist.barrier()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        res = step()
    dt = time.perf_counter() - t0
    tt = torch.tensor([dt], dtype=torch.float64)
    if world > 1:
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
    ms = float(tt.item()) / max(args.steps, 1) * 1e3
    if rank == 0:
        dump = os.environ.get("BENCH_DRYRUN_DUMP")
        if dump:
            np.savez(dump, **{f"{w}{a}": x.numpy() for a, r in enumerate(res)
                              for w, x in zip(("rp", "col", "val"), r)})
        ent = float(sum(V.shape[0] ** 2 for V, _ in axes))
        print(json.dumps({"metric": METRIC, "value": ent / (ms * 1e-3), "unit": UNIT,
                          "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
                          "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
                          "dry_run": True, "backend": "gloo" if world > 1 else "none",
                          "config": {"workload": f"dry run: axes n={[int(V.shape[0]) for V, _ in axes]}"
                                                 ", k=16, top-10 (launcher test only)"}}),
              flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


def run_reference(args):
    """The reference arm: the fp64 CPU oracle (as it stands) on a bounded row sample."""
    world, rank, _ = _dist_env()
    if rank != 0:
        return 0
    import oracle as O
    axes, t = _load_workload(args.config)
    rows_per_axis = args.ref_rows
    rng = np.random.default_rng(0)
    samples = [np.sort(rng.choice(V.shape[0], size=min(rows_per_axis, V.shape[0]),
                                  replace=False)) for V, _ in axes]
    ent_step = sum(len(s) * V.shape[0] for s, (V, _) in zip(samples, axes))

    def step():
        for s, (V, lam) in zip(samples, axes):
            O.sparse_precision(V, lam, 0, 0, rows=s, t=t)
    for _ in range(args.warmup):
        step()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        step()
    dt = (time.perf_counter() - t0) / args.steps
    value = ent_step / dt
    cores = _blas_threads()
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": dt * 1e3,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (synth.gen seeded recipes)",
        "config": {"workload": WORKLOADS[args.config], "sample_rows_per_axis": rows_per_axis},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "oracle",
                         "sample": f"{rows_per_axis} random rows per axis x all n columns per "
                                   f"step (fp64 NumPy oracle, oracle.sparse_precision)"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def _blas_threads():
    try:
        from threadpoolctl import threadpool_info
        info = threadpool_info()
        n = max((i.get("num_threads", 0) for i in info), default=0)
        return int(n) if n else os.cpu_count()
    except Exception:
        return os.cpu_count()


def cpu_baseline(axes, t, rows=4096, full_axis_max=32768):
    """The oracle as it stands on a bounded sample of the step (sampled rows of
    the large axis plus every row of an axis small enough to finish in seconds)."""
    import oracle as O
    rng = np.random.default_rng(1)
    ent, parts = 0, []
    t0 = time.perf_counter()
    for V, lam in axes:
        n = V.shape[0]
        if n <= full_axis_max:
            s = np.arange(n, dtype=np.int64)
            parts.append(f"all {n} rows of the n={n} axis")
        else:
            s = np.sort(rng.choice(n, size=min(rows, n), replace=False))
            parts.append(f"{len(s)} random rows of the n={n} axis")
        O.sparse_precision(V, lam, 0, 0, rows=s, t=t)
        ent += len(s) * n
    dt = time.perf_counter() - t0
    return {"value": ent / dt, "unit": UNIT, "cores": _blas_threads(), "kind": "oracle",
            "sample": " + ".join(parts) + f", all columns ({dt:.1f} s, fp64 NumPy "
                      "oracle.sparse_precision)"}


def stage_timings(G, torch):
    """§8(a) rows a1-a4 (Gram spectrum + eigenvalue MLE) on the data configs C2 and C3:
    device time of ggm_gram_eig per axis and of ggm_solve_eigvals (both synchronise)."""
    from synth import gen
    out = {}
    for name in ("C2", "C3"):
        cfg = gen.config(name)
        X = torch.from_numpy(cfg["X"]).cuda()
        ks = cfg["k"]
        Es, gram_ms = [], []
        for a, k in enumerate(ks):
            G.ggm_gram_eig(X, a, k)              # warm-up (handles, workspace sizing)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            _, E, _ = G.ggm_gram_eig(X, a, k)
            gram_ms.append((time.perf_counter() - t0) * 1e3)
            Es.append(E)
        if X.dim() > 2:                           # all axes, concurrent eigensolves ((1h))
            G.ggm_gram_eig_axes(X, ks)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            G.ggm_gram_eig_axes(X, ks)
            out.setdefault("gram_eig_axes_ms", {})[name] = (time.perf_counter() - t0) * 1e3
        if X.dim() == 2:                          # both axes from one Gram (include/ggm.h (1g))
            G.ggm_gram_eig_matrix(X, ks[0], ks[1])
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            G.ggm_gram_eig_matrix(X, ks[0], ks[1])
            out.setdefault("gram_eig_matrix_ms", {})[name] = (time.perf_counter() - t0) * 1e3
        Ec = torch.cat(Es)
        G.ggm_solve_eigvals(Ec, ks)
        torch.cuda.synchronize()
        solve_ms = float("inf")
        for _ in range(3):                        # whole call incl. host work: best of 3
            t0 = time.perf_counter()
            _, info = G.ggm_solve_eigvals(Ec, ks)
            solve_ms = min(solve_ms, (time.perf_counter() - t0) * 1e3)
        pts = float(np.prod(ks))
        kms = info["kernel_ms"]
        out[name] = {"gram_eig_ms": gram_ms, "solve_ms": solve_ms,
                     "solve_iterations": info["iterations"], "solve_passes": info["passes"],
                     "solve_kernel_ms": kms,
                     "stationarity": info["stationarity"],
                     "grid_points_per_s": pts * info["passes"] / (kms * 1e-3),
                     "grid_points": pts}
        if name == "C3":
            # BK4 roofline (BK4): FP64-pipe bound, 5 FP64-pipe instructions per grid
            # point (s = base + λ, two Newton FMAs, two accumulating adds) + 1 MUFU seed; peak
            # = 64 FP64 lanes/clk/SM x SMs x the max SM clock / 5
            peaks, _ = _peaks()
            f_max = peaks.get("sm_max_mhz", 1965.0) * 1e6
            import torch as _t
            sms = _t.cuda.get_device_properties(0).multi_processor_count
            peak_pts = 64.0 * sms * f_max / 5.0
            ach = pts * info["passes"] / (kms * 1e-3)
            out["roofline_bk4"] = {
                "bound": "alu", "kernel": "solve_kernel (BK4, C3 grid 400x300x200)",
                "achieved": ach / 1e12, "peak": peak_pts / 1e12, "unit": "Tpoints/s",
                "frac": ach / peak_pts, "traffic": None,
                "basis": "grid points x passes / CUDA-event kernel time; peak: FP64 pipe "
                         "(64 lanes/clk/SM) at sm_max_mhz / 5 FP64 instructions per point",
                "passes": info["passes"], "kernel_ms": kms}
    # at-scale spectrum: a 40,000 x 40,000 unfolding (beyond the dense
    # Gram path) of known spectrum, X = U diag(s) W^T, k = 50, randomized subspace iteration
    d = m = 40_000
    g = torch.Generator(device="cuda").manual_seed(11)
    U = torch.linalg.qr(torch.randn(d, 64, device="cuda", dtype=torch.float64, generator=g))[0]
    W = torch.linalg.qr(torch.randn(m, 64, device="cuda", dtype=torch.float64, generator=g))[0]
    sv = torch.logspace(3, 1, 64, device="cuda", dtype=torch.float64)
    X = ((U * sv) @ W.T).float()
    del U, W
    G.ggm_gram_eig_rsi(X, 0, 50)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    _, E, _, it, ch = G.ggm_gram_eig_rsi(X, 0, 50)
    rsi_ms = (time.perf_counter() - t0) * 1e3
    err = float(torch.max(torch.abs(E - sv[:50] ** 2) / sv[:50] ** 2))
    out["rsi_40000x40000_k50"] = {"ms": rsi_ms, "iterations": it, "ritz_change": ch,
                                  "max_rel_err_vs_closed_form": err}
    del X
    torch.cuda.empty_cache()
    return out


def sparse_spectrum_timing(G, torch):
    """§8(f) rows 1 + 4 at the paper's largest real-data scale (PBMC, 1,248,980 cells x 2,200
    genes): a synthetic CSR count matrix (10 % nonzero, log1p of uniform counts,
    generated on the device) -> COCA in its sparse + rank-one form + randomized subspace
    iteration for the cell axis, k = 50, bounded at 20 iterations (time per iteration
    reported)."""
    d, m, dens = 1_248_980, 2_200, 0.10
    g = torch.Generator(device="cuda").manual_seed(13)
    rps, cols, vals = [torch.zeros(1, dtype=torch.int64, device="cuda")], [], []
    base = 0
    for r0 in range(0, d, 65536):
        mask = torch.rand((min(65536, d - r0), m), device="cuda", generator=g) < dens
        idx = mask.nonzero()
        cnt = mask.sum(1)
        rps.append(base + torch.cumsum(cnt, 0))
        base += int(idx.shape[0])
        cols.append(idx[:, 1].to(torch.int32))
        vals.append(torch.log1p(torch.randint(1, 30, (idx.shape[0],), device="cuda",
                                              generator=g).float()))
        del mask, idx
    rp, col, val = torch.cat(rps), torch.cat(cols), torch.cat(vals)
    del rps, cols, vals
    out = {"shape": [d, m], "nnz": int(val.numel()), "k": 50,
           "method": "exact Gram of the 2,200 side: tensor-core chunk Grams (gram_tc.cu, "
                     "3 x fp16 split, fp32 over 4,096-sample slices, fp64 across) of S from "
                     "the CSR + exact fp64 rank-one terms of S + z 1^T (COCA, P:1003-1012) + "
                     "DSYEVD; the long side by a CSR row projection"}
    peaks, _ = _peaks()
    gram_flops = float(d) * m * m   # the symmetric half of 2 d m^2 (algorithmic)

    def run(tag, rp_, col_, val_, mm):
        for npn in (False, True):
            G.ggm_gram_eig_csr(rp_, col_, val_, mm, 50, nonparanormal=npn)  # warm-up
            torch.cuda.synchronize()
            G.set_timing(True)
            t0 = time.perf_counter()
            G.ggm_gram_eig_csr(rp_, col_, val_, mm, 50, nonparanormal=npn)
            torch.cuda.synchronize()
            key = f"{tag}_{'coca' if npn else 'raw'}"
            out[key + "_ms"] = (time.perf_counter() - t0) * 1e3
            gms, ems, pms = G.last_timing()
            out[key + "_stages_ms"] = {"gram": gms, "eigensolve": ems, "projection_store": pms}
            if npn is False and tag == "cell_axis":
                peak = peaks.get("bf16_tflops_sustained", peaks.get("bf16_tflops")) / 3.0
                ach = gram_flops / (gms * 1e-3) / 1e12
                out["roofline_gram"] = {
                    "bound": "tensor", "kernel": "gram_tc (scatter + tcgen05 Gram + fp64 red)",
                    "achieved": ach, "peak": peak, "unit": "TFLOP/s", "frac": ach / peak,
                    "traffic": None,
                    "basis": "d m^2 flops (symmetric half of the 1,248,980 x 2,200 Gram) / "
                             "CUDA-event time of the Gram stage incl. the CSR scatter; peak: "
                             "bf16 sustained / 3 (3-term fp16 split)"}

    run("cell_axis", rp, col, val, m)
    # gene axis: the same matrix as gene-major CSR (2,200 rows of 1,248,980 cells)
    rows = torch.repeat_interleave(torch.arange(d, device="cuda"), rp[1:] - rp[:-1])
    order = torch.argsort(col.to(torch.int64) * d + rows)
    tcol = rows[order].to(torch.int32)
    tval = val[order]
    trp = torch.zeros(m + 1, dtype=torch.int64, device="cuda")
    trp[1:] = torch.cumsum(torch.bincount(col.to(torch.int64), minlength=m), 0)
    del rows, order, rp, col, val
    run("gene_axis", trp, tcol, tval, d)
    del trp, tcol, tval
    torch.cuda.empty_cache()
    return out


def overall_timing(G, torch, V, lam):
    """§8(f) NEXT 2 on the largest axis: whole-graph rules as the paper recommends for
    scRNA-seq: N = 10 n edges overall, degree down-weighting, 1 min edge."""
    n = V.shape[0]
    kw = dict(downweight=True, min_edges=1)
    _, _, _, (ccap, cap) = G.ggm_sparse_precision_overall(V, lam, 10 * n, return_caps=True, **kw)
    torch.cuda.synchronize()
    ms = float("inf")
    for _ in range(2):  # best of two calls (the first may still grow the caching allocator)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        rp, c, v = G.ggm_sparse_precision_overall(V, lam, 10 * n, cand_capacity=ccap,
                                                  capacity=cap, **kw)
        e1.record()
        torch.cuda.synchronize()
        ms = min(ms, e0.elapsed_time(e1))
    path, sat = G.overall_last_path()
    return {"path": {0: "lists", 1: "histogram+threshold", 2: "lists+saturated block",
                     3: "sampled global threshold + one symmetric pass"}.get(path, path),
            "saturated_rows": sat, "phases_ms": G.overall_last_timing(), "n": int(n), "n_edges": 10 * int(n), "downweight": True, "min_edges": 1,
            "edges_kept": int(c.numel()) // 2, "ms": ms, "entries_per_s": float(n) * n / (ms * 1e-3),
            "launches": G.last_launches()}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="C5", choices=sorted(WORKLOADS))
    ap.add_argument("--ref-rows", type=int, default=64)
    ap.add_argument("--cpu-rows", type=int, default=4096)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-stages", action="store_true",
                    help="skip the a1-a4 stage timings (gram_eig + solve on C2/C3)")
    ap.add_argument("--dry-run", action="store_true",
                    help="CPU/gloo launcher + plumbing check with an injected compute (tests)")
    ap.add_argument("--dry-n", type=int, default=2000)
    args = ap.parse_args()
    rc = _maybe_launch(args)
    if rc is not None:
        return rc
    if args.dry_run:
        return run_dry(args)
    if args.impl == "reference":
        return run_reference(args)

    import torch
    import torch.distributed as dist
    import paper_2407_19892_b200 as G
    from paper_2407_19892_b200.parallel import (assemble_rows, exchange_candidates, gather_topk_csr,
                                                shard_rows)

    world, rank, local = _dist_env()
    torch.cuda.set_device(local)
    if world > 1:
        os.environ.setdefault("NCCL_DEBUG", "INFO")          # communicator lines (nranks = N)
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        os.environ.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        print(f"bench.py: rank {rank}/{world} on cuda:{local} "
              f"({torch.cuda.get_device_name(local)})", file=sys.stderr, flush=True)
    if not G.device_supported():
        raise SystemExit("libggm: device is not sm_100a")

    # ---------------- inputs: rank 0 generates, NCCL broadcast replicates (setup, untimed)
    if rank == 0:
        host_axes, t = _load_workload(args.config)
        shapes = [V.shape for V, _ in host_axes]
    else:
        host_axes, t, shapes = None, None, None
    if world > 1:
        obj = [shapes, t]
        dist.broadcast_object_list(obj, src=0)
        shapes, t = obj
    dev_axes = []
    for a, (n, k) in enumerate(shapes):
        if rank == 0:
            V = torch.from_numpy(host_axes[a][0]).cuda()
            lam = torch.from_numpy(host_axes[a][1]).cuda()
        else:
            V = torch.empty((n, k), dtype=torch.float32, device="cuda")
            lam = torch.empty((k,), dtype=torch.float64, device="cuda")
        if world > 1:
            dist.broadcast(V, 0)
            dist.broadcast(lam, 0)
        dev_axes.append((V, lam))
    if host_axes is None:   # host copies for the e2e arm on the other ranks
        host_axes = [(V.cpu().numpy(), lam.cpu().numpy()) for V, lam in dev_axes]

    # per axis: at N > 1, large axes (n >= 65,536, k <= 128) run the distributed symmetric
    # scheme (this rank's share of the block pairs + all-to-all of candidate buckets + merge of
    # its rows); the others run row shards of the plain scheme.  At N = 1 every axis is one
    # ggm_sparse_precision call (symmetric scheme chosen automatically for large axes).
    plans, kinds = [], []
    for (V, lam) in dev_axes:
        n, k = V.shape
        if (world > 1 or os.environ.get("BENCH_FORCE_SYMSHARD")) and n >= 65536 and k <= 128:
            plans.append(G.SymShardPlan(n, k, t, rank, world))
            kinds.append("symshard")
        else:
            b, e = shard_rows(n, world, rank)
            plans.append(G.SparsePlan(n, k, b, e, mode=0, topk=t))
            kinds.append("rows")
    entries_step = float(sum(V.shape[0] ** 2 for V, _ in dev_axes))
    G.set_timing(True)
    stream = torch.cuda.current_stream()

    fused_ms = [[] for _ in plans]
    stage_ms = [[] for _ in plans]   # (prep incl. seed pass, main kernel, merge) per call
    stats = [None for _ in plans]
    launches = [0]

    def run_axis(a, V, lam, record=False):
        """One axis of the hot path; returns its CSR (row_ptr, col, val) (full at N > 1)."""
        plan = plans[a]
        n = V.shape[0]
        if kinds[a] == "symshard":
            thr_all = None
            if world > 1:  # sharded seed pass: one all-reduce(MIN) of n floats
                thr_all = plan.seed(V, lam)
                dist.all_reduce(thr_all, op=dist.ReduceOp.MIN)
            key, val, counts, perm = plan.run(V, lam, thr_all=thr_all)
            if record:
                tm = G.last_timing()
                fused_ms[a].append(tm[1])
                stage_ms[a].append(tuple(tm))
                stats[a] = G.last_stats()
                launches[0] += G.last_launches()
            rkey, rval = exchange_candidates(key, val, counts)
            b, e = G.sym_rows_begin(n, plan.k, t, rank, world), G.sym_rows_begin(n, plan.k, t, rank + 1, world)
            row_id, col, vals = G.sym_merge(n, t, rkey, rval, perm, b, e)
            if record:
                launches[0] += G.last_launches()
            return assemble_rows(row_id, col, vals, n, min(t, n - 1))
        plan.run(V, lam)
        if record:
            tm = G.last_timing()
            fused_ms[a].append(tm[1])
            stage_ms[a].append(tuple(tm))
            stats[a] = G.last_stats()
            launches[0] += G.last_launches()
        if world > 1:
            return gather_topk_csr(plan.col, plan.val, plan.t_eff, n)
        return plan.row_ptr, plan.col, plan.val

    def step(record=False):
        return [run_axis(a, V, lam, record) for a, (V, lam) in enumerate(dev_axes)]

    for _ in range(max(args.warmup, 0)):
        step()
    clocks = ClockSampler(local)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    clocks.start()
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    ev0.record(stream)
    for _ in range(args.steps):
        step(record=True)
    ev1.record(stream)
    torch.cuda.synchronize()
    clk = clocks.stop()
    elapsed_ms = ev0.elapsed_time(ev1)
    if world > 1:
        tt = torch.tensor([elapsed_ms], device="cuda")
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        elapsed_ms = float(tt.item())
        dist.barrier()
    ms_step = elapsed_ms / args.steps
    value = entries_step / (ms_step * 1e-3)

    # ---------------- roofline of the dominant kernel (BK2 on the largest axis)
    peaks, peak_src = _peaks()
    a0 = int(np.argmax([V.shape[0] for V, _ in dev_axes]))
    V0 = dev_axes[a0][0]
    n0, k0 = V0.shape
    rows0 = n0 if kinds[a0] == "symshard" else plans[a0].row_end - plans[a0].row_begin
    avg_fused = float(np.mean(fused_ms[a0]))
    st0 = stats[a0]
    sym0 = st0["scheme"] == "symmetric"
    # algorithmic work of the dominant kernel: 2k flops per entry it must
    # evaluate -- all rows x n entries (plain), or each unordered pair once, n(n+1)/2 entries
    # (symmetric scheme: ψ_ij = ψ_ji)
    alg_entries = n0 * (n0 + 1) / 2.0 if sym0 else float(rows0) * n0
    if kinds[a0] == "symshard":   # this rank's share of the unordered pairs
        alg_entries /= world
    alg_flops = 2.0 * k0 * alg_entries
    achieved = alg_flops / (avg_fused * 1e-3) / 1e12
    # fp32-accurate tensor peak = fp16 (= bf16) dense rate / 3 (3-term split).  The sustained
    # cuBLAS figure is the default; when BK2 runs above it (its clock under the power cap
    # stays higher than cuBLAS's), the burst figure is the honest denominator.
    # With hi*hi screening (symmetric scheme default) the main kernel issues ONE fp16 product
    # per entry (+ the packed 3-term tail) and the candidates are re-evaluated exactly
    # afterwards: its peak is the plain fp16 (= bf16) dense rate.
    screening = st0["mma_k_per_entry"] < 2.0 * k0
    div = 1.0 if screening else 3.0
    peak_sus = peaks.get("bf16_tflops_sustained", peaks.get("bf16_tflops")) / div
    peak_burst = peaks.get("bf16_tflops", peak_sus * div) / div
    peak_is_burst = achieved > peak_sus
    peak = peak_burst if peak_is_burst else peak_sus
    traffic = None
    tp = os.path.join(ROOT, "profiles", "fused_traffic.json")
    if os.path.exists(tp):
        try:
            with open(tp) as f:
                tj = json.load(f)
            if tj.get("config") == args.config and world == 1:
                traffic = tj.get("traffic_bytes_per_launch")
        except Exception:
            traffic = None
    step_ms_fused_share = sum(np.mean(f) for f in fused_ms) / ms_step

    # ---------------- e2e through the same public API from pinned host buffers
    e2e = None
    if not args.no_e2e:
        hV = [torch.from_numpy(np.ascontiguousarray(h[0])).pin_memory() for h in host_axes]
        hL = [torch.from_numpy(np.ascontiguousarray(h[1])).pin_memory() for h in host_axes]
        outs = step()
        hout = [(torch.empty(o[0].numel(), dtype=torch.int64).pin_memory(),
                 torch.empty(o[1].numel(), dtype=torch.int32).pin_memory(),
                 torch.empty(o[2].numel(), dtype=torch.float32).pin_memory()) for o in outs]
        h2d = sum(v.numel() * 4 + l.numel() * 8 for v, l in zip(hV, hL))
        d2h = sum(o[0].numel() * 8 + o[1].numel() * 4 + o[2].numel() * 4 for o in hout)

        # Every step uploads its inputs from pinned host memory and reads its CSR back.  The
        # upload of step i+1 runs on a copy stream while step i computes (double-buffered
        # device inputs) and step i's download overlaps step i+1, as a streaming service
        # would; the first upload and the last download are on the timed path.
        copy_s = torch.cuda.Stream()
        bufs = [[(torch.empty_like(V), torch.empty_like(lam)) for V, lam in dev_axes]
                for _ in range(2)]
        ev_in = [torch.cuda.Event(), torch.cuda.Event()]
        ev_used = [torch.cuda.Event(), torch.cuda.Event()]

        def upload(slot):
            with torch.cuda.stream(copy_s):
                copy_s.wait_event(ev_used[slot])   # the slot's previous step is done with it
                for a in range(len(plans)):
                    bufs[slot][a][0].copy_(hV[a], non_blocking=True)
                    bufs[slot][a][1].copy_(hL[a], non_blocking=True)
                ev_in[slot].record(copy_s)

        # downloads: the step's CSR is copied (device to device) into one of two output
        # slots and read back to pinned host memory on a third stream while the next step
        # computes
        dl_s = torch.cuda.Stream()
        dslots = [[tuple(torch.empty_like(x) for x in o) for o in outs] for _ in range(2)]
        hslots = [hout, [tuple(torch.empty_like(x).pin_memory() for x in h) for h in hout]]
        ev_out = [torch.cuda.Event(), torch.cuda.Event()]
        ev_dl = [torch.cuda.Event(), torch.cuda.Event()]

        def e2e_run(nsteps):
            copy_s.wait_stream(stream)   # uploads start after the timing event
            dl_s.wait_stream(stream)
            upload(0)
            for i in range(nsteps):
                slot = i % 2
                if i + 1 < nsteps:
                    upload(1 - slot)
                stream.wait_event(ev_in[slot])
                stream.wait_event(ev_dl[slot])   # this output slot's previous download is done
                for a in range(len(plans)):
                    res = run_axis(a, *bufs[slot][a])
                    for d, x in zip(dslots[slot][a], res):
                        d.copy_(x, non_blocking=True)
                ev_used[slot].record(stream)
                ev_out[slot].record(stream)
                with torch.cuda.stream(dl_s):
                    dl_s.wait_event(ev_out[slot])
                    for a in range(len(plans)):
                        for h, d in zip(hslots[slot][a], dslots[slot][a]):
                            h.copy_(d, non_blocking=True)
                    ev_dl[slot].record(dl_s)
            torch.cuda.synchronize()
        e2e_run(2)
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        e2e_run(args.steps)
        e1.record(stream)
        torch.cuda.synchronize()
        ems = e0.elapsed_time(e1)
        if world > 1:
            tt = torch.tensor([ems], device="cuda")
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            ems = float(tt.item())
        e2e = {"value": entries_step / (ems / args.steps * 1e-3), "unit": UNIT,
               "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h)}

    if rank == 0:
        cpu = None if (args.no_cpu or world > 1) else cpu_baseline(host_axes, t, args.cpu_rows)
        stages = None if args.no_stages else stage_timings(G, torch)
        if stages is not None:
            stages["overall_rules_axisA"] = overall_timing(G, torch, *dev_axes[a0])
            stages["sparse_coca_spectrum_pbmc_scale"] = sparse_spectrum_timing(G, torch)
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": DTYPE, "data": "synthetic (synth.gen seeded recipes of BASELINE.json configs)",
            "config": {"workload": WORKLOADS[args.config], "axes_n": [int(V.shape[0]) for V, _ in dev_axes],
                       "k": [int(V.shape[1]) for V, _ in dev_axes], "topk": int(t),
                       "parallelism": (f"symmetric block-pair shards + all-to-all x{world} (axes n >= 65536), "
                                       f"row shards (others)" if world > 1 else "single GPU"), "l2": "inputs > L2 (no flush needed)"},
            "roofline": {"bound": "tensor", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                         "frac": achieved / peak, "frac_vs_sustained": achieved / peak_sus,
                         "traffic": traffic,
                         "kernel": "fused_recon_topk (BK2, %s scheme%s)" % (
                             st0["scheme"], ", CTA pairs" if st0["cta_pair"] else ""),
                         "achieved_basis": "2k flops per entry (SURVEY 8(d)) x %s / mean CUDA-event "
                                           "duration of BK2 on the largest axis" % (
                                               "n(n+1)/2 unordered entries" if sym0 else "rows x n"),
                         "peak_basis": (f"{peak_src} bf16_tflops{'' if peak_is_burst else '_sustained'} "
                                        "(hi*hi screening: one fp16 MMA product per entry, fp16 rate = "
                                        "bf16 rate; candidates re-evaluated exactly in fp64 afterwards)"
                                        if screening else
                                        f"{peak_src} bf16_tflops{'' if peak_is_burst else '_sustained'} / 3 "
                                        "(3-term fp16 split = 3 MMAs per fp32-accurate product; fp16 rate = "
                                        "bf16 rate)") + ("; burst figure because BK2 runs above the cuBLAS "
                                                         "sustained rate" if peak_is_burst else ""),
                         "screening": bool(screening),
                         "kernel_ms": avg_fused, "step_share": step_ms_fused_share,
                         "tensor_pipe_tflops": st0["entries_main"] * 2.0 * st0["mma_k_per_entry"]
                         / (avg_fused * 1e-3) / 1e12,
                         "stages_ms_axis": {"prep_incl_seed": float(np.mean([x[0] for x in stage_ms[a0]])),
                                            "main": avg_fused,
                                            "merge": float(np.mean([x[2] for x in stage_ms[a0]]))},
                         "candidates_per_row": st0["candidates"] / n0 if sym0 else None},
            "cpu_baseline": cpu,
            "e2e": e2e,
            "clocks": clk,
            "gpu_launches": int(launches[0]),
            "stages_a1_a4": stages,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
