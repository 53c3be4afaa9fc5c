#!/usr/bin/env python3
"""Block-CG throughput bench (BASELINE.json metric: RHS*iterations/s, FP64).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c2] [--impl ours|reference]

Workload (config.workload): BASELINE.json configs[1] = C2, 3D 7-point Poisson
128^3 (n = 2,097,152, CSR FP64), k = 32 right-hand sides B ~ N(0,1) (seed 7),
X0 = 0, hybrid subalgebra p = 8, stop at per-column relative residual 1e-8.
One *step* = one complete solve (all iterations to convergence).

value  : k * iterations / device time, inputs resident in HBM (DeviceSolver),
         CUDA events on the library stream, W warm-up solves first.
e2e    : the same metric through the public drop-in call
         blockkrylov.bcg_solve(A, B, M, cfg, opts) from pinned host buffers:
         CSR + B uploaded and X downloaded inside every timed step.
roofline: dominant fused kernel (per-launch CUDA-event time from an untimed
         profiling pass on the same stream) vs algorithmic bytes.
cpu_baseline: the reference CPU solver (oracle/_ref, built from
         /root/reference) or its C restatement (oracle port) on this host's
         cores, on a bounded sample of the same workload.
--impl reference: the reference CPU implementation alone (all host threads).

Multi-GPU (torchrun, N > 1): the same C2 system, rows split into N
contiguous slabs (one per rank), P halo via ncclSend/Recv and the Gram
partials via ncclAllReduce (paper_1912_11930_b200/partitioned.py); strong
scaling, value = k * iterations / max-over-ranks solve time.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "BCG RHS·iterations/sec (FP64) and achieved HBM fraction at 1/2/4/8 B200"
UNIT = "RHS·iterations/s"

CONFIGS = {
    # name: (kind, nx, ny, nz, k, p, mode, rhs, tol, max_iter, description)
    "c1": (0, 128, 128, 1, 8, 8, "hybrid", "normal", 1e-8, 500,
           "C1 2D 5-pt Poisson 128^2, k=8, classical, tol 1e-8 / 500"),
    "c2": (3, 128, 128, 128, 32, 8, "hybrid", "normal", 1e-8, 0,
           "C2 3D 7-pt Poisson 128^3, k=32, hybrid p=8, tol 1e-8"),
    "c3p": (2, 1024, 1024, 1, 64, 1, "hybrid", "uniform", 1e-8, 200,
            "C3 2D lognormal diffusion 1024^2, k=64, parallel p=1 (200-iteration sample)"),
    "c3g": (2, 1024, 1024, 1, 64, 4, "global", "uniform", 1e-8, 200,
            "C3 2D lognormal diffusion 1024^2, k=64, global p=4 (200-iteration sample)"),
    "c4c": (4, 192, 192, 192, 16, 16, "hybrid", "normal", 1e-300, 200,
            "C4 3D 27-pt 192^3, k=16, classical, fixed 200 iterations"),
    "c4h": (4, 192, 192, 192, 16, 4, "hybrid", "normal", 1e-300, 200,
            "C4 3D 27-pt 192^3, k=16, hybrid p=4, fixed 200 iterations"),
    "c4g": (4, 192, 192, 192, 16, 4, "global", "normal", 1e-300, 200,
            "C4 3D 27-pt 192^3, k=16, global p=4, fixed 200 iterations"),
    "c5": (3, 256, 256, 256, 64, 16, "hybrid", "normal", 1e-300, 100,
           "C5 (1-GPU subgrid) 3D 7-pt 256^3, k=64, hybrid p=16, fixed 100 iterations"),
}
RHS_SEED = 7
COEFF_SEED = 11
CPU_SAMPLE_ITERS = 2


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def make_inputs(cfg_name, gen):
    kind, nx, ny, nz, k, p, mode, rhs, tol, max_iter, desc = CONFIGS[cfg_name]
    a = gen.stencil(kind, nx, ny, nz, seed=COEFF_SEED if kind == 2 else 0)
    n = a.n()
    b = np.empty((n, k))
    if rhs == "normal":
        gen.normal_block_rhs(n, k, RHS_SEED, out=b)
    else:
        gen.random_block_rhs(n, k, RHS_SEED, out=b)
    return a, b


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, device=0):
        self.device = device
        self.rows = []
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except (OSError, FileNotFoundError):
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [x.strip() for x in line.split(",")]
            if len(parts) == 6:
                self.rows.append(parts)

    def __exit__(self, *exc):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if r[2 + i] == "Active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.rows)}


def measured_peak():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            return float(json.load(f)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except (OSError, KeyError, ValueError):
        return 6650.0, "fallback (B200_PROFILING.md)"


def ncu_traffic(kernel_class):
    """Per-launch DRAM bytes of the kernel from the committed ncu summary."""
    path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        with open(path) as f:
            return json.load(f).get(kernel_class)
    except (OSError, ValueError):
        return None


def cpu_threads_for(n, k):
    cores = os.cpu_count() or 1
    try:
        import psutil
        avail = psutil.virtual_memory().available
    except Exception:
        avail = 32 << 30
    per_solve = 7 * n * k * 8  # x, r, q, p, z, b copy, final ax (solver.hpp:365-446)
    return max(1, min(cores, int(avail * 0.6 // per_solve)))


def cpu_sample(cfg_name, a, b, threads=None):
    """One bounded sample of the reference CPU solver: `threads` concurrent
    solves of the workload, each capped at CPU_SAMPLE_ITERS iterations."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    from oracle import Oracle, available
    kind = "reference" if available("reference") else "port"
    orc = Oracle(kind)
    _, _, _, _, k, p, mode, _, tol, _, _ = CONFIGS[cfg_name]
    n = a.n()
    threads = threads or cpu_threads_for(n, k)
    csr = (a.row_offsets(), a.col_indices(), a.values())
    dt, its = orc.bench_solve(threads, csr, b, p, mode == "global", tol, CPU_SAMPLE_ITERS)
    return kind, threads, dt, its


def run_reference(args):
    ws, rank, _ = dist_env()
    if rank != 0:
        return 0
    import paper_1912_11930_b200 as bk  # generators only (inputs); solve is the reference's
    a, b = make_inputs(args.config, bk)
    k = CONFIGS[args.config][4]
    threads = cpu_threads_for(a.n(), k)
    for _ in range(args.warmup):
        cpu_sample(args.config, a, b, threads)
    total_t = 0.0
    total_it = 0
    kind = "port"
    for _ in range(args.steps):
        kind, threads, dt, its = cpu_sample(args.config, a, b, threads)
        total_t += dt
        total_it += its
    value = k * total_it / total_t
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * total_t / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic",
        "config": {"workload": CONFIGS[args.config][10], "n": a.n(), "nnz": a.nnz(), "k": k,
                   "parallelism": f"cpu x{threads} independent solves"},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind":
                         "reference" if kind == "reference" else "port",
                         "sample": f"{threads} concurrent reference bcg_solve calls x "
                                   f"{CPU_SAMPLE_ITERS} iterations per step (wall time incl. "
                                   "per-solve setup and final residual)"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def run_ours(args):
    import torch
    import paper_1912_11930_b200 as bk
    ws, rank, local = dist_env()
    dist = ws > 1
    if dist:
        import torch.distributed as tdist
        torch.cuda.set_device(local)
        tdist.init_process_group("nccl", device_id=torch.device("cuda", local))
    kind, nx, ny, nz, k, p, mode, rhs, tol, max_iter, desc = CONFIGS[args.config]
    ctx = bk.Context(local, "fast")
    stream = torch.cuda.ExternalStream(ctx.stream(), device=torch.device("cuda", local))

    t0 = time.time()
    a, b = make_inputs(args.config, bk)
    n, nnz = a.n(), a.nnz()
    log(f"[rank {rank}] inputs n={n} nnz={nnz} k={k} ({time.time() - t0:.1f}s)")
    cfg = bk.SubalgebraConfig(k, p, mode)

    def barrier_sync():
        torch.cuda.synchronize(local)
        if dist:
            tdist.barrier()
        torch.cuda.synchronize(local)

    def timed(fn, steps):
        """Max-over-ranks device time of `steps` calls of fn (CUDA events on
        the library stream, barrier + synchronize on both sides)."""
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        barrier_sync()
        e0.record(stream)
        out = [fn() for _ in range(steps)]
        e1.record(stream)
        barrier_sync()
        ms = e0.elapsed_time(e1)
        if dist:
            t = torch.tensor([ms], device=f"cuda:{local}")
            tdist.all_reduce(t, op=tdist.ReduceOp.MAX)
            ms = float(t.item())
        return ms, out

    if dist:
        return run_partitioned(args, bk, ctx, stream, a, b, cfg, timed, rank, ws, local)

    # ---------------- value: resident inputs -------------------------------
    solver = bk.DeviceSolver(a, cfg, ctx)
    solver.set_rhs(b)
    for _ in range(args.warmup):
        rep = solver.run(tol, max_iter)
    launches0 = ctx.launch_count()
    with ClockSampler(local) as clocks:
        ms, reps = timed(lambda: solver.run(tol, max_iter), args.steps)
    launches = ctx.launch_count() - launches0
    its = [int(r.iterations) for r in reps]
    total_its = sum(its)
    value_rank = k * total_its / (ms * 1e-3)
    value = value_rank * ws  # every rank runs the same fixed work
    log(f"[rank {rank}] value: {args.steps} solves, iterations/solve={its[0]}, "
        f"{ms / args.steps:.2f} ms/solve, {value_rank:.1f} RHS*it/s")

    # ---------------- roofline: per-kernel profile pass --------------------
    prof = solver.profile(20)
    kbytes = solver.kernel_bytes()
    names = ["K1_spmm_gram", "K2_update_gram", "K3_update_p"]
    shares = prof[:3] / max(prof[3], 1e-30)
    dom = int(np.argmax(prof[:3]))
    peak, peak_src = measured_peak()
    achieved = kbytes[dom] / (prof[dom] * 1e-3) / 1e9
    traffic = ncu_traffic(names[dom])
    iter_bytes_model = 8.0 * (2 * nnz + 17 * n * k)  # paper Table 1 beta
    iter_ms = ms / max(total_its, 1)
    solver.close()

    # ---------------- e2e: public drop-in call, host buffers ---------------
    pin_b = torch.empty((n, k), dtype=torch.float64, pin_memory=True).numpy()
    pin_b[...] = b
    pin_off = torch.empty(n + 1, dtype=torch.int64, pin_memory=True).numpy().view(np.uint64)
    pin_off[...] = a.row_offsets()
    pin_col = torch.empty(nnz, dtype=torch.int64, pin_memory=True).numpy().view(np.uint64)
    pin_col[...] = a.col_indices()
    pin_val = torch.empty(nnz, dtype=torch.float64, pin_memory=True).numpy()
    pin_val[...] = a.values()
    pin_x = torch.empty((n, k), dtype=torch.float64, pin_memory=True).numpy()
    m = bk.Preconditioner.identity(n)
    opts = bk.SolveOptions(tol=tol, max_iter=max_iter)

    def e2e_step():
        t0 = time.perf_counter()
        am = bk.SparseMatrix(n, pin_off, pin_col, pin_val, validate=False)
        res = bk.bcg_solve(am, pin_b, m, cfg, opts, ctx=ctx, out=pin_x)
        am.release_device()
        if os.environ.get("BKG_BENCH_DEBUG"):
            print(f"e2e step {1e3 * (time.perf_counter() - t0):.1f} ms host, loop "
                  f"{1e3 * res.report.loop_seconds:.1f} ms", file=sys.stderr)
        return res.report.iterations

    e2e_step()  # warm-up (allocator, module load)
    e2e_steps = max(1, min(args.steps, 3))
    e2e_ms, e2e_its = timed(e2e_step, e2e_steps)
    e2e_value = ws * k * sum(e2e_its) / (e2e_ms * 1e-3)
    h2d = 8 * (n + 1) + 16 * nnz + 8 * n * k
    d2h = 8 * n * k + 8 * k

    # ---------------- CPU baseline (rank 0, N = 1 only) --------------------
    cpu = None
    if rank == 0 and ws == 1 and not args.no_cpu:
        ck, threads, dt, cits = cpu_sample(args.config, a, b)
        cpu = {"value": k * cits / dt, "unit": UNIT, "cores": threads, "kind": ck,
               "sample": f"{threads} concurrent reference bcg_solve calls x {CPU_SAMPLE_ITERS} "
                         f"iterations on the same C2 inputs, {dt:.1f} s wall (incl. per-solve "
                         "setup and final residual)"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded generators, DESIGN.md §Inputs)",
            "config": {"workload": desc, "n": n, "nnz": nnz, "k": k, "p": p, "mode": mode,
                       "tol": tol, "iterations_per_solve": its[0],
                       "l2": "inputs larger than L2 (one block vector = "
                             f"{8 * n * k / 1e6:.0f} MB > 126 MB)",
                       "parallelism": "single GPU" if ws == 1 else f"{ws} replicas (weak)"},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic, "kernel": names[dom],
                         "kernel_ms": prof[dom], "kernel_share": float(shares[dom]),
                         "algorithmic_bytes_per_launch": kbytes[dom], "peak_source": peak_src,
                         "per_kernel_ms": {nm: float(v) for nm, v in zip(names, prof[:3])},
                         "iteration_model_bytes": iter_bytes_model,
                         "iteration_model_frac": iter_bytes_model / (iter_ms * 1e-3) / 1e9 / peak,
                         "iteration_fused_bytes": kbytes[3],
                         "iteration_fused_frac": kbytes[3] / (iter_ms * 1e-3) / 1e9 / peak},
            "cpu_baseline": cpu,
            "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": d2h, "steps": e2e_steps},
            "clocks": clocks.summary(),
            "gpu_launches": launches,
        }
        print(json.dumps(line), flush=True)
    if dist:
        tdist.destroy_process_group()
    return 0


def run_partitioned(args, bk, ctx, stream, a, b, cfg, timed, rank, ws, local):
    """N > 1: one C2 system, rows split into N contiguous slabs (z-slabs of the
    lexicographic grid), one slab per rank; halo of P with ncclSend/Recv,
    Gram partials with ncclAllReduce (paper_1912_11930_b200/partitioned.py).
    Strong scaling: value = k * iterations / (max-over-ranks solve time)."""
    import torch
    import torch.distributed as tdist
    from paper_1912_11930_b200.partitioned import (PartitionedSolver, local_csr, nccl_unique_id,
                                                   row_blocks)
    kind, nx, ny, nz, k, p, mode, rhs, tol, max_iter, desc = CONFIGS[args.config]
    n, nnz = a.n(), a.nnz()
    rb = row_blocks(n, ws)
    r0, r1 = rb[rank], rb[rank + 1]
    lrp, cols, vals = local_csr(a, r0, r1)
    obj = [nccl_unique_id() if rank == 0 else None]
    tdist.broadcast_object_list(obj, src=0)
    nid = obj[0]
    s = PartitionedSolver.nccl(n, r0, r1, lrp, cols, vals, cfg, rank, ws, nid, ctx)
    s.set_rhs(b[r0:r1])
    for _ in range(args.warmup):
        s.run(tol, max_iter)
    launches0 = ctx.launch_count()
    with ClockSampler(local) as clocks:
        ms, reps = timed(lambda: s.run(tol, max_iter)[0], args.steps)
    launches = ctx.launch_count() - launches0
    its = [int(r.iterations) for r in reps]
    value = k * sum(its) / (ms * 1e-3)
    s.close()

    # e2e: host slab in (CSR + B), X slab out, through the partitioned API
    def e2e_step():
        t = PartitionedSolver.nccl(n, r0, r1, lrp, cols, vals, cfg, rank, ws, nid, ctx)
        t.set_rhs(b[r0:r1])
        rep, _ = t.run(tol, max_iter)
        t.x()
        t.close()
        return int(rep.iterations)

    e2e_ms, e2e_its = timed(e2e_step, 1)
    nloc = r1 - r0
    h2d = 8 * (nloc + 1) + 16 * len(vals) + 8 * nloc * k
    line = None
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded generators, DESIGN.md §Inputs)",
            "config": {"workload": desc, "n": n, "nnz": nnz, "k": k, "p": p, "mode": mode,
                       "tol": tol, "iterations_per_solve": its[0],
                       "parallelism": f"row-partitioned x{ws} (z-slabs), NCCL halo + allreduce",
                       "l2": "inputs larger than L2 per rank"},
            "roofline": None, "cpu_baseline": None,
            "e2e": {"value": k * sum(e2e_its) / (e2e_ms * 1e-3), "unit": UNIT,
                    "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": 8 * nloc * k},
            "clocks": clocks.summary(), "gpu_launches": launches,
        }
        print(json.dumps(line), flush=True)
    tdist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="c2", choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline sample")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
