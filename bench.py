#!/usr/bin/env python3
"""Block-CG throughput bench (BASELINE.json metric: RHS*iterations/s, FP64).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c5] [--impl ours|reference]

Workload (config.workload), default `c5` = BASELINE.json configs[4], the
largest configuration that fits one B200: 3D 7-point Poisson on the 256^3
subgrid (n = 16,777,216, CSR FP64, 117M nonzeros), k = 64 right-hand sides
B ~ N(0,1) (seed 7), X0 = 0, hybrid subalgebra p = 16, fixed 100 iterations.
One *step* = one complete 100-iteration solve.  Other configs (`--config
c1|c2|c3p|c3g|c4c|c4h|c4g`) are secondary lines; `c5_384` is the BASELINE
384^3 system for N >= 2 GPUs.

value  : k * iterations / device time, inputs resident in HBM (DeviceSolver),
         CUDA events on the library stream, W warm-up solves first.  One
         block vector is 8.6 GB > 126 MB L2: every step streams from HBM.
e2e    : the same metric through the public drop-in call
         blockkrylov.bcg_solve(A, B, M, cfg, opts) from pinned host buffers:
         CSR + B uploaded and X downloaded inside every timed step.
roofline: per-kernel CUDA-event times from an untimed profiling pass on the
         library stream; achieved = algorithmic bytes per launch (DESIGN.md
         §4) / time; traffic = ncu DRAM bytes of the same kernel on the same
         config (profiles/ncu_traffic.json, written by tools/ncu_summary.py).
cpu_baseline: the reference CPU solver (oracle/_ref = the unmodified
         reference compiled here) on this host's cores, iterations timed by
         the reference's own on_iterate observer on a bounded slab of the
         workload, scaled to the full system by the paper's traffic model.
--impl reference: that reference CPU measurement alone; imports nothing
         from paper_1912_11930_b200 (inputs from the oracle's generators).

Multi-GPU: `--gpus N` (N > 1) relaunches itself under torch.distributed.run
when WORLD_SIZE is unset.  Each rank generates its own z-slab of A and B on
its device; halo of P over NVLink (NCCL send/recv on a side stream,
overlapped with the interior rows of K1), Gram partials by ncclAllReduce
(paper_1912_11930_b200/partitioned.py).  Default config: strong scaling of
the same 256^3 C5 system (value = k * iterations / max-over-ranks time).
"""
from __future__ import annotations

import argparse
import json
import os
import socket
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "BCG RHS·iterations/sec (FP64) and achieved HBM fraction at 1/2/4/8 B200"
UNIT = "RHS·iterations/s"

# name: (kind, nx, ny, nz, k, p, mode, rhs, tol, max_iter, description)
CONFIGS = {
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
    "c5_384": (3, 384, 384, 384, 64, 16, "hybrid", "normal", 1e-300, 100,
               "C5 3D 7-pt 384^3 z-slabs, k=64, hybrid p=16, fixed 100 iterations (N >= 2)"),
}
DEFAULT_CONFIG = "c5"
RHS_SEED = 7
COEFF_SEED = 11
CPU_SAMPLE_ITERS = 2
CPU_SAMPLE_DOUBLES = 1 << 26  # rows x k of the CPU sample slab (~0.5 GB per block vector)
STENCIL_NNZ_PER_ROW = {0: 5, 1: 5, 2: 5, 3: 7, 4: 27}


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def config_dict(name, n, nnz, ws, extra=None):
    """The `config` object; identical in both arms (same_config)."""
    kind, nx, ny, nz, k, p, mode, rhs, tol, max_iter, desc = CONFIGS[name]
    d = {"workload": desc, "name": name, "grid": [nx, ny, nz], "n": n, "nnz": nnz, "k": k,
         "p": p, "mode": mode, "tol": tol, "max_iter": max_iter, "rhs": rhs,
         "l2": f"inputs larger than L2: one block vector = {8 * n * k / 1e6:.0f} MB vs 126 MB"
               if 8 * n * k > 126e6 else
               f"block vectors {8 * n * k / 1e6:.1f} MB fit in the 126 MB L2 (latency-bound "
               "small system; no flush)",
         "parallelism": "single GPU" if ws == 1 else f"row-partitioned x{ws} (z-slabs)"}
    if extra:
        d.update(extra)
    return d


def stencil_size(name):
    kind, nx, ny, nz, k = CONFIGS[name][:5]
    n = nx * ny * nz
    if kind == 4:
        nnz = (3 * nx - 2) * (3 * ny - 2) * (3 * nz - 2)
    elif kind == 3:
        nnz = n + 2 * ((nx - 1) * ny * nz + nx * (ny - 1) * nz + nx * ny * (nz - 1))
    else:
        nnz = n + 2 * ((nx - 1) * ny + nx * (ny - 1))
    return n, nnz


def model_bytes(n, nnz, k):
    """Paper Table 1 beta summed over one iteration."""
    return 8.0 * (2 * nnz + 17 * n * k)


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


def ncu_traffic(config, kernel_class):
    """Per-launch DRAM bytes of the kernel class on this config, from the
    committed ncu summary (tools/ncu_summary.py); None (and a warning) when
    that (config, kernel) pair was never captured."""
    path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        with open(path) as f:
            ent = json.load(f).get(config, {}).get(kernel_class)
    except (OSError, ValueError):
        ent = None
    if ent is None:
        log(f"WARNING: no ncu traffic for ({config}, {kernel_class}) in {path}")
        return None, None
    return float(ent["dram_bytes"]), ent.get("source")


# ------------------------------------------------------------ CPU baseline --
def cpu_sample_grid(cfg_name):
    """A slab of the workload's grid (same stencil, k, p, mode) small enough
    for a CPU sample: whole planes (3D) or lines (2D) of the full grid."""
    kind, nx, ny, nz, k = CONFIGS[cfg_name][:5]
    if nz > 1:
        plane = nx * ny
        nzs = max(3, min(nz, CPU_SAMPLE_DOUBLES // (plane * k)))
        return nx, ny, nzs
    nys = max(3, min(ny, CPU_SAMPLE_DOUBLES // (nx * k)))
    return nx, nys, 1


def cpu_threads_for(n, k):
    cores = os.cpu_count() or 1
    try:
        import psutil
        avail = psutil.virtual_memory().available
    except Exception:
        avail = 32 << 30
    per_solve = 8 * n * k * 8  # x, r, q, p, z, b copy, final ax + slack (solver.hpp:121-208)
    return max(1, min(cores, int(avail * 0.5 // per_solve)))


class CpuSample:
    """The reference CPU solver on a bounded slab of the workload.  Inputs come
    from the oracle's generators (bit-identical to the product's, tests/
    test_generators.py), so this never imports paper_1912_11930_b200."""

    def __init__(self, cfg_name, threads=None):
        sys.path.insert(0, os.path.join(ROOT, "oracle"))
        from oracle import Oracle, available
        self.kind = "reference" if available("reference") else "port"
        self.orc = Oracle(self.kind)
        gen = Oracle("port")
        kind, nx, ny, nz, k, p, mode, rhs, tol, max_iter, desc = CONFIGS[cfg_name]
        self.k, self.p, self.glob = k, p, mode == "global"
        sx, sy, sz = cpu_sample_grid(cfg_name)
        self.grid = (sx, sy, sz)
        self.csr = gen.stencil(kind, sx, sy, sz, seed=COEFF_SEED if kind == 2 else 0)
        self.n = len(self.csr[0]) - 1
        self.nnz = int(self.csr[0][-1])
        self.b = (gen.normal_block_rhs(self.n, k, RHS_SEED) if rhs == "normal"
                  else gen.random_block_rhs(self.n, k, RHS_SEED))
        n_full, nnz_full = stencil_size(cfg_name)
        # per-iteration cost of the reference is linear in its row loops:
        # scale by the paper's traffic model (Table 1 beta)
        self.scale = model_bytes(n_full, nnz_full, k) / model_bytes(self.n, self.nnz, k)
        self.threads = threads or cpu_threads_for(self.n, k)

    def step(self):
        """(seconds, iterations) of one sample: `threads` concurrent solves x
        CPU_SAMPLE_ITERS iterations (reference: observer-timed loop window)."""
        if self.kind == "reference":
            return self.orc.bench_iterations(self.threads, self.csr, self.b, self.p, self.glob,
                                             CPU_SAMPLE_ITERS)
        return self.orc.bench_solve(self.threads, self.csr, self.b, self.p, self.glob, 1e-300,
                                    CPU_SAMPLE_ITERS)

    def value(self, dt, its):
        return self.k * its / (dt * self.scale)

    def describe(self, dt):
        sx, sy, sz = self.grid
        how = ("iterations 1..{} timed by the reference's on_iterate observer (setup and final "
               "residual excluded)".format(CPU_SAMPLE_ITERS) if self.kind == "reference" else
               "whole-solve wall time incl. setup")
        return (f"{self.threads} concurrent reference bcg_solve calls on a {sx}x{sy}x{sz} slab "
                f"of the workload grid (n={self.n}, same stencil/k/p/mode), {how}; {dt:.2f} s; "
                f"RHS*it/s scaled to the full system by the Table-1 traffic ratio "
                f"{self.scale:.3f}")


# ----------------------------------------------------------- reference arm --
def run_reference(args):
    ws, rank, _ = dist_env()
    if rank != 0:
        return 0
    cs = CpuSample(args.config)
    n, nnz = stencil_size(args.config)
    for _ in range(args.warmup):
        cs.step()
    total_t = 0.0
    total_it = 0
    for _ in range(args.steps):
        dt, its = cs.step()
        total_t += dt
        total_it += its
    value = cs.value(total_t, total_it)
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * total_t / args.steps,
        "higher_is_better": True, "scaling": scaling_of(args.config, ws), "vs_baseline": None,
        "dtype": "f64", "data": "synthetic (seeded generators, DESIGN.md §6)",
        "config": config_dict(args.config, n, nnz, ws),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cs.threads, "kind": cs.kind,
                         "sample": cs.describe(total_t / args.steps)},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def scaling_of(cfg_name, ws):
    # default config: the same 256^3 system at every N (strong scaling)
    return "strong"


# ----------------------------------------------------------------- our arm --
def run_ours(args):
    import torch
    import paper_1912_11930_b200 as bk
    ws, rank, local = dist_env()
    dist = ws > 1
    if dist:
        import torch.distributed as tdist
        torch.cuda.set_device(local)
        tdist.init_process_group("nccl", device_id=torch.device("cuda", local))
    ctx = bk.Context(local, "fast")
    stream = torch.cuda.ExternalStream(ctx.stream(), device=torch.device("cuda", local))

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
        rc = run_partitioned(args, bk, ctx, timed, rank, ws, local)
        tdist.destroy_process_group()
        return rc

    kind, nx, ny, nz, k, p, mode, rhs, tol, max_iter, desc = CONFIGS[args.config]
    t0 = time.time()
    a, b = make_inputs(args.config, bk)
    n, nnz = a.n(), a.nnz()
    log(f"inputs n={n} nnz={nnz} k={k} ({time.time() - t0:.1f}s)")
    cfg = bk.SubalgebraConfig(k, p, mode)

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
    value = k * total_its / (ms * 1e-3)
    k1_name = solver.k1()
    log(f"value: {args.steps} solves, iterations/solve={its[0]}, {ms / args.steps:.2f} "
        f"ms/solve, {value:.1f} RHS*it/s (K1 = {k1_name})")

    # ---------------- roofline: per-kernel profile pass --------------------
    prof = solver.profile(20)
    kbytes = solver.kernel_bytes()
    names = ["K1_spmm_gram", "K2_update_gram", "K3_update_p"]
    peak, peak_src = measured_peak()
    per_kernel = {}
    for i, nm in enumerate(names):
        ach = kbytes[i] / (prof[i] * 1e-3) / 1e9
        tr, src = ncu_traffic(args.config, nm)
        per_kernel[nm] = {"ms": float(prof[i]), "algorithmic_bytes": float(kbytes[i]),
                          "achieved_gbs": ach, "frac": ach / peak, "ncu_dram_bytes": tr,
                          "ncu_source": src, "share": float(prof[i] / max(prof[3], 1e-30))}
    dom = names[int(np.argmax(prof[:3]))]
    d = per_kernel[dom]
    iter_ms = ms / max(total_its, 1)
    iter_model = model_bytes(n, nnz, k)
    solver.close()

    # ---------------- e2e: public drop-in call, host buffers ---------------
    pin_b = torch.empty((n, k), dtype=torch.float64, pin_memory=True).numpy()
    pin_b[...] = b
    del b
    pin_off = torch.empty(n + 1, dtype=torch.int64, pin_memory=True).numpy().view(np.uint64)
    pin_off[...] = a.row_offsets()
    pin_col = torch.empty(nnz, dtype=torch.int64, pin_memory=True).numpy().view(np.uint64)
    pin_col[...] = a.col_indices()
    pin_val = torch.empty(nnz, dtype=torch.float64, pin_memory=True).numpy()
    pin_val[...] = a.values()
    del a
    pin_x = torch.empty((n, k), dtype=torch.float64, pin_memory=True).numpy()
    m = bk.Preconditioner.identity(n)
    opts = bk.SolveOptions(tol=tol, max_iter=max_iter)

    def e2e_step():
        am = bk.SparseMatrix(n, pin_off, pin_col, pin_val, validate=False)
        res = bk.bcg_solve(am, pin_b, m, cfg, opts, ctx=ctx, out=pin_x)
        am.release_device()
        return res.report.iterations

    e2e_step()  # warm-up (allocator, module load, sliced-ELL build)
    e2e_steps = max(1, min(args.steps, 3))
    e2e_ms, e2e_its = timed(e2e_step, e2e_steps)
    e2e_value = k * sum(e2e_its) / (e2e_ms * 1e-3)
    h2d = 8 * (n + 1) + 16 * nnz + 8 * n * k
    d2h = 8 * n * k + 8 * k

    # ---------------- CPU baseline (N = 1) --------------------------------
    cpu = None
    if not args.no_cpu:
        cs = CpuSample(args.config)
        dt, cits = cs.step()
        cpu = {"value": cs.value(dt, cits), "unit": UNIT, "cores": cs.threads, "kind": cs.kind,
               "sample": cs.describe(dt)}

    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True,
        "scaling": scaling_of(args.config, ws), "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded generators, DESIGN.md §6)",
        "config": config_dict(args.config, n, nnz, ws),
        "iterations_per_solve": its[0], "k1_kernel": k1_name,
        "roofline": {"bound": "hbm", "kernel": dom, "achieved": d["achieved_gbs"], "peak": peak,
                     "unit": "GB/s", "frac": d["frac"], "traffic": d["ncu_dram_bytes"],
                     "traffic_source": d["ncu_source"], "kernel_ms": d["ms"],
                     "kernel_share": d["share"],
                     "algorithmic_bytes_per_launch": d["algorithmic_bytes"],
                     "peak_source": peak_src, "per_kernel": per_kernel,
                     # whole iteration: bytes the fused kernels must move / loop time
                     "iteration_fused_bytes": float(kbytes[3]),
                     "iteration_fused_frac": kbytes[3] / (iter_ms * 1e-3) / 1e9 / peak,
                     # paper Table-1 traffic at the loop time: an EFFECTIVE
                     # bandwidth (the fused kernels move fewer bytes than it)
                     "iteration_model_bytes": iter_model,
                     "iteration_model_effective_gbs": iter_model / (iter_ms * 1e-3) / 1e9},
        "cpu_baseline": cpu,
        "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": d2h, "steps": e2e_steps},
        "clocks": clocks.summary(),
        "gpu_launches": launches,
    }
    print(json.dumps(line), flush=True)
    return 0


def run_partitioned(args, bk, ctx, timed, rank, ws, local):
    """N > 1: one system, rows split into N contiguous z-slabs, one per rank.
    Each rank generates its slab of A (device CSR, global columns) and of B on
    its own GPU.  value = k * iterations / (max-over-ranks solve time)."""
    from paper_1912_11930_b200.partitioned import PartitionedSolver, nccl_unique_id, row_blocks
    import torch.distributed as tdist
    kind, nx, ny, nz, k, p, mode, rhs, tol, max_iter, desc = CONFIGS[args.config]
    n, nnz = stencil_size(args.config)
    rb = row_blocks(n, ws)
    r0, r1 = rb[rank], rb[rank + 1]
    obj = [nccl_unique_id() if rank == 0 else None]
    tdist.broadcast_object_list(obj, src=0)
    nid = obj[0]
    cfg = bk.SubalgebraConfig(k, p, mode)
    t0 = time.time()
    s = PartitionedSolver.nccl_generated(kind, nx, ny, nz, r0, r1, cfg, rank, ws, nid, ctx,
                                         rhs=rhs, seed=RHS_SEED,
                                         coeff_seed=COEFF_SEED if kind == 2 else 0)
    log(f"[rank {rank}] slab rows [{r0}, {r1}) generated on device ({time.time() - t0:.1f}s)")
    for _ in range(args.warmup):
        s.run(tol, max_iter)
    launches0 = ctx.launch_count()
    with ClockSampler(local) as clocks:
        ms, reps = timed(lambda: s.run(tol, max_iter)[0], args.steps)
    launches = ctx.launch_count() - launches0
    its = [int(r.iterations) for r in reps]
    value = k * sum(its) / (ms * 1e-3)

    # e2e: this rank's B slab in from pinned host memory, X slab out, per step
    import torch
    nloc = r1 - r0
    pin_b = torch.empty((nloc, k), dtype=torch.float64, pin_memory=True).numpy()
    pin_b[...] = s.rhs()
    pin_x = torch.empty((nloc, k), dtype=torch.float64, pin_memory=True).numpy()

    def e2e_step():
        s.set_rhs(pin_b)
        rep, _ = s.run(tol, max_iter)
        s.x(out=pin_x)
        return int(rep.iterations)

    e2e_ms, e2e_its = timed(e2e_step, 1)
    s.close()
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True,
            "scaling": scaling_of(args.config, ws), "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded generators, each rank's slab generated on its GPU)",
            "config": config_dict(args.config, n, nnz, ws,
                                  {"halo": "NCCL send/recv on a side stream, overlapped with "
                                           "K1's interior rows",
                                   "allreduce": "ncclAllReduce x2 per iteration"}),
            "iterations_per_solve": its[0],
            # n*k*it/s: the per-row throughput §8(e)'s efficiency is defined on
            "row_rhs_iterations_per_s": n * value,
            "roofline": None, "cpu_baseline": None,
            "e2e": {"value": k * sum(e2e_its) / (e2e_ms * 1e-3), "unit": UNIT,
                    "h2d_bytes_per_step": 8 * nloc * k, "d2h_bytes_per_step": 8 * nloc * k,
                    "note": "per rank: B slab up, X slab down; the device-generated matrix "
                            "stays resident"},
            "clocks": clocks.summary(), "gpu_launches": launches,
        }
        print(json.dumps(line), flush=True)
    return 0


def free_port():
    with socket.socket(socket.AF_INET, socket.SOCK_STREAM) as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def relaunch(args):
    """--gpus N > 1 without a launcher: one process per GPU via torchrun."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr=127.0.0.1",
           f"--master-port={free_port()}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default=DEFAULT_CONFIG, choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline sample")
    args = ap.parse_args()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return relaunch(args)
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
