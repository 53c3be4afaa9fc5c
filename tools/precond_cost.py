#!/usr/bin/env python3
"""Per-iteration device time of preconditioned solves on a bench config:
    python tools/precond_cost.py [config] [iterations]
identity / Jacobi (fused into K2/K3) / ILU(0) (level-scheduled sweeps), fast
numerics, SolveOptions.time_kernels for the per-class split."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_1912_11930_b200 as bk  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 20
kind, nx, ny, nz, k, p, mode, rhs, tol, max_iter, desc = bench.CONFIGS[cfg]
a, b = bench.make_inputs(cfg, bk)
ctx = bk.Context(0, "fast")
sc = bk.SubalgebraConfig(k, p, mode)
for name in ("identity", "jacobi", "ilu0"):
    t0 = time.perf_counter()
    m = {"identity": lambda: bk.Preconditioner.identity(a.n()),
         "jacobi": lambda: bk.Preconditioner.jacobi(a),
         "ilu0": lambda: bk.ilu0_factor(a, ctx)}[name]()
    setup = time.perf_counter() - t0
    for timed in (False, True):
        opts = bk.SolveOptions(tol=1e-300, max_iter=iters, time_kernels=timed)
        bk.bcg_solve(a, b, m, sc, opts, ctx=ctx)  # warm-up
        t0 = time.perf_counter()
        r = bk.bcg_solve(a, b, m, sc, opts, ctx=ctx).report
        wall = time.perf_counter() - t0
        sec = r.seconds
        print(f"{cfg} {name:8s} timed={int(timed)} it={r.iterations} loop {1e3 * r.loop_seconds / r.iterations:.3f} ms/it "
              f"wall {1e3 * wall:.1f} ms  classes[bdot,baxpy,bop,precond] ms/it = "
              f"{[round(1e3 * x / r.iterations, 3) for x in (sec.bdot, sec.baxpy, sec.bop, sec.precond)]}"
              f"  setup {setup:.2f}s", flush=True)
