#!/usr/bin/env python3
"""Host-timer breakdown of one drop-in bcg_solve call from pinned buffers (C2)."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_1912_11930_b200 as bk  # noqa: E402
from paper_1912_11930_b200 import _native as N  # noqa: E402

cfg_name = sys.argv[1] if len(sys.argv) > 1 and not sys.argv[1].startswith("-") else "c2"
kind, nx, ny, nz, k, p, mode, rhs, tol, max_iter, desc = bench.CONFIGS[cfg_name]
a, b = bench.make_inputs(cfg_name, bk)
n, nnz = a.n(), a.nnz()
pin = lambda shape, dt: torch.empty(shape, dtype=dt, pin_memory=True).numpy()
pb = pin((n, k), torch.float64); pb[...] = b
po = pin(n + 1, torch.int64).view(np.uint64); po[...] = a.row_offsets()
pc = pin(nnz, torch.int64).view(np.uint64); pc[...] = a.col_indices()
pv = pin(nnz, torch.float64); pv[...] = a.values()
px = pin((n, k), torch.float64)
ctx = bk.Context(0, "fast")
cfg = bk.SubalgebraConfig(k, p, mode)
m = bk.Preconditioner.identity(n)
if "--after-resident" in sys.argv:  # the bench's order: resident runs first
    s = bk.DeviceSolver(a, cfg, ctx)
    s.set_rhs(b)
    for _ in range(8):
        s.run(tol, max_iter)
    s.close()
for it in range(4):
    t0 = time.perf_counter()
    am = bk.SparseMatrix(n, po, pc, pv, validate=False)
    h = am.device(ctx)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    res = bk.bcg_solve(am, pb, m, cfg, bk.SolveOptions(tol=tol, max_iter=max_iter), ctx=ctx, out=px)
    t2 = time.perf_counter()
    am.release_device()
    t3 = time.perf_counter()
    print(f"matrix_create {1e3*(t1-t0):.1f} ms  bcg_solve {1e3*(t2-t1):.1f} ms "
          f"(loop {1e3*res.report.loop_seconds:.1f} ms)  release {1e3*(t3-t2):.1f} ms")
