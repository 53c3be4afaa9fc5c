#!/usr/bin/env python3
"""Where a small solve's time goes: loop_seconds (device events around the
loop) vs the whole run() call, resident kernel on/off.
    python tools/c1_latency.py [config]"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_1912_11930_b200 as bk  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c1"
kind, nx, ny, nz, k, p, mode, rhs, tol, max_iter, desc = bench.CONFIGS[cfg]
a, b = bench.make_inputs(cfg, bk)
for res in ("1", "0"):
    os.environ["BKG_RESIDENT"] = res
    ctx = bk.Context(0, "fast")
    s = bk.DeviceSolver(a, bk.SubalgebraConfig(k, p, mode), ctx)
    s.set_rhs(b)
    for cap in (max_iter, max_iter, 1, 1, 50, 50, 100, 100, 200, 200):
        t0 = time.perf_counter()
        rep = s.run(tol, cap)
        t1 = time.perf_counter()
        print(f"resident={res} max_iter {cap}: wall {1e3 * (t1 - t0):.3f} ms, loop {1e3 * rep.loop_seconds:.3f} ms, "
              f"iterations {rep.iterations}, k1 {s.k1()}", flush=True)
    s.close()
    ctx.close()

# Clock check: the same small solves right after a heavy kernel sequence (a
# large fixed-iteration solve).  If the small solve gets much faster, its
# per-iteration time above was set by the idle SM clock, not by the kernel.
import numpy as np  # noqa: E402
os.environ["BKG_RESIDENT"] = "1"
ctx = bk.Context(0, "fast")
big_a = bk.stencil(3, 160, 160, 160, seed=11)
big_b = bk.normal_block_rhs(big_a.n(), 32, 7)
big = bk.DeviceSolver(big_a, bk.SubalgebraConfig(32, 8, "hybrid"), ctx)
big.set_rhs(big_b)
s = bk.DeviceSolver(a, bk.SubalgebraConfig(k, p, mode), ctx)
s.set_rhs(b)
for rep_i in range(3):
    big.run(1e-300, 150)
    for cap in (200, 200, 200):
        rep = s.run(tol, cap)
        print(f"after heavy load: max_iter {cap}: loop {1e3 * rep.loop_seconds:.3f} ms, "
              f"iterations {rep.iterations}", flush=True)
s.close()
big.close()
ctx.close()
