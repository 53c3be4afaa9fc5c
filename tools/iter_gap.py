#!/usr/bin/env python3
"""Graph-launched iteration time vs the per-kernel profile on one config:
    python tools/iter_gap.py [config] [iterations]
Prints ms/iteration of DeviceSolver.run (fixed iteration count, CUDA events
inside the library) next to the sum of the per-kernel event times."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_1912_11930_b200 as bk  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 320
kind, nx, ny, nz, k, p, mode, rhs, tol, max_iter, desc = bench.CONFIGS[cfg]
a, b = bench.make_inputs(cfg, bk)
s = bk.DeviceSolver(a, bk.SubalgebraConfig(k, p, mode))
s.set_rhs(b)
s.run(1e-300, 64)  # warm-up (graph capture)
for rep in range(3):
    t0 = time.perf_counter()
    r = s.run(1e-300, iters)
    wall = time.perf_counter() - t0
    print(f"run: {r.iterations} it, loop {1e3 * r.loop_seconds / r.iterations:.4f} ms/it, "
          f"wall {1e3 * wall / r.iterations:.4f} ms/it")
prof = s.profile(20)
print("profile ms [K1,K2,K3,iter]:", [round(float(x), 4) for x in prof])
