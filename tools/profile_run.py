#!/usr/bin/env python3
"""Short fused-iteration run for ncu captures: C2 inputs, DeviceSolver.profile.
    python tools/profile_run.py [config] [iterations]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_1912_11930_b200 as bk  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 5
kind, nx, ny, nz, k, p, mode, rhs, tol, max_iter, desc = bench.CONFIGS[cfg]
a, b = bench.make_inputs(cfg, bk)
s = bk.DeviceSolver(a, bk.SubalgebraConfig(k, p, mode))
s.set_rhs(b)
print(cfg, "ms per kernel [K1,K2,K3,iter]:", s.profile(iters))
