#!/usr/bin/env python3
"""SM clock while only small solves run: nvidia-smi samples (50 ms) during 3 s
of back-to-back C1 solves, and the per-iteration time.
    python tools/c1_clocks.py"""
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_1912_11930_b200 as bk  # noqa: E402

kind, nx, ny, nz, k, p, mode, rhs, tol, max_iter, desc = bench.CONFIGS["c1"]
a, b = bench.make_inputs("c1", bk)
ctx = bk.Context(0, "fast")
s = bk.DeviceSolver(a, bk.SubalgebraConfig(k, p, mode), ctx)
s.set_rhs(b)
rows = []
proc = subprocess.Popen(["nvidia-smi", "--query-gpu=clocks.sm,clocks.max.sm,pstate,power.draw,utilization.gpu",
                         "--format=csv,noheader,nounits", "-lms", "50"], stdout=subprocess.PIPE, text=True)
t = threading.Thread(target=lambda: [rows.append(l.strip()) for l in proc.stdout], daemon=True)
t.start()
t0 = time.time()
loops, its = [], 0
while time.time() - t0 < 3.0:
    rep = s.run(tol, max_iter)
    loops.append(rep.loop_seconds)
    its = rep.iterations
proc.terminate()
print(f"{len(loops)} solves, {its} iterations each, loop {1e3 * min(loops):.3f} .. {1e3 * max(loops):.3f} ms "
      f"= {1e6 * min(loops) / its:.2f} us / iteration")
print("nvidia-smi samples (sm MHz, max MHz, pstate, W, util%):")
for r in rows[:: max(1, len(rows) // 12)]:
    print("  ", r)
