#!/usr/bin/env python3
"""Variable-coefficient 3-D 7-point system (D A D of the constant stencil, D a
random positive diagonal): per-kernel times with k1_grid's DIA path on / off.
    python tools/var3d_probe.py [n1d] [k] [p]"""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def child(n1, k, p):
    import numpy as np
    import paper_1912_11930_b200 as bk
    a0 = bk.stencil(3, n1, n1, n1, seed=11)
    rp, ci, v = a0.row_offsets(), a0.col_indices(), a0.values()
    n = a0.n()
    d = np.exp(0.5 * np.random.default_rng(5).standard_normal(n))
    rows = np.repeat(np.arange(n), np.diff(rp.astype(np.int64)))
    v2 = v * d[rows] * d[ci.astype(np.int64)]
    a = bk.SparseMatrix(n, rp, ci, v2, validate=False)
    b = bk.normal_block_rhs(n, k, 7)
    s = bk.DeviceSolver(a, bk.SubalgebraConfig(k, p, "hybrid"))
    s.set_rhs(b)
    ms = s.profile(20)
    print(f"VAR={os.environ.get('BKG_GRID_VAR')} n={n} k={k} p={p} k1={s.k1()} "
          f"ms K1,K2,K3,iter = {[round(float(x), 4) for x in ms]}", flush=True)


if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "--child":
        child(int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4]))
    else:
        n1 = sys.argv[1] if len(sys.argv) > 1 else "128"
        k = sys.argv[2] if len(sys.argv) > 2 else "32"
        p = sys.argv[3] if len(sys.argv) > 3 else "8"
        for var in ("1", "0"):
            env = dict(os.environ, BKG_GRID_VAR=var)
            subprocess.run([sys.executable, __file__, "--child", n1, k, p], env=env)
