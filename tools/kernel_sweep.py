#!/usr/bin/env python3
"""Per-kernel device times of the fused Block-CG iteration for each library
variant under paper_1912_11930_b200/_build/variants/ (or the default build).

    python tools/kernel_sweep.py [--configs c2,c4c,3:96:96:96:32:4:hybrid] [--variants a,b]
                                 [--envs "BKG_K1_STAGE=0;BKG_STAGE_NS=4,BKG_STAGE_CTAS=2"]

Each (variant, env set) runs in its own subprocess (BKG_LIB selects the .so;
--envs: ';'-separated sets of ','-separated NAME=VALUE)."""
import argparse
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
VDIR = os.path.join(ROOT, "paper_1912_11930_b200", "_build", "variants")


def child(cfg, iters):
    sys.path.insert(0, ROOT)
    import numpy as np
    import bench
    import paper_1912_11930_b200 as bk
    if ":" in cfg:  # ad-hoc shape "kind:nx:ny:nz:k:p:mode" (tuning only)
        f = cfg.split(":")
        bench.CONFIGS[cfg] = (int(f[0]), int(f[1]), int(f[2]), int(f[3]), int(f[4]), int(f[5]),
                              f[6], "normal", 1e-8, 0, "ad-hoc")
    kind, nx, ny, nz, k, p, mode, rhs, tol, max_iter, desc = bench.CONFIGS[cfg]
    a, b = bench.make_inputs(cfg, bk)
    s = bk.DeviceSolver(a, bk.SubalgebraConfig(k, p, mode))
    s.set_rhs(b)
    ms = s.profile(iters)
    by = s.kernel_bytes()
    peak, _ = bench.measured_peak()
    out = {"config": cfg, "k1": s.k1(), "ms": [round(float(x), 4) for x in ms],
           "GBps": [round(float(by[i] / (ms[i] * 1e-3) / 1e9), 1) for i in range(4)],
           "frac": [round(float(by[i] / (ms[i] * 1e-3) / 1e9 / peak), 3) for i in range(4)]}
    print(json.dumps(out), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="c2")
    ap.add_argument("--variants", default="")
    ap.add_argument("--iters", type=int, default=20)
    ap.add_argument("--child", default="")
    ap.add_argument("--envs", default="")
    args = ap.parse_args()
    if args.child:
        return child(args.child, args.iters)
    variants = [v for v in args.variants.split(",") if v] or (
        sorted(os.listdir(VDIR)) if os.path.isdir(VDIR) else [])
    variants = variants or ["default"]
    envsets = [e for e in args.envs.split(";") if e] or [""]
    for v in variants:
        for es in envsets:
            env = dict(os.environ)
            if v != "default":
                env["BKG_LIB"] = os.path.join(VDIR, v, "libbkgpu.so")
            for kv in [x for x in es.split(",") if x]:
                name, val = kv.split("=", 1)
                env[name] = val
            for cfg in args.configs.split(","):
                r = subprocess.run([sys.executable, __file__, "--child", cfg, "--iters",
                                    str(args.iters)], env=env, capture_output=True, text=True)
                line = r.stdout.strip().splitlines()[-1] if r.stdout.strip() else r.stderr[-300:]
                print(f"{v:10s} {es:40s} {line}", flush=True)


if __name__ == "__main__":
    sys.exit(main())
