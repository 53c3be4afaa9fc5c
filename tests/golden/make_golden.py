"""Generate tests/golden/*.npz from the UNMODIFIED reference.

Runs in the build container only (needs oracle/_ref/libbkref.so, compiled from
/root/reference by oracle/Makefile).  Inputs come from the oracle's generators
(which tests/test_oracle.py pins to the reference's poisson2d /
random_block_rhs bit-for-bit); the solve itself is the reference's
blockkrylov::bcg_solve.  Each fixture stores the full defect history, the
report integers, the final true-residual norms, the SHA-256 of X's bytes and a
few rows of X.

    python tests/golden/make_golden.py [case ...]
"""
from __future__ import annotations

import hashlib
import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, os.path.join(ROOT, "oracle"))
sys.path.insert(0, os.path.join(ROOT, "tests"))

from oracle import Oracle  # noqa: E402
from cases import BY_NAME, CASES, FULL_NAMES, build_inputs  # noqa: E402


def sample_rows(n):
    idx = sorted(set([0, 1, 2, n // 3, n // 2, n - 2, n - 1]))
    return np.array(idx, dtype=np.int64)


def reversed_system(csr, b, x0):
    """J A J, J B, J X0 with J the row-reversal permutation: the same maths in
    a different summation order (SURVEY.md §8c self-consistency floor)."""
    rp, cols, vals = csr
    n = len(rp) - 1
    cnt = np.diff(rp.astype(np.int64))[::-1]
    nrp = np.zeros(n + 1, np.uint64)
    nrp[1:] = np.cumsum(cnt)
    nc, nv = [], []
    for r in range(n - 1, -1, -1):
        s, e = int(rp[r]), int(rp[r + 1])
        nc.append((n - 1 - cols[s:e].astype(np.int64))[::-1])
        nv.append(vals[s:e][::-1])
    return ((nrp, np.concatenate(nc).astype(np.uint64), np.concatenate(nv)), b[::-1].copy(),
            None if x0 is None else x0[::-1].copy())


def floor_of(case, port, csr, b, x0, out):
    """The reference's own drift under row reversal (port == reference bitwise)."""
    csr2, b2, x02 = reversed_system(csr, b, x0)
    o2 = port.bcg_solve(csr2, b2, case.p, case.glob, x0=x02, tol=case.tol,
                        max_iter=case.max_iter, record_history=True, precond=case.precond)
    rows = min(len(out.history), len(o2.history))
    h, h2 = out.history[:rows], o2.history[:rows]
    drift = float(np.max(np.abs(h - h2) / np.maximum(h, 1e-300))) if rows else 0.0
    x2 = o2.x[::-1]
    xd = float(np.max(np.linalg.norm(out.x - x2, axis=0) /
                      np.maximum(np.linalg.norm(out.x, axis=0), 1e-300)))
    return dict(floor_hist_drift=drift, floor_x_drift=xd,
                floor_iterations=int(o2.report.iterations))


def make(case, ref, port):
    csr, b, x0 = build_inputs(case, port)
    t0 = time.time()
    out = ref.bcg_solve(csr, b, case.p, case.glob, x0=x0, tol=case.tol, max_iter=case.max_iter,
                        record_history=True, precond=case.precond)
    dt = time.time() - t0
    r = out.report
    n = b.shape[0]
    rows = sample_rows(n)
    meta = dict(case=case.name, iterations=int(r.iterations), converged=int(r.converged),
                breakdown=int(r.breakdown), breakdown_iteration=int(r.breakdown_iteration),
                breakdown_block=int(r.breakdown_block), flops_bdot=int(r.flops_bdot),
                flops_baxpy=int(r.flops_baxpy), flops_bop=int(r.flops_bop),
                flops_precond=int(r.flops_precond), history_rows=int(r.history_rows),
                x_sha256=hashlib.sha256(out.x.tobytes()).hexdigest(),
                b_sha256=hashlib.sha256(b.tobytes()).hexdigest(),
                n=int(n), nnz=int(csr[0][-1]), ref_seconds=dt, source="oracle/_ref/libbkref.so")
    meta["full"] = case.name in FULL_NAMES
    if not meta["full"]:
        meta.update(floor_of(case, port, csr, b, x0, out))
    np.savez_compressed(os.path.join(HERE, f"{case.name}.npz"), history=out.history,
                        final_norms=out.final_norms, x_rows=rows, x_sample=out.x[rows],
                        meta=np.array(json.dumps(meta)))
    print(f"{case.name}: it={r.iterations} conv={r.converged} bd={r.breakdown} {dt:.2f}s "
          f"floor drift={meta.get('floor_hist_drift', float('nan')):.2e} "
          f"it={meta.get('floor_iterations', -1)}", flush=True)


def main(names):
    ref = Oracle("reference")
    port = Oracle("port")
    todo = [BY_NAME[n] for n in names] if names else CASES
    for c in todo:
        make(c, ref, port)


if __name__ == "__main__":
    main(sys.argv[1:])
