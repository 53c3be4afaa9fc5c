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
from cases import BY_NAME, CASES, build_inputs  # noqa: E402


def sample_rows(n):
    idx = sorted(set([0, 1, 2, n // 3, n // 2, n - 2, n - 1]))
    return np.array(idx, dtype=np.int64)


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
    np.savez_compressed(os.path.join(HERE, f"{case.name}.npz"), history=out.history,
                        final_norms=out.final_norms, x_rows=rows, x_sample=out.x[rows],
                        meta=np.array(json.dumps(meta)))
    print(f"{case.name}: it={r.iterations} conv={r.converged} bd={r.breakdown} {dt:.2f}s")


def main(names):
    ref = Oracle("reference")
    port = Oracle("port")
    todo = [BY_NAME[n] for n in names] if names else CASES
    for c in todo:
        make(c, ref, port)


if __name__ == "__main__":
    main(sys.argv[1:])
