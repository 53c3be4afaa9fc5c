"""The CPU oracle (oracle/bcg_oracle.c) pinned against the reference.

(a) frozen generator goldens of the reference's own tests
    (proj/tests/test_problems.cpp:67-78);
(b) the committed fixtures tests/golden/*.npz produced by the reference
    itself (oracle/_ref, tests/golden/make_golden.py) — bit-for-bit;
(c) the live reference library, when it is present in this container.
"""
import hashlib

import numpy as np
import pytest

import golden_io
from cases import BY_NAME, build_inputs


def test_rng_stream_is_frozen(port):
    # test_problems.cpp:67-78
    v = port.rng_symmetric(7, 4)
    assert v.tolist() == [-0.83658888099278883, -0.48347120732218873, -0.29183092906755803,
                          0.10674871259488627]
    b = port.random_block_rhs(3, 2, 42)
    assert b[0, 0] == -0.61178816493163479
    assert b[0, 1] == 0.12526365453124133
    assert b[2, 1] == 0.16404302513089042


@pytest.mark.parametrize("name", golden_io.names())
def test_port_reproduces_reference_fixture(port, name):
    g = golden_io.load(name)
    case = BY_NAME[name]
    csr, b, x0 = build_inputs(case, port)
    assert hashlib.sha256(b.tobytes()).hexdigest() == g["meta"]["b_sha256"]
    out = port.bcg_solve(csr, b, case.p, case.glob, x0=x0, tol=case.tol, max_iter=case.max_iter,
                         record_history=True, precond=case.precond)
    m = g["meta"]
    r = out.report
    assert r.iterations == m["iterations"]
    assert r.converged == m["converged"]
    assert r.breakdown == m["breakdown"]
    assert r.breakdown_iteration == m["breakdown_iteration"]
    assert r.breakdown_block == m["breakdown_block"]
    for key in ("flops_bdot", "flops_baxpy", "flops_bop", "flops_precond"):
        assert getattr(r, key) == m[key], key
    assert out.history.tobytes() == g["history"].tobytes()
    assert out.final_norms.tobytes() == g["final_norms"].tobytes()
    assert hashlib.sha256(out.x.tobytes()).hexdigest() == m["x_sha256"]


def _csr_small(port):
    from oracle import POISSON2D_LOGUNI
    return port.stencil(POISSON2D_LOGUNI, 5, 5, seed=77)


@pytest.mark.parametrize("k,p,glob", [(4, 1, 0), (4, 2, 0), (4, 2, 1), (8, 4, 1), (8, 8, 0),
                                      (9, 3, 0), (6, 3, 1), (3, 1, 0)])
def test_port_kernels_match_live_reference(port, ref, k, p, glob):
    n = 25
    x = port.random_block_rhs(n, k, 3)
    y = port.random_block_rhs(n, k, 4)
    assert port.bdot(x, y, p, glob).tobytes() == ref.bdot(x, y, p, glob).tobytes()
    blocks = 1 if glob else k // p
    gam = port.rng_symmetric(33, blocks * p * p)
    assert port.baxpy(x, y, gam, p, glob).tobytes() == ref.baxpy(x, y, gam, p, glob).tobytes()
    csr = _csr_small(port)
    assert port.bop(csr, x).tobytes() == ref.bop(csr, x).tobytes()
    assert port.column_norms(x).tobytes() == ref.column_norms(x).tobytes()
    g = port.bdot(x, x, p, glob) + np.eye(p)
    d = port.bdot(x, y, p, glob)
    o1, b1 = port.bsolve(g, d, k, p, glob)
    o2, b2 = ref.bsolve(g, d, k, p, glob)
    assert b1 == b2 and o1.tobytes() == o2.tobytes()


def test_port_generators_match_live_reference(port, ref):
    from oracle import POISSON2D_CONST, POISSON2D_LOGUNI
    for kind in (POISSON2D_CONST, POISSON2D_LOGUNI):
        for nx, ny in ((2, 2), (5, 3), (16, 16)):
            a = port.stencil(kind, nx, ny, seed=7)
            b = ref.stencil(kind, nx, ny, seed=7)
            assert all(u.tobytes() == v.tobytes() for u, v in zip(a, b))
    assert port.random_block_rhs(17, 5, 9).tobytes() == ref.random_block_rhs(17, 5, 9).tobytes()


def test_port_bsolve_breakdown_index(port):
    # test_kernels.cpp:327-342: block 1 rank deficient
    g = np.zeros((2, 2, 2))
    g[0] = np.eye(2)
    g[1] = [[1.0, 2.0], [1.0, 2.0]]
    d = np.zeros((2, 2, 2))
    d[0] = d[1] = np.eye(2)
    _, bad = port.bsolve(g, d, 4, 2, False)
    assert bad == 1
