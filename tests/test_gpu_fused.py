"""Fused fast-path building blocks against the oracle: the first K1 launch
(SpMM + alpha Gram + on-device lambda solve) for every tuned (k, p, mode)."""
import numpy as np
import pytest

import paper_1912_11930_b200 as bk

pytestmark = pytest.mark.gpu

SHAPES = [(8, 8, False), (8, 4, True), (16, 16, False), (16, 4, False), (16, 4, True),
          (32, 8, False), (32, 1, False), (64, 16, False), (64, 4, True), (64, 1, False),
          (4, 2, False), (16, 8, True),
          # k = 128: the paper's experiment width
          (128, 16, False), (128, 8, False), (128, 4, True), (128, 1, False)]


@pytest.mark.parametrize("k,p,glob", SHAPES)
@pytest.mark.parametrize("kind,dims", [(3, (9, 7, 5)), (4, (6, 5, 7)), (3, (64, 64, 40)), (0, (256, 200, 1))])
def test_first_step_matches_oracle(port, k, p, glob, kind, dims):
    a = bk.stencil(kind, *dims, seed=11)
    b = bk.normal_block_rhs(a.n(), k, 7)
    ctx = bk.Context(0, "fast")
    s = bk.DeviceSolver(a, bk.SubalgebraConfig(k, p, "global" if glob else "hybrid"), ctx)
    s.set_rhs(b)
    q, coef = s.debug_first_step()
    csr = (a.row_offsets(), a.col_indices(), a.values())
    qref = port.bop(csr, b)
    np.testing.assert_allclose(q, qref, rtol=1e-13, atol=1e-12)
    gl = glob and p != k
    alpha = port.bdot(b, qref, p, gl)
    rho = port.bdot(b, b, p, gl)
    lam, bad = port.bsolve(alpha, rho, k, p, gl)
    assert bad is None
    cs = alpha.size
    np.testing.assert_allclose(coef[cs:], rho.ravel(), rtol=1e-11)
    np.testing.assert_allclose(coef[:cs], lam.ravel(), rtol=1e-9, atol=1e-12)
    s.close()
    ctx.close()
