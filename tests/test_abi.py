"""C-ABI surface checks that need no GPU: the library loads, exports every
symbol include/bkg.h declares, fails loudly without a device, and the host
mirror validates arguments before any launch (test_kernels.cpp:85-89,221-228,
test_solver.cpp:379-393)."""
import ctypes as C
import os
import re

import numpy as np
import pytest

import paper_1912_11930_b200 as bk
from paper_1912_11930_b200 import _native as N

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    src = open(os.path.join(ROOT, "include", "bkg.h")).read()
    return sorted(set(re.findall(r"\b(bkg_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    lib = N.lib()
    syms = header_symbols()
    assert len(syms) >= 30
    missing = [s for s in syms if not hasattr(lib, s)]
    assert not missing, missing
    declared = {name for name, _, _ in N.SIGNATURES}
    assert set(syms) == declared, set(syms) ^ declared


def test_oracle_is_not_linked_by_product():
    so = open(N.LIB_PATH, "rb").read()
    assert b"orc_" not in so and b"bkref_" not in so


def test_no_device_fails_loudly():
    try:
        import torch
        if torch.cuda.is_available():
            pytest.skip("GPU present")
    except ImportError:
        pass
    h = C.c_void_p()
    st = N.lib().bkg_ctx_create(0, C.byref(h))
    assert st == N.BKG_CUDA
    assert "CUDA" in N.last_error() or "device" in N.last_error()


def test_subalgebra_config_mirror():
    # test_kernels.cpp:27-43
    with pytest.raises(bk.ConfigError):
        bk.SubalgebraConfig(8, 3)
    with pytest.raises(bk.ConfigError):
        bk.SubalgebraConfig(0, 1)
    with pytest.raises(bk.ConfigError):
        bk.SubalgebraConfig(4, 0, "global")
    c = bk.SubalgebraConfig.classical(8)
    assert (c.p, c.q, c.mode) == (8, 1, "hybrid")
    c = bk.SubalgebraConfig.parallel(8)
    assert (c.p, c.q, c.mode) == (1, 8, "hybrid")
    assert bk.SubalgebraConfig(8, 2, "global").block_count() == 1


def test_dimension_errors_before_launch():
    cfg = bk.SubalgebraConfig(4, 2)
    with pytest.raises(bk.DimensionError):
        bk.bdot(np.zeros((5, 4)), np.zeros((6, 4)), cfg)
    with pytest.raises(bk.DimensionError):
        bk.bdot(np.zeros((5, 2)), np.zeros((5, 2)), cfg)
    x = np.zeros((5, 4))
    with pytest.raises(bk.DimensionError):
        bk.baxpy(x, np.zeros((6, 4)), bk.BlockCoefficient(cfg))
    with pytest.raises(bk.DimensionError):
        bk.baxpy(x, x, bk.BlockCoefficient(cfg))
    with pytest.raises(bk.DimensionError):
        bk.bsolve(bk.BlockCoefficient.identity(cfg),
                  bk.BlockCoefficient.identity(bk.SubalgebraConfig(4, 2, "global")))
    a = bk.SparseMatrix.from_triplets(4, [(i, i, 1.0) for i in range(4)])
    m = bk.Preconditioner.identity(4)
    c2 = bk.SubalgebraConfig.classical(2)
    b = np.zeros((4, 2))
    with pytest.raises(bk.DimensionError):
        bk.bcg_solve(a, np.zeros((5, 2)), m, c2)
    with pytest.raises(bk.DimensionError):
        bk.bcg_solve(a, np.zeros((4, 3)), m, c2)
    with pytest.raises(bk.DimensionError):
        bk.bcg_solve(a, b, np.zeros((4, 3)), m, c2)
    with pytest.raises(bk.DimensionError):
        bk.bcg_solve(a, b, bk.Preconditioner.identity(5), c2)
    with pytest.raises(bk.ConfigError):
        bk.bcg_solve(a, b, m, c2, bk.SolveOptions(tol=0.0))


def test_sparse_matrix_validation_mirror():
    # sparse_matrix.hpp:89-125
    with pytest.raises(bk.ConfigError):
        bk.SparseMatrix(2, [0, 1, 2], [0, 0], [1.0, 1.0])  # (1,0) without (0,1)
    with pytest.raises(bk.ConfigError):
        bk.SparseMatrix(2, [0, 2, 2], [1, 0], [1.0, 1.0])  # not ascending
    with pytest.raises(bk.ConfigError):
        bk.SparseMatrix(2, [0, 1, 1], [1], [1.0])  # no symmetric counterpart
    with pytest.raises(bk.ConfigError):
        bk.SparseMatrix(2, [0, 2, 4], [0, 1, 0, 1], [2.0, 1.0, 1.1, 2.0])  # values not symmetric
    a = bk.SparseMatrix.from_triplets(3, [(0, 0, 1.0), (0, 0, 1.0), (1, 1, 3.0), (2, 2, 1.0)])
    assert a.at(0, 0) == 2.0 and a.nnz() == 3
