"""paper_1912_11930_b200 — B200-native Block Conjugate Gradients (arXiv 1912.11930).

The host API mirrors the reference ``blockkrylov`` C++ headers (see
``blockkrylov.py`` and the C++ drop-in headers under ``include/blockkrylov``);
the hot path runs in hand-written sm_100a kernels in ``_build/libbkgpu.so``
behind the C ABI of ``include/bkg.h``.
"""
from .blockkrylov import *  # noqa: F401,F403
from .blockkrylov import (BlockCoefficient, BreakdownError, ConfigError, Context,  # noqa: F401
                          DimensionError, FlopCounter, Preconditioner, SolveOptions, SparseMatrix,
                          SubalgebraConfig, baxpy, bcg_solve, bdot, bop, bsolve, column_norms,
                          default_context, set_numerics)
from .generate import DeviceMatrix  # noqa: F401
from .resident import DeviceSolver  # noqa: F401
from .textio import (IoError, load_block_vector, load_matrix_market,  # noqa: F401
                     save_block_vector, save_matrix_market)

__version__ = "0.1.0"
