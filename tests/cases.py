"""Parity case registry shared by the golden generator and the tests.

Each case names an input (matrix generator + RHS generator, all seeded) and a
solver configuration.  Shapes follow BASELINE.json's configs C1-C5; the ones
the CPU oracle cannot finish in seconds are reduced grids of the same
generator, k, p and subalgebra.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Optional

# matrix kinds (oracle.orc_stencil_* / bkg_stencil_*)
POISSON2D_CONST, POISSON2D_LOGUNI, DIFFUSION2D_LOGNORMAL, LAPLACE3D_7PT, STENCIL3D_27PT = range(5)

RHS_SEED = 7     # acceptance_test.cpp:35-37 uses seed 7 for the reference instance
COEFF_SEED = 11  # C3 lognormal field


@dataclass(frozen=True)
class Case:
    name: str
    kind: int
    nx: int
    ny: int
    nz: int
    k: int
    p: int
    glob: bool
    rhs: str              # "normal" | "uniform"
    tol: float = 1e-8
    max_iter: int = 0
    coeff_seed: int = 0
    contrast: float = 2.0
    precond: str = "identity"
    x0_seed: Optional[int] = None
    dup_col: Optional[int] = None   # copy column 0 into this column (rank deficiency)
    zero_rhs: bool = False

    @property
    def mode(self) -> str:
        return "global" if self.glob else "hybrid"


def _c1(name, p, glob):
    return Case(name, POISSON2D_CONST, 128, 128, 1, 8, p, glob, "normal", 1e-8, 500)


CASES = [
    # C1 at full size: 2D 5-pt Poisson 128^2, k=8, N(0,1), stop 1e-8 or 500
    _c1("c1_classical", 8, False),
    _c1("c1_hybrid4", 4, False),
    _c1("c1_global4", 4, True),
    _c1("c1_parallel", 1, False),
    # reference acceptance instance (acceptance_test.cpp:33-37): het. Poisson 32^2 seed 7
    Case("acc32_p1", POISSON2D_LOGUNI, 32, 32, 1, 8, 1, False, "uniform", coeff_seed=7),
    Case("acc32_p2", POISSON2D_LOGUNI, 32, 32, 1, 8, 2, False, "uniform", coeff_seed=7),
    Case("acc32_p4", POISSON2D_LOGUNI, 32, 32, 1, 8, 4, False, "uniform", coeff_seed=7),
    Case("acc32_p8", POISSON2D_LOGUNI, 32, 32, 1, 8, 8, False, "uniform", coeff_seed=7),
    Case("acc32_g2", POISSON2D_LOGUNI, 32, 32, 1, 8, 2, True, "uniform", coeff_seed=7),
    Case("acc32_g4", POISSON2D_LOGUNI, 32, 32, 1, 8, 4, True, "uniform", coeff_seed=7),
    # C2 reduced: 3D 7-pt, k=32, hybrid p=8
    Case("c2_24", LAPLACE3D_7PT, 24, 24, 24, 32, 8, False, "normal"),
    # C3 reduced: 2D lognormal diffusion, k=64, parallel vs global p=4
    Case("c3_48_parallel", DIFFUSION2D_LOGNORMAL, 48, 48, 1, 64, 1, False, "uniform",
         coeff_seed=COEFF_SEED),
    Case("c3_48_global4", DIFFUSION2D_LOGNORMAL, 48, 48, 1, 64, 4, True, "uniform",
         coeff_seed=COEFF_SEED),
    # C4 reduced: 3D 27-pt, k=16: classical / hybrid p=4 / global p=4, 200-iteration cap
    Case("c4_14_classical", STENCIL3D_27PT, 14, 14, 14, 16, 16, False, "normal", 1e-8, 200),
    Case("c4_14_hybrid4", STENCIL3D_27PT, 14, 14, 14, 16, 4, False, "normal", 1e-8, 200),
    Case("c4_14_global4", STENCIL3D_27PT, 14, 14, 14, 16, 4, True, "normal", 1e-8, 200),
    # C5 reduced: 3D 7-pt, k=64, hybrid p=16, 100-iteration cap
    Case("c5_16", LAPLACE3D_7PT, 16, 16, 16, 64, 16, False, "normal", 1e-8, 100),
    # solver semantics (test_solver.cpp): nonzero X0, breakdown, max_iter, zero RHS
    Case("x0_classical4", POISSON2D_LOGUNI, 8, 8, 1, 4, 4, False, "uniform", 1e-10,
         coeff_seed=3, x0_seed=99),
    Case("dup_breakdown", POISSON2D_LOGUNI, 8, 8, 1, 4, 4, False, "uniform", coeff_seed=7,
         dup_col=3),
    Case("maxiter3", POISSON2D_LOGUNI, 8, 8, 1, 2, 2, False, "uniform", 1e-30, 3, coeff_seed=41),
    Case("zero_rhs", POISSON2D_CONST, 8, 8, 1, 2, 2, False, "uniform", zero_rhs=True),
    # preconditioned (preconditioners.hpp): the reference's own tests run ILU(0)
    # (acceptance_test.cpp:70-99 OracleCorrectness instance; test_solver.cpp)
    Case("acc32_ilu_p1", POISSON2D_LOGUNI, 32, 32, 1, 8, 1, False, "uniform", coeff_seed=7,
         precond="ilu0"),
    Case("acc32_ilu_p2", POISSON2D_LOGUNI, 32, 32, 1, 8, 2, False, "uniform", coeff_seed=7,
         precond="ilu0"),
    Case("acc32_ilu_p4", POISSON2D_LOGUNI, 32, 32, 1, 8, 4, False, "uniform", coeff_seed=7,
         precond="ilu0"),
    Case("acc32_ilu_p8", POISSON2D_LOGUNI, 32, 32, 1, 8, 8, False, "uniform", coeff_seed=7,
         precond="ilu0"),
    Case("acc32_ilu_g4", POISSON2D_LOGUNI, 32, 32, 1, 8, 4, True, "uniform", coeff_seed=7,
         precond="ilu0"),
    Case("acc32_jacobi_p4", POISSON2D_LOGUNI, 32, 32, 1, 8, 4, False, "uniform", coeff_seed=7,
         precond="jacobi"),
    Case("c2_16_ilu", LAPLACE3D_7PT, 16, 16, 16, 32, 8, False, "normal", precond="ilu0"),
    Case("c2_16_jacobi", LAPLACE3D_7PT, 16, 16, 16, 32, 8, False, "normal", precond="jacobi"),
    Case("x0_ilu_classical4", POISSON2D_LOGUNI, 8, 8, 1, 4, 4, False, "uniform", 1e-10,
         coeff_seed=3, x0_seed=99, precond="ilu0"),
    Case("dup_breakdown_ilu", POISSON2D_LOGUNI, 8, 8, 1, 4, 4, False, "uniform", coeff_seed=7,
         dup_col=3, precond="ilu0"),
]

# Full-size BASELINE configs whose reference solve takes minutes to hours on
# one core: fixtures are produced once in the background (make_golden.py
# --full) and checked on the GPU (exact: bit-identical; fast: bars).
FULL_CASES = [
    Case("c2_full", LAPLACE3D_7PT, 128, 128, 128, 32, 8, False, "normal"),
    Case("c4_full_classical", STENCIL3D_27PT, 192, 192, 192, 16, 16, False, "normal", 1e-300,
         200),
    Case("c4_full_hybrid4", STENCIL3D_27PT, 192, 192, 192, 16, 4, False, "normal", 1e-300, 200),
    Case("c4_full_global4", STENCIL3D_27PT, 192, 192, 192, 16, 4, True, "normal", 1e-300, 200),
    Case("c3_full_parallel", DIFFUSION2D_LOGNORMAL, 1024, 1024, 1, 64, 1, False, "uniform",
         coeff_seed=COEFF_SEED),
    Case("c3_full_global4", DIFFUSION2D_LOGNORMAL, 1024, 1024, 1, 64, 4, True, "uniform",
         coeff_seed=COEFF_SEED),
    # C5 at 128^3 (n = 2,097,152): k=64, hybrid p=16, 100 iterations -- large
    # enough that the solver auto-selects k1_line, the kernel of the C5 headline
    Case("c5_full_128", LAPLACE3D_7PT, 128, 128, 128, 64, 16, False, "normal", 1e-8, 100),
]

BY_NAME = {c.name: c for c in CASES + FULL_CASES}
FULL_NAMES = {c.name for c in FULL_CASES}


def build_inputs(case: Case, gen):
    """Matrix (rowptr, cols, vals as uint64/uint64/float64) and B, X0 from a
    generator object exposing stencil / normal_block_rhs / random_block_rhs
    (the oracle or the product's host generators)."""
    import numpy as np

    csr = gen.stencil(case.kind, case.nx, case.ny, case.nz, seed=case.coeff_seed,
                      contrast=case.contrast)
    n = len(csr[0]) - 1
    if case.rhs == "normal":
        b = gen.normal_block_rhs(n, case.k, RHS_SEED)
    else:
        b = gen.random_block_rhs(n, case.k, RHS_SEED)
    if case.zero_rhs:
        b = np.zeros_like(b)
    if case.dup_col is not None:
        b[:, case.dup_col] = b[:, 0]
    x0 = None
    if case.x0_seed is not None:
        x0 = gen.random_block_rhs(n, case.k, case.x0_seed)
    return csr, b, x0
