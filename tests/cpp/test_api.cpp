// test_api.cpp — the C++ drop-in API (paper_1912_11930_b200/include/blockkrylov)
// exercised the way the reference's GoogleTest suites exercise the reference
// headers (proj/tests/test_kernels.cpp, test_solver.cpp): same calls, same
// expectations, restated here with a tiny self-contained harness (GoogleTest
// is not installed).  Runs every check under both numerics modes.
//   usage: test_api [exact|fast|both]
#include <blockkrylov/blockkrylov.hpp>

#include <cmath>
#include <cstdio>
#include <cstring>
#include <functional>
#include <string>
#include <tuple>
#include <vector>

using namespace blockkrylov;

namespace {

int g_fail = 0, g_checks = 0;
std::string g_test;

#define CHECK(cond)                                                                  \
  do {                                                                               \
    ++g_checks;                                                                      \
    if (!(cond)) {                                                                   \
      ++g_fail;                                                                      \
      std::printf("  FAIL %s:%d [%s] %s\n", __FILE__, __LINE__, g_test.c_str(), #cond); \
    }                                                                                \
  } while (0)
#define CHECK_NEAR(a, b, tol) CHECK(std::abs((a) - (b)) <= (tol))
#define CHECK_THROWS(expr, type)   \
  do {                             \
    bool caught = false;           \
    try {                          \
      (void)(expr);                \
    } catch (const type&) {        \
      caught = true;               \
    }                              \
    CHECK(caught);                 \
  } while (0)

struct Dense {
  std::size_t r, c;
  std::vector<double> a;
  Dense(std::size_t rr, std::size_t cc) : r(rr), c(cc), a(rr * cc, 0.0) {}
  double& operator()(std::size_t i, std::size_t j) { return a[i * c + j]; }
  double operator()(std::size_t i, std::size_t j) const { return a[i * c + j]; }
};

Dense dense(const SparseMatrix& m) {
  Dense d(m.n(), m.n());
  for (std::size_t r = 0; r < m.n(); ++r)
    for (std::size_t i = m.row_offsets()[r]; i < m.row_offsets()[r + 1]; ++i)
      d(r, m.col_indices()[i]) = m.values()[i];
  return d;
}

SparseMatrix identity_matrix(std::size_t n, double v = 1.0) {
  std::vector<std::tuple<std::size_t, std::size_t, double>> t;
  for (std::size_t i = 0; i < n; ++i) t.emplace_back(i, i, v);
  return SparseMatrix::from_triplets(n, t);
}

void kernels_tests() {
  g_test = "bdot orthonormal";
  {
    BlockVector x(6, 4);
    for (std::size_t c = 0; c < 4; ++c) x(c, c) = 1.0;
    for (std::size_t p : {1u, 2u, 4u}) {
      const auto g = bdot(x, x, SubalgebraConfig(4, p, SubalgebraMode::hybrid));
      for (std::size_t b = 0; b < g.block_count(); ++b)
        for (std::size_t i = 0; i < p; ++i)
          for (std::size_t j = 0; j < p; ++j) CHECK(g.entry(b, i, j) == (i == j ? 1.0 : 0.0));
    }
  }
  g_test = "bdot hybrid/global vs dense";
  {
    const BlockVector x = random_block_rhs(4, 4, 11);
    double xtx[4][4] = {};
    for (std::size_t i = 0; i < 4; ++i)
      for (std::size_t j = 0; j < 4; ++j)
        for (std::size_t r = 0; r < 4; ++r) xtx[i][j] += x(r, i) * x(r, j);
    const auto h = bdot(x, x, SubalgebraConfig(4, 2, SubalgebraMode::hybrid));
    const auto g = bdot(x, x, SubalgebraConfig(4, 2, SubalgebraMode::global));
    for (std::size_t b = 0; b < 2; ++b)
      for (std::size_t i = 0; i < 2; ++i)
        for (std::size_t j = 0; j < 2; ++j) {
          CHECK_NEAR(h.entry(b, i, j), xtx[2 * b + i][2 * b + j], 1e-14);
          if (b == 0) CHECK_NEAR(g.entry(0, i, j), xtx[i][j] + xtx[2 + i][2 + j], 1e-13);
        }
    CHECK_THROWS(bdot(BlockVector(5, 4), BlockVector(6, 4), SubalgebraConfig(4, 2, SubalgebraMode::hybrid)),
                 DimensionError);
  }
  g_test = "bdot transpose symmetry";
  {
    const BlockVector x = random_block_rhs(7, 8, 3), y = random_block_rhs(7, 8, 4);
    for (auto mode : {SubalgebraMode::hybrid, SubalgebraMode::global})
      for (std::size_t p : {1u, 2u, 4u, 8u}) {
        const SubalgebraConfig cfg(8, p, mode);
        const auto xy = bdot(x, y, cfg), yx = bdot(y, x, cfg);
        for (std::size_t b = 0; b < cfg.block_count(); ++b)
          for (std::size_t i = 0; i < p; ++i)
            for (std::size_t j = 0; j < p; ++j) CHECK_NEAR(xy.entry(b, i, j), yx.entry(b, j, i), 1e-14);
      }
  }
  g_test = "baxpy zero / identity / negate";
  {
    const SubalgebraConfig cfg(4, 2, SubalgebraMode::hybrid);
    BlockVector x = random_block_rhs(5, 4, 1);
    const BlockVector y = random_block_rhs(5, 4, 2), before = x;
    baxpy(x, y, BlockCoefficient(cfg));
    CHECK(x == before);
    baxpy(x, y, BlockCoefficient::identity(cfg));
    for (std::size_t i = 0; i < x.size(); ++i) CHECK(x.data()[i] == before.data()[i] + y.data()[i]);
    BlockVector z = random_block_rhs(16, 8, 41);
    const BlockVector z0 = z, w = random_block_rhs(16, 8, 42);
    BlockCoefficient gam(SubalgebraConfig(8, 4, SubalgebraMode::hybrid));
    Xorshift64Star rng(43);
    for (std::size_t i = 0; i < 32; ++i) gam.data()[i] = rng.next_symmetric();
    baxpy(z, w, gam);
    baxpy(z, w, gam.negated());
    for (std::size_t i = 0; i < z.size(); ++i) CHECK_NEAR(z.data()[i], z0.data()[i], 1e-13);
    CHECK_THROWS(baxpy(x, x, BlockCoefficient(cfg)), DimensionError);
  }
  g_test = "bop identity / poisson";
  {
    const BlockVector x = random_block_rhs(6, 3, 51);
    CHECK(bop(identity_matrix(6), x) == x);
    const BlockVector y2 = bop(identity_matrix(6, 2.0), x);
    for (std::size_t i = 0; i < x.size(); ++i) CHECK(y2.data()[i] == 2.0 * x.data()[i]);
    const SparseMatrix a = poisson2d(PoissonSpec::constant(4, 4));
    const BlockVector v = random_block_rhs(16, 4, 52);
    const BlockVector av = bop(a, v);
    const Dense d = dense(a);
    for (std::size_t r = 0; r < 16; ++r)
      for (std::size_t c = 0; c < 4; ++c) {
        double s = 0.0;
        for (std::size_t l = 0; l < 16; ++l) s += d(r, l) * v(l, c);
        CHECK_NEAR(av(r, c), s, 1e-13);
      }
    FlopCounter f;
    const SparseMatrix a5 = poisson2d(PoissonSpec::constant(5, 5));
    bop(a5, random_block_rhs(25, 4, 83), &f);
    CHECK(f.multiply_adds_bop == 2ull * 4 * a5.nnz());
  }
  g_test = "bsolve";
  {
    const SubalgebraConfig cfg(4, 2, SubalgebraMode::hybrid);
    BlockCoefficient g = BlockCoefficient::identity(cfg), d(cfg);
    Xorshift64Star rng(61);
    for (std::size_t i = 0; i < 8; ++i) d.data()[i] = rng.next_symmetric();
    const auto out = bsolve(g, d);
    for (std::size_t i = 0; i < 8; ++i) CHECK(out.data()[i] == d.data()[i]);
    g.entry(1, 0, 0) = 1.0;
    g.entry(1, 0, 1) = 2.0;
    g.entry(1, 1, 0) = 1.0;
    g.entry(1, 1, 1) = 2.0;
    std::size_t idx = 99;
    try {
      bsolve(g, d);
    } catch (const BreakdownError& e) {
      idx = e.block_index();
    }
    CHECK(idx == 1);
    CHECK_THROWS(bsolve(BlockCoefficient::identity(cfg),
                        BlockCoefficient::identity(SubalgebraConfig(4, 2, SubalgebraMode::global))),
                 DimensionError);
  }
  g_test = "column norms / flops";
  {
    const auto z = column_norms(BlockVector(5, 3));
    CHECK(z == std::vector<double>(3, 0.0));
    const BlockVector x = random_block_rhs(17, 5, 71);
    const auto nrm = column_norms(x);
    for (std::size_t c = 0; c < 5; ++c) {
      double s = 0.0;
      for (std::size_t r = 0; r < 17; ++r) s += x(r, c) * x(r, c);
      CHECK_NEAR(nrm[c], std::sqrt(s), 1e-14 * std::sqrt(s));
    }
    for (std::size_t n : {16u, 25u})
      for (std::size_t k : {4u, 8u})
        for (std::size_t p : {1u, 2u, 4u, 8u}) {
          if (k % p) continue;
          for (auto mode : {SubalgebraMode::hybrid, SubalgebraMode::global}) {
            const SubalgebraConfig cfg(k, p, mode);
            FlopCounter f;
            BlockVector y = random_block_rhs(n, k, 82);
            bdot(random_block_rhs(n, k, 81), y, cfg, &f);
            CHECK(f.multiply_adds_bdot == 2ull * n * p * p * (k / p));
            baxpy(y, random_block_rhs(n, k, 81), BlockCoefficient::identity(cfg), &f);
            CHECK(f.multiply_adds_baxpy == 2ull * n * p * p * (k / p));
          }
        }
  }
}

void solver_tests() {
  g_test = "identity operator";
  {
    const BlockVector b = random_block_rhs(12, 4, 1);
    const auto res = bcg_solve(identity_matrix(12), b, Preconditioner::identity(12),
                               SubalgebraConfig::classical(4));
    CHECK(res.report.converged && res.report.iterations == 1);
    for (std::size_t i = 0; i < b.size(); ++i) CHECK_NEAR(res.x.data()[i], b.data()[i], 1e-13);
  }
  g_test = "zero rhs";
  {
    const auto res = bcg_solve(identity_matrix(8), BlockVector(8, 2), Preconditioner::identity(8),
                               SubalgebraConfig::classical(2));
    CHECK(res.report.converged && res.report.iterations == 0);
  }
  g_test = "nonzero x0 / final residual";
  {
    const SparseMatrix a = poisson2d(PoissonSpec::heterogeneous(8, 8, 3));
    SolveOptions o;
    o.tol = 1e-10;
    const auto res = bcg_solve(a, random_block_rhs(64, 4, 4), random_block_rhs(64, 4, 99),
                               Preconditioner::identity(64), SubalgebraConfig::classical(4), o);
    CHECK(res.report.converged);
    for (double d : res.report.final_defect_norms) CHECK(d < 1e-7);
  }
  g_test = "rank deficient breakdown";
  {
    const SparseMatrix a = poisson2d(PoissonSpec::heterogeneous(8, 8, 3));
    BlockVector b = random_block_rhs(64, 4, 4);
    for (std::size_t r = 0; r < 64; ++r) b(r, 3) = b(r, 0);
    const auto res = bcg_solve(a, b, Preconditioner::identity(64), SubalgebraConfig::classical(4));
    CHECK(!res.report.converged && res.report.breakdown.has_value());
    CHECK(res.report.breakdown && res.report.breakdown->iteration == 1 &&
          res.report.breakdown->block_index == 0 && res.report.iterations == 0);
  }
  g_test = "max_iter / history / flops / observer";
  {
    const SparseMatrix a = poisson2d(PoissonSpec::heterogeneous(8, 8, 41));
    SolveOptions o;
    o.tol = 1e-30;
    o.max_iter = 3;
    auto res = bcg_solve(a, random_block_rhs(64, 2, 42), Preconditioner::identity(64),
                         SubalgebraConfig::classical(2), o);
    CHECK(!res.report.converged && res.report.iterations == 3 && !res.report.breakdown);
    SolveOptions h;
    h.record_history = true;
    std::vector<std::size_t> seen;
    h.on_iterate = [&](std::size_t i, const BlockVector&, const BlockVector&) { seen.push_back(i); };
    const BlockVector b = random_block_rhs(64, 4, 52);
    res = bcg_solve(a, b, Preconditioner::identity(64), SubalgebraConfig(4, 2, SubalgebraMode::hybrid), h);
    CHECK(res.report.converged);
    CHECK(res.report.defect_history.size() == res.report.iterations + 1);
    CHECK(seen.size() == res.report.iterations + 1);
    const auto bn = column_norms(b);
    for (std::size_t c = 0; c < 4; ++c) CHECK_NEAR(res.report.defect_history.front()[c], bn[c], 1e-13 * bn[c]);
    const std::uint64_t i = res.report.iterations, n = 64, z = a.nnz();
    CHECK(res.report.flops.multiply_adds_bdot == 3 * i * 2 * n * 4 * 2);
    CHECK(res.report.flops.multiply_adds_baxpy == 3 * i * 2 * n * 4 * 2);
    CHECK(res.report.flops.multiply_adds_bop == i * 2 * 4 * z);
  }
  g_test = "argument validation";
  {
    const SparseMatrix a = identity_matrix(4);
    const Preconditioner m = Preconditioner::identity(4);
    const auto cfg = SubalgebraConfig::classical(2);
    CHECK_THROWS(bcg_solve(a, BlockVector(5, 2), m, cfg), DimensionError);
    CHECK_THROWS(bcg_solve(a, BlockVector(4, 3), m, cfg), DimensionError);
    CHECK_THROWS(bcg_solve(a, BlockVector(4, 2), BlockVector(4, 3), m, cfg), DimensionError);
    CHECK_THROWS(bcg_solve(a, BlockVector(4, 2), Preconditioner::identity(5), cfg), DimensionError);
    SolveOptions bad;
    bad.tol = 0.0;
    CHECK_THROWS(bcg_solve(a, BlockVector(4, 2), m, cfg, bad), ConfigError);
    CHECK_THROWS(SubalgebraConfig(8, 3, SubalgebraMode::hybrid), ConfigError);
  }
}

}  // namespace

int main(int argc, char** argv) {
  const std::string which = argc > 1 ? argv[1] : "both";
  for (const char* mode : {"exact", "fast"}) {
    if (which != "both" && which != mode) continue;
    gpu::set_numerics(std::strcmp(mode, "exact") == 0 ? gpu::Numerics::exact : gpu::Numerics::fast);
    const int before = g_fail;
    kernels_tests();
    solver_tests();
    std::printf("[%s] %s numerics: %d failures\n", g_fail == before ? "PASS" : "FAIL", mode,
                g_fail - before);
  }
  std::printf("%d checks, %d failures\n", g_checks, g_fail);
  return g_fail == 0 ? 0 : 1;
}
