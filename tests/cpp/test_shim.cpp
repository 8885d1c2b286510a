// tests/cpp/test_shim.cpp — the reference's Catch2 cases (tests/test_linalg.cpp,
// test_prox.cpp, test_solvers.cpp, test_reference.cpp), restated against the C++ drop-in
// include/admmgpu/admmgpu.hpp so they "read like the reference's own tests".  Catch2 is
// not in this image, so a ten-line harness stands in for TEST_CASE / CHECK.
// Inputs come from the product generator (bit-identical to the reference's gen_problem),
// the expected values from the test-only C oracle (oracle/liboracle.so).
#include <unistd.h>

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <limits>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "admmgpu/admmgpu.hpp"
extern "C" {
#include "../../oracle/admm_oracle.h"
}

using namespace admmgpu;

static int g_fail = 0, g_checks = 0;
#define CHECK(cond)                                                          \
  do {                                                                       \
    ++g_checks;                                                              \
    if (!(cond)) {                                                           \
      ++g_fail;                                                              \
      std::printf("  FAILED %s:%d: %s\n", __FILE__, __LINE__, #cond);        \
    }                                                                        \
  } while (0)
#define CHECK_THROWS_AS(expr, Exc)                                           \
  do {                                                                       \
    bool ok_ = false;                                                        \
    try { (void)(expr); } catch (const Exc&) { ok_ = true; } catch (...) {}  \
    CHECK(ok_ && #Exc);                                                      \
  } while (0)
#define TEST_CASE(name) static void name()

static SensingProblem desk_problem(std::size_t rows, std::size_t cols, std::size_t k, std::uint64_t seed) {
  SensingProblem p;
  p.h = CMatrix(rows, cols);
  p.g.resize(rows);
  CVector truth(cols);
  double ns = 0;
  check(admm_gen_problem(rows, cols, k, std::numeric_limits<double>::infinity(), seed, 1, p.h.data(), ADMM_C128,
                         reinterpret_cast<double*>(p.g.data()), reinterpret_cast<double*>(truth.data()), &ns));
  p.truth = truth;
  return p;
}

static double lambda_rel(const SensingProblem& p, double c) {  // c * max|H^H g| (test_solvers.cpp:20-26)
  CVector hg(p.h.cols());
  orc_adjoint_matvec(reinterpret_cast<const double*>(p.h.data()), p.h.rows(), p.h.cols(),
                     reinterpret_cast<const double*>(p.g.data()), reinterpret_cast<double*>(hg.data()));
  double m = 0;
  for (auto& z : hg) m = std::max(m, std::abs(z));
  return c * m;
}

static double max_abs_diff(const CVector& a, const CVector& b) {
  double m = 0;
  for (std::size_t i = 0; i < a.size(); ++i) m = std::max(m, std::abs(a[i] - b[i]));
  return m;
}

TEST_CASE(matvec_known_answers) {  // test_linalg.cpp:21-53
  const Complex I(0, 1);
  CMatrix a(2, 2);
  a(0, 0) = 1; a(0, 1) = I; a(1, 1) = 2;
  const CVector y = matvec(a, {Complex(1, 0), Complex(1, 0)});
  CHECK(y[0] == Complex(1, 1) && y[1] == Complex(2, 0));
  CMatrix b(1, 1);
  b(0, 0) = I;
  CHECK(adjoint_matvec(b, {Complex(1, 0)})[0] == Complex(0, -1));
  CHECK_THROWS_AS(matvec(CMatrix(2, 3), CVector(2)), DimensionError);
}

TEST_CASE(prox_known_answers) {  // test_prox.cpp:8-54
  const CVector out = soft_threshold_vec({Complex(5, 0), Complex(-1, 0), Complex(3, 4)}, 2.0);
  CHECK(std::abs(out[0] - Complex(3, 0)) < 1e-15);
  CHECK(out[1] == Complex(0, 0));
  CHECK(std::abs(out[2] - Complex(1.8, 2.4)) < 1e-15);
}

TEST_CASE(gram_solver) {  // test_linalg.cpp:74-98
  CHECK(GramSolver::strategy_for(540, 22500) == GramSolver::Strategy::Woodbury);
  CHECK(GramSolver::strategy_for(5, 3) == GramSolver::Strategy::Direct);
  const CVector x = GramSolver(CMatrix(2, 2), 2.0).solve({Complex(4, 0), Complex(6, 0)});
  CHECK(std::abs(x[0] - Complex(2, 0)) < 1e-12 && std::abs(x[1] - Complex(3, 0)) < 1e-12);
  CHECK_THROWS_AS(GramSolver(CMatrix(2, 3), 0.0), ParameterError);
}

static CMatrix random_matrix(std::size_t rows, std::size_t cols, std::uint64_t seed) {
  CMatrix a(rows, cols);
  orc_random_gauss(rows * cols, seed, reinterpret_cast<double*>(a.data()));
  return a;
}
static CVector random_vector(std::size_t n, std::uint64_t seed) {
  CVector v(n);
  orc_random_gauss(n, seed, reinterpret_cast<double*>(v.data()));
  return v;
}
static double rel_error(const CVector& a, const CVector& b) {
  double num = 0, den = 0;
  for (std::size_t i = 0; i < a.size(); ++i) {
    num += std::norm(a[i] - b[i]);
    den += std::norm(b[i]);
  }
  return std::sqrt(num / den);
}

TEST_CASE(gram_solver_strategies) {  // test_linalg.cpp:100-161, gram.hpp:36-53
  CHECK_THROWS_AS(GramSolver(random_matrix(2, 3, 5), -1.0), ParameterError);
  CMatrix bad(2, 2);
  bad(0, 0) = Complex(std::numeric_limits<double>::quiet_NaN(), 0.0);
  CHECK_THROWS_AS(GramSolver(bad, 1.0), NumericalError);
  const GramSolver ok(random_matrix(2, 3, 6), 1.0);
  CHECK_THROWS_AS(ok.solve(CVector(2)), DimensionError);
  for (std::uint64_t seed = 1; seed <= 10; ++seed) {  // "woodbury and direct strategies agree"
    const CMatrix h = random_matrix(3 + seed % 4, 12, seed);
    const double rho = 0.25 * static_cast<double>(1 + seed % 3);
    const CVector rhs = random_vector(12, 50 + seed);
    const GramSolver woodbury(h, rho, GramSolver::Strategy::Woodbury);
    const GramSolver direct(h, rho, GramSolver::Strategy::Direct);
    CHECK(woodbury.strategy() == GramSolver::Strategy::Woodbury && woodbury.inner_dim() == h.rows());
    CHECK(direct.strategy() == GramSolver::Strategy::Direct && direct.inner_dim() == 12);
    CHECK(rel_error(woodbury.solve(rhs), direct.solve(rhs)) <= 1e-8);
  }
  for (std::uint64_t seed = 1; seed <= 8; ++seed) {  // residual, both automatic strategies
    const bool wide = seed % 2 == 0;
    const CMatrix h = wide ? random_matrix(5, 14, seed) : random_matrix(14, 5, seed);
    const GramSolver gram(h, 1.5);
    CHECK(gram.strategy() == (wide ? GramSolver::Strategy::Woodbury : GramSolver::Strategy::Direct));
    const CVector rhs = random_vector(h.cols(), 300 + seed);
    const CVector x = gram.solve(rhs);
    const CVector x2 = gram.solve(rhs);  // factored once, reused: bit-identical
    CHECK(x == x2);
    CVector hx(h.rows()), hthx(h.cols());
    orc_matvec(reinterpret_cast<const double*>(h.data()), h.rows(), h.cols(), reinterpret_cast<const double*>(x.data()),
               reinterpret_cast<double*>(hx.data()));
    orc_adjoint_matvec(reinterpret_cast<const double*>(h.data()), h.rows(), h.cols(),
                       reinterpret_cast<const double*>(hx.data()), reinterpret_cast<double*>(hthx.data()));
    double num = 0, den = 0;
    for (std::size_t i = 0; i < x.size(); ++i) {
      num += std::norm(hthx[i] + 1.5 * x[i] - rhs[i]);
      den += std::norm(rhs[i]);
    }
    CHECK(std::sqrt(num / den) <= 1e-8);
  }
  auto shared = std::make_shared<const CMatrix>(random_matrix(4, 9, 77));
  const GramSolver from_shared(shared, 0.5);  // gram.hpp:36-37
  CHECK(&from_shared.block() == shared.get());
}

TEST_CASE(problem_views_devices_and_observer) {
  const SensingProblem p = desk_problem(48, 192, 4, 1011);
  SolverConfig cfg;
  cfg.lambda = lambda_rel(p, 0.05);
  cfg.max_iters = 30;
  const SolveReport base = hybrid_solve(p, cfg, 2, 4);
  // the same problem through a non-owning view, and on the plan-owned NCCL path (one device)
  CHECK(rel_error(hybrid_solve(view(p), cfg, 2, 4).solution, base.solution) == 0.0);
  SolveOptions multi;
  multi.devices = {0};
  const SolveReport m1 = hybrid_solve(p, cfg, 2, 4, multi);
  CHECK(rel_error(m1.solution, base.solution) <= 1e-12 && m1.iterations_run == base.iterations_run);
  // complex64 H straight from the caller's memory into a c64 plan
  std::vector<std::complex<float>> h64(p.h.size());
  for (std::size_t i = 0; i < h64.size(); ++i) h64[i] = std::complex<float>((float)p.h.data()[i].real(), (float)p.h.data()[i].imag());
  SolveOptions o64;
  o64.dtype = ADMM_C64;
  CHECK(rel_error(hybrid_solve(view_c64(h64.data(), 48, 192, p.g), cfg, 2, 4, o64).solution, base.solution) <= 1e-4);
  // an exception thrown by the observer propagates out of the solve (solvers.hpp:150-160)
  SolveOptions obs;
  int calls = 0;
  obs.observer = [&](const IterateSnapshot& s) {
    ++calls;
    if (s.iteration == 3) throw std::out_of_range("stop at 3");
  };
  CHECK_THROWS_AS(hybrid_solve(p, cfg, 2, 4, obs), std::out_of_range);
  CHECK(calls == 3);
  SensingProblem neg = p;  // problem.hpp:35-49 order: non-finite before negative noise_sigma
  neg.noise_sigma = -1.0;
  CHECK_THROWS_AS(hybrid_solve(neg, cfg, 2, 4), ParameterError);
  neg.g[0] = Complex(std::numeric_limits<double>::infinity(), 0.0);
  CHECK_THROWS_AS(hybrid_solve(neg, cfg, 2, 4), NumericalError);
}

TEST_CASE(degeneracy_lattice) {  // test_solvers.cpp:42-93
  const SensingProblem p = desk_problem(20, 40, 4, 1001);
  SolverConfig cfg;
  cfg.lambda = lambda_rel(p, 1e-3);
  cfg.max_iters = 10;
  auto series = [&](auto fn) {
    std::vector<CVector> out;
    SolveOptions o;
    o.observer = [&](const IterateSnapshot& s) { out.push_back(s.v); };
    fn(o);
    return out;
  };
  auto diff = [](const std::vector<CVector>& a, const std::vector<CVector>& b) {
    double w = 0;
    for (std::size_t k = 0; k < a.size(); ++k) w = std::max(w, max_abs_diff(a[k], b[k]));
    return a.size() == b.size() ? w : 1e300;
  };
  const auto ref = series([&](const SolveOptions& o) { return lasso_admm_reference(p, cfg, o); });
  CHECK(diff(series([&](const SolveOptions& o) { return consensus_solve(p, cfg, 1, o); }), ref) <= 1e-12);
  CHECK(diff(series([&](const SolveOptions& o) { return sectioning_solve(p, cfg, 1, o); }), ref) <= 1e-12);
  CHECK(diff(series([&](const SolveOptions& o) { return hybrid_solve(p, cfg, 1, 1, o); }), ref) <= 1e-12);
  CHECK(diff(series([&](const SolveOptions& o) { return consensus_solve(p, cfg, 2, o); }),
             series([&](const SolveOptions& o) { return hybrid_solve(p, cfg, 2, 1, o); })) <= 1e-12);
  CHECK(diff(series([&](const SolveOptions& o) { return sectioning_solve(p, cfg, 2, o); }),
             series([&](const SolveOptions& o) { return hybrid_solve(p, cfg, 1, 2, o); })) <= 1e-12);
}

TEST_CASE(oracle_parity_and_ledger) {  // solution vs the C oracle; ledger = closed form
  const SensingProblem p = desk_problem(12, 20, 3, 1002);
  SolverConfig cfg;
  cfg.lambda = lambda_rel(p, 1e-3);
  cfg.max_iters = 4;
  const SolveReport r = hybrid_solve(p, cfg, 3, 4);
  CVector sol(20);
  std::vector<double> tr(12);
  std::uint64_t it = 0, lg = 0;
  double obj = 0;
  CHECK(orc_solve(ORC_HYBRID, reinterpret_cast<const double*>(p.h.data()), reinterpret_cast<const double*>(p.g.data()),
                  12, 20, 3, 4, 0, cfg.rho, cfg.lambda, 1.0, 4, 0, 0, reinterpret_cast<double*>(sol.data()), tr.data(),
                  &it, &obj, &lg, nullptr) == ORC_OK);
  double num = 0, den = 0;
  for (std::size_t i = 0; i < 20; ++i) {
    num += std::norm(r.solution[i] - sol[i]);
    den += std::norm(sol[i]);
  }
  CHECK(std::sqrt(num / den) <= 1e-9);
  CHECK(r.ledger.node_count() == 12 && r.ledger.iteration_count() == 4);
  for (std::size_t n = 0; n < 12; ++n)
    for (std::size_t k = 0; k < 4; ++k) CHECK(r.ledger.counts(n, k).total() == 4 * (12 / 3) + 2 * (20 / 4));
}

TEST_CASE(errors_follow_reference) {  // test_solvers.cpp:221-243, test_reference.cpp:118-139
  const SensingProblem p = desk_problem(10, 12, 3, 1007);
  SolverConfig cfg;
  cfg.lambda = lambda_rel(p, 1e-3);
  CHECK_THROWS_AS(consensus_solve(p, cfg, 4), PartitionError);
  SolveOptions rag;
  rag.ragged = true;
  CHECK(consensus_solve(p, cfg, 4, rag).iterations_run == cfg.max_iters);
  SensingProblem huge = desk_problem(6, 9, 2, 1008);
  for (std::size_t i = 0; i < huge.h.size(); ++i) huge.h.data()[i] *= 1e300;
  for (auto& z : huge.g) z *= 1e300;
  CHECK_THROWS_AS(consensus_solve(huge, cfg, 2), NumericalError);
  SolverConfig bad;
  bad.rho = 0.0;
  CHECK_THROWS_AS(consensus_solve(p, bad, 2), ParameterError);
}

TEST_CASE(cmat_round_trip_and_malformed) {  // test_problem_gen.cpp:105-164 (host only)
  const std::string dir = "/tmp/admmgpu_shim_cmat_" + std::to_string(::getpid());
  std::system(("mkdir -p " + dir).c_str());
  const SensingProblem p = desk_problem(7, 5, 2, 33);
  write_cmat(dir + "/roundtrip.cmat", p.h);
  const CMatrix back = read_cmat(dir + "/roundtrip.cmat");
  bool same = back.rows() == 7 && back.cols() == 5;
  for (std::size_t i = 0; same && i < back.size(); ++i) same = back.data()[i] == p.h.data()[i];
  CHECK(same);
  write_cvec(dir + "/v.cmat", p.g);
  CHECK(read_cvec(dir + "/v.cmat") == p.g);
  write_cmat(dir + "/h64.cmat", p.h, /*c64=*/true);
  const CMatrix h64 = read_cmat(dir + "/h64.cmat");
  bool rounded = true;
  for (std::size_t i = 0; i < h64.size(); ++i)
    rounded = rounded && h64.data()[i] == Complex((float)p.h.data()[i].real(), (float)p.h.data()[i].imag());
  CHECK(rounded);
  std::FILE* f = std::fopen((dir + "/empty.cmat").c_str(), "wb");
  std::fclose(f);
  CHECK_THROWS_AS(read_cmat(dir + "/empty.cmat"), FormatError);
  std::system(("truncate -s 68 " + dir + "/roundtrip.cmat").c_str());
  try {
    read_cmat(dir + "/roundtrip.cmat");
    CHECK(false);
  } catch (const FormatError& e) {
    CHECK(e.byte_offset() == 20 + 3 * sizeof(Complex));
  }
  CHECK_THROWS_AS(read_cvec(dir + "/h64.cmat"), FormatError);
  CHECK_THROWS_AS(read_cmat(dir + "/does_not_exist.cmat"), IoError);
  CHECK_THROWS_AS(write_cvec(dir + "/e.cmat", CVector{}), ParameterError);
  CMatrix bad(1, 1);
  bad(0, 0) = Complex(std::numeric_limits<double>::infinity(), 0.0);
  CHECK_THROWS_AS(write_cmat(dir + "/inf.cmat", bad), NumericalError);
  std::system(("rm -rf " + dir).c_str());
}

int main(int argc, char** argv) {
  if (argc > 1 && std::string(argv[1]) == "host") {  // cases that need no device
    cmat_round_trip_and_malformed();
    std::printf("%s cmat_round_trip_and_malformed\n%d checks, %d failures\n", g_fail ? "FAIL" : "PASS", g_checks,
                g_fail);
    return g_fail ? 1 : 0;
  }
  struct { const char* name; void (*fn)(); } cases[] = {
      {"cmat_round_trip_and_malformed", cmat_round_trip_and_malformed},
      {"matvec_known_answers", matvec_known_answers}, {"prox_known_answers", prox_known_answers},
      {"gram_solver", gram_solver}, {"gram_solver_strategies", gram_solver_strategies},
      {"problem_views_devices_and_observer", problem_views_devices_and_observer},
      {"degeneracy_lattice", degeneracy_lattice},
      {"oracle_parity_and_ledger", oracle_parity_and_ledger}, {"errors_follow_reference", errors_follow_reference}};
  for (auto& c : cases) {
    const int before = g_fail;
    try {
      c.fn();
    } catch (const std::exception& e) {
      ++g_fail;
      std::printf("  EXCEPTION in %s: %s\n", c.name, e.what());
    }
    std::printf("%s %s\n", g_fail == before ? "PASS" : "FAIL", c.name);
  }
  std::printf("%d checks, %d failures\n", g_checks, g_fail);
  return g_fail ? 1 : 0;
}
