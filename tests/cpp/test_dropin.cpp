// tests/cpp/test_dropin.cpp — the drop-in header admmgpu/admmsplit_dropin.hpp against the
// UNMODIFIED reference in the same process: admmsplit:: types in, admmsplit:: types out, the
// reference's own CPU solvers (compiled from /root/reference/proj/include) as the checker.
// Built in the build container (the reference headers exist only there) by
// tests/test_cpp_shim.py; the binary travels to the GPU box.
#include <cmath>
#include <cstdio>
#include <memory>
#include <stdexcept>
#include <string>

#include "admmgpu/admmsplit_dropin.hpp"

static int g_fail = 0, g_checks = 0;
#define CHECK(cond)                                                   \
  do {                                                                \
    ++g_checks;                                                       \
    if (!(cond)) {                                                    \
      ++g_fail;                                                       \
      std::printf("  FAILED %s:%d: %s\n", __FILE__, __LINE__, #cond); \
    }                                                                 \
  } while (0)
#define CHECK_THROWS_AS(expr, Exc)                                          \
  do {                                                                      \
    bool ok_ = false;                                                       \
    try { (void)(expr); } catch (const Exc&) { ok_ = true; } catch (...) {} \
    CHECK(ok_ && #Exc);                                                     \
  } while (0)

using admmsplit::CMatrix;
using admmsplit::Complex;
using admmsplit::CVector;

static double rel(const CVector& a, const CVector& b) {
  double num = 0, den = 0, mx = 0;
  for (const auto& z : b) mx = std::max(mx, std::abs(z));
  for (std::size_t i = 0; i < a.size(); ++i) {
    num += std::norm((a[i] - b[i]) / mx);
    den += std::norm(b[i] / mx);
  }
  return std::sqrt(num / den);
}

static CMatrix random_matrix(std::size_t r, std::size_t c, std::uint64_t seed) {
  admmsplit::Xoshiro256pp rng(seed);
  CMatrix a(r, c);
  for (std::size_t i = 0; i < a.size(); ++i) a.data()[i] = rng.next_complex_gauss();
  return a;
}
static CVector random_vector(std::size_t n, std::uint64_t seed) {
  admmsplit::Xoshiro256pp rng(seed);
  CVector v(n);
  for (auto& z : v) z = rng.next_complex_gauss();
  return v;
}

// tests/test_linalg.cpp:123-134, verbatim in substance, against the device GramSolver
static void woodbury_and_direct_strategies_agree() {
  using admmgpu::ref::GramSolver;
  for (std::uint64_t seed = 1; seed <= 10; ++seed) {
    const CMatrix h = random_matrix(3 + seed % 4, 12, seed);
    const double rho = 0.25 * static_cast<double>(1 + seed % 3);
    const CVector rhs = random_vector(12, 50 + seed);
    const GramSolver woodbury(h, rho, GramSolver::Strategy::Woodbury);
    const GramSolver direct(h, rho, GramSolver::Strategy::Direct);
    const CVector xw = woodbury.solve(rhs);
    const CVector xd = direct.solve(rhs);
    CHECK(rel(xw, xd) <= 1e-8);
    // and against the reference's own GramSolver (gram.hpp, CPU)
    CHECK(rel(xw, admmsplit::GramSolver(h, rho).solve(rhs)) <= 1e-12);
  }
  CHECK_THROWS_AS(GramSolver(random_matrix(2, 3, 5), 0.0), admmsplit::ParameterError);
  CMatrix bad(2, 2);
  bad(0, 0) = Complex(std::nan(""), 0.0);
  CHECK_THROWS_AS(GramSolver(bad, 1.0), admmsplit::NumericalError);
  auto shared = std::make_shared<const CMatrix>(random_matrix(4, 9, 77));
  const GramSolver g(shared, 0.5);
  CHECK(&g.block() == shared.get() && g.inner_dim() == 4 && g.strategy() == GramSolver::Strategy::Woodbury);
}

// every solver entry point: reference types in/out, the reference's own solver as checker
static void solvers_match_the_reference_in_process() {
  const admmsplit::SensingProblem p =
      admmsplit::gen_problem(48, 192, 6, 30.0, 4242, admmsplit::ProblemKind::ComplexGaussian);
  admmsplit::SolverConfig cfg;
  cfg.lambda = 0.05 * admmsplit::norm_inf(admmsplit::adjoint_matvec(p.h, p.g));
  cfg.max_iters = 40;
  struct Case { const char* name; std::size_t m, n; };
  for (const Case c : {Case{"reference", 1, 1}, Case{"consensus", 4, 1}, Case{"sectioning", 1, 4},
                       Case{"hybrid", 2, 4}}) {
    admmsplit::SolveReport want, got;
    const std::string name = c.name;
    std::size_t calls = 0;
    admmsplit::SolveOptions opts;
    opts.observer = [&](const admmsplit::IterateSnapshot& s) { calls += s.iteration > 0; };
    if (name == "reference") {
      want = admmsplit::lasso_admm_reference(p, cfg);
      got = admmgpu::ref::lasso_admm_reference(p, cfg, opts);
    } else if (name == "consensus") {
      want = admmsplit::consensus_solve(p, cfg, c.m);
      got = admmgpu::ref::consensus_solve(p, cfg, c.m, opts);
    } else if (name == "sectioning") {
      want = admmsplit::sectioning_solve(p, cfg, c.n);
      got = admmgpu::ref::sectioning_solve(p, cfg, c.n, opts);
    } else {
      want = admmsplit::hybrid_solve(p, cfg, c.m, c.n);
      got = admmgpu::ref::hybrid_solve(p, cfg, c.m, c.n, opts);
    }
    const double e = rel(got.solution, want.solution);
    std::printf("  %s: rel err vs admmsplit %.2e\n", c.name, e);
    CHECK(e <= 1e-9);
    CHECK(got.iterations_run == want.iterations_run && calls == want.iterations_run);
    CHECK(std::abs(got.objective - want.objective) <= 1e-9 * std::abs(want.objective));
    CHECK(got.metrics && want.metrics && got.metrics->support_recall == want.metrics->support_recall);
    CHECK(got.ledger.node_count() == want.ledger.node_count() &&
          got.ledger.iteration_count() == want.ledger.iteration_count());
    for (std::size_t nd = 0; nd < want.ledger.node_count(); ++nd)
      for (std::size_t k = 0; k < want.ledger.iteration_count(); ++k)
        CHECK(got.ledger.counts(nd, k).total() == want.ledger.counts(nd, k).total());
    for (std::size_t k = 0; k < want.trace.size(); ++k)
      CHECK(std::abs(got.trace.dual[k] - want.trace.dual[k]) <= 1e-8 * std::abs(want.trace.dual[k]));
  }
  // the reference's exception classes, in its validation order
  CHECK_THROWS_AS(admmgpu::ref::consensus_solve(p, cfg, 5), admmsplit::PartitionError);
  admmsplit::SolverConfig bad = cfg;
  bad.rho = 0.0;
  CHECK_THROWS_AS(admmgpu::ref::consensus_solve(p, bad, 4), admmsplit::ParameterError);
  admmsplit::SolveOptions boom;
  boom.observer = [](const admmsplit::IterateSnapshot& s) {
    if (s.iteration == 2) throw std::runtime_error("observer");
  };
  CHECK_THROWS_AS(admmgpu::ref::consensus_solve(p, cfg, 4, boom), std::runtime_error);
}

int main() {
  struct { const char* name; void (*fn)(); } cases[] = {
      {"woodbury_and_direct_strategies_agree", woodbury_and_direct_strategies_agree},
      {"solvers_match_the_reference_in_process", solvers_match_the_reference_in_process}};
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
