// include/admmgpu/admmgpu.hpp — C++ drop-in for the reference solver API on the B200.
//
// Same type names, member names, signatures and exception classes as the reference
// headers (/root/reference/proj/include/admmsplit/*.hpp), in namespace admmgpu, over
// the C ABI of include/admm_b200.h (libadmm_b200.so).  A reference caller switches by
// replacing `#include "admmsplit/admmsplit.hpp"` / `admmsplit::` with this header /
// `admmgpu::`.  Header-only; link with -ladmm_b200.
//
//   consensus_solve   solvers.hpp:74      sectioning_solve   solvers.hpp:179
//   hybrid_solve      solvers.hpp:306     lasso_admm_reference reference.hpp:27
//   SolverConfig admm_core.hpp:17   SensingProblem problem.hpp:25   SolveOptions report.hpp:42
//   SolveReport report.hpp:16   IterateSnapshot report.hpp:28   CommLedger comm.hpp:45
//   errors errors.hpp:10-81   GramSolver gram.hpp:26   matvec/adjoint_matvec linalg.hpp:97/114
//   read_cmat/write_cmat/read_cvec/write_cvec cmat_io.hpp:44-125
//
// Beyond the reference: SolveOptions::devices (several GPUs, plan-owned NCCL), ProblemRef
// (a non-owning view: the reference's own SensingProblem -- same memory layout -- or a
// complex64 H, passed to the device without a host copy), and admmgpu/admmsplit_dropin.hpp,
// which takes and returns the reference's own types (namespace admmsplit).
#pragma once

#include <algorithm>
#include <cmath>
#include <complex>
#include <cstddef>
#include <cstdint>
#include <exception>
#include <functional>
#include <memory>
#include <mutex>
#include <optional>
#include <stdexcept>
#include <string>
#include <vector>

#include "admm_b200.h"

namespace admmgpu {

using Complex = std::complex<double>;
using CVector = std::vector<Complex>;

// ---- errors.hpp:10-81 --------------------------------------------------------
class Error : public std::runtime_error {
 public:
  using std::runtime_error::runtime_error;
};
class DimensionError : public Error { public: using Error::Error; };
class IndexError : public Error { public: using Error::Error; };
class NumericalError : public Error {
 public:
  explicit NumericalError(const std::string& what, std::size_t last_good_iteration = 0)
      : Error(what), last_good_(last_good_iteration) {}
  std::size_t last_good_iteration() const { return last_good_; }
 private:
  std::size_t last_good_ = 0;
};
class SingularityError : public Error { public: using Error::Error; };
class PartitionError : public Error { public: using Error::Error; };
class ParameterError : public Error { public: using Error::Error; };
class MetricsError : public Error { public: using Error::Error; };
class FormatError : public Error {
 public:
  explicit FormatError(const std::string& what, std::size_t byte_offset = 0) : Error(what), offset_(byte_offset) {}
  std::size_t byte_offset() const { return offset_; }
 private:
  std::size_t offset_ = 0;
};
class IoError : public Error { public: using Error::Error; };
class DeviceError : public Error { public: using Error::Error; };  // ADMM_E_CUDA
class NcclError : public Error { public: using Error::Error; };    // ADMM_E_NCCL

inline void check(admm_status st) {
  if (st == ADMM_OK) return;
  const std::string msg = admm_last_error();
  switch (st) {
    case ADMM_E_DIMENSION: throw DimensionError(msg);
    case ADMM_E_INDEX: throw IndexError(msg);
    case ADMM_E_NUMERICAL: throw NumericalError(msg, admm_last_good_iteration());
    case ADMM_E_SINGULARITY: throw SingularityError(msg);
    case ADMM_E_PARTITION: throw PartitionError(msg);
    case ADMM_E_PARAMETER: throw ParameterError(msg);
    case ADMM_E_CUDA: throw DeviceError(msg);
    case ADMM_E_FORMAT: throw FormatError(msg, admm_cmat_error_offset());
    case ADMM_E_IO: throw IoError(msg);
    case ADMM_E_NCCL: throw NcclError(msg);
    default: throw Error(msg);
  }
}

// ---- linalg.hpp:21-73 (row-major complex<double>) -----------------------------
class CMatrix {
 public:
  CMatrix() = default;
  CMatrix(std::size_t rows, std::size_t cols) : rows_(rows), cols_(cols), data_(rows * cols) {
    if (rows == 0 || cols == 0) throw ParameterError("CMatrix dimensions must be positive");
  }
  std::size_t rows() const { return rows_; }
  std::size_t cols() const { return cols_; }
  bool empty() const { return data_.empty(); }
  Complex& operator()(std::size_t r, std::size_t c) { return data_[r * cols_ + c]; }
  const Complex& operator()(std::size_t r, std::size_t c) const { return data_[r * cols_ + c]; }
  Complex* data() { return data_.data(); }
  const Complex* data() const { return data_.data(); }
  std::size_t size() const { return data_.size(); }
  static CMatrix identity(std::size_t n) {
    CMatrix m(n, n);
    for (std::size_t i = 0; i < n; ++i) m(i, i) = Complex(1.0, 0.0);
    return m;
  }
 private:
  std::size_t rows_ = 0, cols_ = 0;
  CVector data_;
};

inline CVector zeros(std::size_t n) { return CVector(n, Complex(0.0, 0.0)); }

// ---- admm_core.hpp:17-50 ------------------------------------------------------
struct SolverConfig {
  double rho = 1.0;
  double lambda = 1.0;
  double scl = 1.0;
  std::size_t max_iters = 50;
  double eps_pri = 0.0;
  double eps_dual = 0.0;
  std::uint64_t seed = 0;
  void validate() const {
    if (!(rho > 0.0)) throw ParameterError("SolverConfig: rho must be positive");
    if (!(lambda > 0.0)) throw ParameterError("SolverConfig: lambda must be positive");
    if (!(scl > 0.0)) throw ParameterError("SolverConfig: scl must be positive");
    if (max_iters < 1) throw ParameterError("SolverConfig: max_iters must be >= 1");
    if (eps_pri < 0.0 || eps_dual < 0.0)
      throw ParameterError("SolverConfig: residual thresholds must be non-negative");
  }
};

struct ResidualTrace {
  std::vector<double> primal, dual, objective;
  std::size_t size() const { return primal.size(); }
  void push(double rp, double rd, double obj) {
    primal.push_back(rp);
    dual.push_back(rd);
    objective.push_back(obj);
  }
};

// ---- problem.hpp:25-49 ---------------------------------------------------------
enum class ProblemKind { ComplexGaussian, RandomPhase, FromFile };
struct SensingProblem {
  CMatrix h;
  CVector g;
  std::optional<CVector> truth;
  double noise_sigma = 0.0;
  ProblemKind kind = ProblemKind::FromFile;
  std::size_t n_meas() const { return h.rows(); }
  std::size_t n_pix() const { return h.cols(); }
};

// ---- comm.hpp:25-107 -----------------------------------------------------------
enum class Convention { SenderOnceBroadcast, PerLink };
class CommLedger {
 public:
  struct Counts {
    std::uint64_t received = 0, sent = 0;
    std::uint64_t total() const { return received + sent; }
  };
  void record_recv(std::size_t n, std::size_t k, std::uint64_t e) { cell(n, k).received += e; }
  void record_send(std::size_t n, std::size_t k, std::uint64_t e) {
    cell(n, k).sent_once += e;
    cell(n, k).sent_links += e;
  }
  void record_broadcast(std::size_t n, std::size_t k, std::uint64_t e, std::uint64_t peers) {
    cell(n, k).sent_once += e;
    cell(n, k).sent_links += e * peers;
  }
  std::size_t node_count() const { return cells_.size(); }
  std::size_t iteration_count() const {
    std::size_t it = 0;
    for (const auto& c : cells_) it = std::max(it, c.size());
    return it;
  }
  Counts counts(std::size_t n, std::size_t k, Convention c = Convention::SenderOnceBroadcast) const {
    Counts out;
    if (n >= cells_.size() || k >= cells_[n].size()) return out;
    out.received = cells_[n][k].received;
    out.sent = c == Convention::SenderOnceBroadcast ? cells_[n][k].sent_once : cells_[n][k].sent_links;
    return out;
  }
  bool empty() const { return cells_.empty(); }
 private:
  struct Cell { std::uint64_t received = 0, sent_once = 0, sent_links = 0; };
  Cell& cell(std::size_t n, std::size_t k) {
    if (n >= cells_.size()) cells_.resize(n + 1);
    if (k >= cells_[n].size()) cells_[n].resize(k + 1);
    return cells_[n][k];
  }
  std::vector<std::vector<Cell>> cells_;
};

// ---- metrics.hpp / report.hpp ---------------------------------------------------
struct RecoveryMetrics {
  double nmse = 0.0, support_precision = 0.0, support_recall = 0.0;
};
inline RecoveryMetrics recovery_metrics(const CVector& est, const CVector& truth) {  // metrics.hpp:20-43
  if (est.size() != truth.size()) throw DimensionError("recovery_metrics: length mismatch");
  double tsq = 0.0, d = 0.0, mx = 0.0;
  for (const auto& z : truth) tsq += std::norm(z);
  if (tsq == 0.0) throw MetricsError("recovery_metrics: truth is identically zero");
  for (std::size_t i = 0; i < est.size(); ++i) {
    d += std::norm(est[i] - truth[i]);
    mx = std::max(mx, std::abs(est[i]));
  }
  std::size_t es = 0, ts = 0, hits = 0;
  for (std::size_t i = 0; i < est.size(); ++i) {
    const bool a = std::abs(est[i]) > 1e-3 * mx, b = truth[i] != Complex(0.0, 0.0);
    es += a;
    ts += b;
    hits += a && b;
  }
  RecoveryMetrics m;
  m.nmse = d / tsq;
  m.support_precision = es == 0 ? 1.0 : double(hits) / double(es);
  m.support_recall = double(hits) / double(ts);
  return m;
}

struct SolveReport {
  CVector solution;
  ResidualTrace trace;
  CommLedger ledger;
  std::size_t iterations_run = 0;
  double objective = 0.0;
  std::optional<RecoveryMetrics> metrics;
};

struct IterateSnapshot {
  std::size_t iteration = 0;
  CVector v, v_prev;
  std::vector<CVector> replica_u, segment_v, segment_v_prev;
};
using IterateObserver = std::function<void(const IterateSnapshot&)>;

struct SolveOptions {
  std::size_t threads = 1;  // no meaning on the device; kept for source compatibility
  bool ragged = false;
  IterateObserver observer;
  // B200 knobs
  admm_dtype dtype = ADMM_C128;  // storage of the streamed matrices (iterates stay FP64)
  int device = 0;
  bool trace_objective = true;
  std::vector<int> devices;      // non-empty: one shard per listed GPU, plan-owned NCCL
};

// Non-owning view of a sensing problem: H row-major interleaved (re, im) of h_dtype, g and
// the optional truth complex128.  Any type with the reference's members (h.data(),
// h.rows(), h.cols(), g, truth, noise_sigma) converts through view(); H is read straight
// from the caller's memory by the upload (no host copy), complex64 included.
struct ProblemRef {
  const void* h = nullptr;
  admm_dtype h_dtype = ADMM_C128;
  std::size_t rows = 0, cols = 0;
  const Complex* g = nullptr;
  std::size_t g_size = 0;
  const CVector* truth = nullptr;
  double noise_sigma = 0.0;
};
template <class Problem>
ProblemRef view(const Problem& p) {
  ProblemRef r;
  r.h = p.h.data();
  r.rows = p.h.empty() ? 0 : p.h.rows();
  r.cols = p.h.empty() ? 0 : p.h.cols();
  r.g = p.g.data();
  r.g_size = p.g.size();
  r.truth = p.truth ? &*p.truth : nullptr;
  r.noise_sigma = p.noise_sigma;
  return r;
}
// complex64 H (e.g. the c64 configs' 32 GiB operator) with a complex128 g.
inline ProblemRef view_c64(const std::complex<float>* h, std::size_t rows, std::size_t cols, const CVector& g,
                           const CVector* truth = nullptr, double noise_sigma = 0.0) {
  ProblemRef r;
  r.h = h;
  r.h_dtype = ADMM_C64;
  r.rows = rows;
  r.cols = cols;
  r.g = g.data();
  r.g_size = g.size();
  r.truth = truth;
  r.noise_sigma = noise_sigma;
  return r;
}

namespace detail {

inline std::vector<std::size_t> split_bounds(std::size_t total, std::size_t parts, bool ragged) {
  const std::size_t base = total / parts, rem = total % parts;
  std::vector<std::size_t> b(parts + 1, 0);
  for (std::size_t k = 0; k < parts; ++k) b[k + 1] = b[k] + base + (k < rem ? 1 : 0);
  (void)ragged;
  return b;
}

struct ObserverCtx {
  const IterateObserver* obs;
  std::vector<std::size_t> cb;
  std::exception_ptr raised;  // an exception of the observer, rethrown after the solve
};

inline int observer_trampoline(const admm_snapshot* s, void* user) {
  auto* ctx = static_cast<ObserverCtx*>(user);
  try {
  IterateSnapshot snap;
  snap.iteration = s->iteration;
  const auto* v = reinterpret_cast<const Complex*>(s->v);
  const auto* vp = reinterpret_cast<const Complex*>(s->v_prev);
  snap.v.assign(v, v + s->n_pix);
  snap.v_prev.assign(vp, vp + s->n_pix);
  for (std::size_t w = 0; w < s->n_workers; ++w) {
    const auto* u = reinterpret_cast<const Complex*>(s->replica_u[w]);
    snap.replica_u.emplace_back(u, u + s->replica_len[w]);
  }
  for (std::size_t j = 0; j + 1 < ctx->cb.size(); ++j) {
    snap.segment_v.emplace_back(snap.v.begin() + ctx->cb[j], snap.v.begin() + ctx->cb[j + 1]);
    snap.segment_v_prev.emplace_back(snap.v_prev.begin() + ctx->cb[j], snap.v_prev.begin() + ctx->cb[j + 1]);
  }
  (*ctx->obs)(snap);
  } catch (...) {
    ctx->raised = std::current_exception();
    return 1;  // stop the solve; solve() rethrows (solvers.hpp:150-160: the observer's exception propagates)
  }
  return 0;
}

// Fills the ledger with the reference's per-iteration records (solvers.hpp:111,128,
// 219-224, 358-369, 400).
template <class Ledger>
inline void fill_ledger(Ledger& led, admm_method m, const std::vector<std::size_t>& rb,
                        const std::vector<std::size_t>& cb, std::size_t iters) {
  const std::size_t M = rb.size() - 1, N = cb.size() - 1, nm = rb.back(), np = cb.back();
  for (std::size_t k = 0; k < iters; ++k) {
    if (m == ADMM_CONSENSUS) {
      for (std::size_t i = 0; i < M; ++i) {
        led.record_recv(i, k, np);
        led.record_send(i, k, np);
      }
    } else if (m == ADMM_SECTIONING) {
      for (std::size_t j = 0; j < N; ++j) {
        led.record_broadcast(j, k, nm, N - 1);
        for (std::size_t q = 0; q < N; ++q)
          if (q != j) led.record_recv(q, k, nm);
      }
    } else if (m == ADMM_HYBRID) {
      for (std::size_t i = 0; i < M; ++i)
        for (std::size_t j = 0; j < N; ++j) led.record_recv(i * N + j, k, cb[j + 1] - cb[j]);
      for (std::size_t i = 0; i < M; ++i)
        for (std::size_t j = 0; j < N; ++j) {
          const std::size_t rl = rb[i + 1] - rb[i];
          led.record_broadcast(i * N + j, k, rl, N - 1);
          for (std::size_t q = 0; q < N; ++q)
            if (q != j) led.record_recv(i * N + q, k, rl);
        }
      for (std::size_t i = 0; i < M; ++i)
        for (std::size_t j = 0; j < N; ++j) led.record_send(i * N + j, k, cb[j + 1] - cb[j]);
    }
  }
}

// Host validation in the reference's order (admm_core.hpp:26-34, problem.hpp:35-49; the
// device side scans H and g for non-finite entries, then checks noise_sigma, then the
// partition -- the same order), plan creation (single GPU, or one shard per device),
// solve, and the reference's report fields.
inline SolveReport solve(admm_method method, const ProblemRef& problem, const SolverConfig& cfg, std::size_t m,
                         std::size_t n, const SolveOptions& opts) {
  cfg.validate();
  if (!problem.h || problem.rows == 0 || problem.cols == 0) throw DimensionError("SensingProblem: empty sensing matrix");
  if (problem.g_size != problem.rows)
    throw DimensionError("SensingProblem: g length " + std::to_string(problem.g_size) + " != H rows " +
                         std::to_string(problem.rows));
  if (problem.truth && problem.truth->size() != problem.cols)
    throw DimensionError("SensingProblem: truth length " + std::to_string(problem.truth->size()) + " != H cols " +
                         std::to_string(problem.cols));
  if (problem.truth)
    for (const Complex& z : *problem.truth)
      if (!std::isfinite(z.real()) || !std::isfinite(z.imag())) throw NumericalError("SensingProblem: non-finite entries");
  admm_plan_options o{};
  o.method = method;
  o.M = m;
  o.N = n;
  o.ragged = opts.ragged ? 1 : 0;
  o.dtype = opts.dtype;
  o.device = opts.devices.empty() ? opts.device : opts.devices[0];
  o.trace_objective = opts.trace_objective ? 1 : 0;
  o.noise_sigma = problem.noise_sigma;
  admm_solver_config c{cfg.rho, cfg.lambda, cfg.scl, cfg.max_iters, cfg.eps_pri, cfg.eps_dual, cfg.seed};
  admm_plan* plan = nullptr;
  const double* g = reinterpret_cast<const double*>(problem.g);
  if (opts.devices.empty())
    check(admm_plan_create(&o, &c, problem.rows, problem.cols, problem.h, problem.h_dtype, g, &plan));
  else
    check(admm_plan_create_multi(&o, &c, problem.rows, problem.cols, problem.h, problem.h_dtype, g,
                                 (int)opts.devices.size(), opts.devices.data(), &plan));
  const std::size_t M = method == ADMM_CONSENSUS || method == ADMM_HYBRID ? m : 1;
  const std::size_t N = method == ADMM_SECTIONING || method == ADMM_HYBRID ? n : 1;
  const auto rb = split_bounds(problem.rows, M, opts.ragged);
  const auto cb = split_bounds(problem.cols, N, opts.ragged);
  SolveReport r;
  r.solution.assign(problem.cols, Complex());
  std::vector<double> tr(cfg.max_iters * 3, 0.0);
  std::uint64_t it = 0;
  double obj = 0.0;
  ObserverCtx ctx{&opts.observer, cb, nullptr};
  const admm_status st = admm_plan_solve(plan, reinterpret_cast<double*>(r.solution.data()), tr.data(), &it, &obj,
                                         opts.observer ? observer_trampoline : nullptr, &ctx);
  admm_plan_destroy(plan);
  if (ctx.raised) std::rethrow_exception(ctx.raised);
  check(st);
  for (std::size_t k = 0; k < it; ++k) r.trace.push(tr[3 * k], tr[3 * k + 1], tr[3 * k + 2]);
  r.iterations_run = it;
  r.objective = obj;
  fill_ledger(r.ledger, method, rb, cb, it);
  if (problem.truth) r.metrics = recovery_metrics(r.solution, *problem.truth);
  return r;
}

}  // namespace detail

// The reference's entry points (reference.hpp:27, solvers.hpp:74/179/306).  Each takes the
// shim's SensingProblem or a ProblemRef (view(reference_problem), view_c64(...)).
inline SolveReport lasso_admm_reference(const ProblemRef& p, const SolverConfig& cfg, const SolveOptions& opts = {}) {
  return detail::solve(ADMM_REFERENCE, p, cfg, 1, 1, opts);
}
inline SolveReport consensus_solve(const ProblemRef& p, const SolverConfig& cfg, std::size_t m,
                                   const SolveOptions& opts = {}) {
  return detail::solve(ADMM_CONSENSUS, p, cfg, m, 1, opts);
}
inline SolveReport sectioning_solve(const ProblemRef& p, const SolverConfig& cfg, std::size_t n,
                                    const SolveOptions& opts = {}) {
  return detail::solve(ADMM_SECTIONING, p, cfg, 1, n, opts);
}
inline SolveReport hybrid_solve(const ProblemRef& p, const SolverConfig& cfg, std::size_t m, std::size_t n,
                                const SolveOptions& opts = {}) {
  return detail::solve(ADMM_HYBRID, p, cfg, m, n, opts);
}
inline SolveReport lasso_admm_reference(const SensingProblem& p, const SolverConfig& cfg,
                                        const SolveOptions& opts = {}) {
  return lasso_admm_reference(view(p), cfg, opts);
}
inline SolveReport consensus_solve(const SensingProblem& p, const SolverConfig& cfg, std::size_t m,
                                   const SolveOptions& opts = {}) {
  return consensus_solve(view(p), cfg, m, opts);
}
inline SolveReport sectioning_solve(const SensingProblem& p, const SolverConfig& cfg, std::size_t n,
                                    const SolveOptions& opts = {}) {
  return sectioning_solve(view(p), cfg, n, opts);
}
inline SolveReport hybrid_solve(const SensingProblem& p, const SolverConfig& cfg, std::size_t m, std::size_t n,
                                const SolveOptions& opts = {}) {
  return hybrid_solve(view(p), cfg, m, n, opts);
}

// ---- linalg.hpp:97-127, prox.hpp:21-25 on the device ------------------------------
inline CVector matvec(const CMatrix& a, const CVector& x, int device = 0) {
  if (a.cols() != x.size()) throw DimensionError("matvec: dimension mismatch");
  CVector y(a.rows());
  check(admm_matvec(reinterpret_cast<const double*>(a.data()), a.rows(), a.cols(),
                    reinterpret_cast<const double*>(x.data()), reinterpret_cast<double*>(y.data()), device));
  return y;
}
inline CVector adjoint_matvec(const CMatrix& a, const CVector& x, int device = 0) {
  if (a.rows() != x.size()) throw DimensionError("adjoint_matvec: dimension mismatch");
  CVector y(a.cols());
  check(admm_adjoint_matvec(reinterpret_cast<const double*>(a.data()), a.rows(), a.cols(),
                            reinterpret_cast<const double*>(x.data()), reinterpret_cast<double*>(y.data()), device));
  return y;
}
inline CVector soft_threshold_vec(const CVector& a, double kappa, int device = 0) {
  CVector out(a.size());
  check(admm_soft_threshold(reinterpret_cast<const double*>(a.data()), a.size(), kappa,
                            reinterpret_cast<double*>(out.data()), device));
  return out;
}

// ---- gram.hpp:26-128 -------------------------------------------------------------
// Validated and factored ONCE on the device at construction (gram.hpp:48-53); solve() runs
// the stored factor (Woodbury: the rows x rows inverse through the inversion lemma; Direct:
// the cols x cols inverse).  Immutable; copies share the device factor; solve() is safe to
// call concurrently (gram.hpp:25).
class GramSolver {
 public:
  enum class Strategy { Direct, Woodbury };
  static Strategy strategy_for(std::size_t rows, std::size_t cols) {
    return rows < cols ? Strategy::Woodbury : Strategy::Direct;
  }
  GramSolver(std::shared_ptr<const CMatrix> block, double rho) : GramSolver(std::move(block), rho, std::nullopt) {}
  GramSolver(CMatrix block, double rho) : GramSolver(std::make_shared<const CMatrix>(std::move(block)), rho) {}
  GramSolver(CMatrix block, double rho, Strategy strategy)
      : GramSolver(std::make_shared<const CMatrix>(std::move(block)), rho, strategy) {}
  GramSolver(std::shared_ptr<const CMatrix> block, double rho, std::optional<Strategy> strategy, int device = 0)
      : block_(std::move(block)), rho_(rho) {
    admm_gram* g = nullptr;
    const int s = strategy ? (*strategy == Strategy::Woodbury ? 1 : 0) : -1;
    check(admm_gram_create(reinterpret_cast<const double*>(block_->empty() ? nullptr : block_->data()),
                           block_->empty() ? 0 : block_->rows(), block_->empty() ? 0 : block_->cols(), rho, s, device,
                           &g));
    factor_.reset(g, admm_gram_destroy);
    int used = 1;
    std::uint64_t dim = 0;
    check(admm_gram_info(g, &used, &dim));
    strategy_ = used ? Strategy::Woodbury : Strategy::Direct;
    inner_ = dim;
  }
  Strategy strategy() const { return strategy_; }
  double rho() const { return rho_; }
  const CMatrix& block() const { return *block_; }
  std::size_t inner_dim() const { return inner_; }
  CVector solve(const CVector& rhs) const {
    if (rhs.size() != block_->cols())
      throw DimensionError("GramSolver::solve: rhs length " + std::to_string(rhs.size()) + " != block cols " +
                           std::to_string(block_->cols()));
    CVector x(rhs.size());
    check(admm_gram_apply(factor_.get(), reinterpret_cast<const double*>(rhs.data()), reinterpret_cast<double*>(x.data())));
    return x;
  }
 private:
  std::shared_ptr<const CMatrix> block_;
  double rho_;
  Strategy strategy_ = Strategy::Woodbury;
  std::size_t inner_ = 0;
  std::shared_ptr<admm_gram> factor_;
};
inline GramSolver make_gram_solver(CMatrix block, double rho) { return GramSolver(std::move(block), rho); }

// ---- cmat_io.hpp:44-125 (host file I/O; CMX1 = the reference format) ----------------
// Same names, checks and exceptions as the reference.  write_cmat's `c64` flag writes the
// complex64 "CMF1" variant; read_cmat reads either (CMF1 widens exactly).  To feed a c64
// plan without an FP64 host copy call admm_cmat_read(path, float buffer, n, ADMM_C64).
inline void write_cmat(const std::string& path, const CMatrix& a, bool c64 = false) {
  if (a.empty()) throw ParameterError("write_cmat: empty matrix");
  check(admm_cmat_write(path.c_str(), a.data(), a.rows(), a.cols(), ADMM_C128, c64 ? ADMM_C64 : ADMM_C128));
}
inline CMatrix read_cmat(const std::string& path) {
  uint64_t rows = 0, cols = 0;
  admm_dtype t = ADMM_C128;
  check(admm_cmat_info(path.c_str(), &rows, &cols, &t));
  CMatrix a(rows, cols);
  check(admm_cmat_read(path.c_str(), a.data(), rows * cols, ADMM_C128));
  return a;
}
inline void write_cvec(const std::string& path, const CVector& v, bool c64 = false) {
  if (v.empty()) throw ParameterError("write_cvec: empty vector");
  check(admm_cmat_write(path.c_str(), v.data(), v.size(), 1, ADMM_C128, c64 ? ADMM_C64 : ADMM_C128));
}
inline CVector read_cvec(const std::string& path) {
  uint64_t rows = 0, cols = 0;
  admm_dtype t = ADMM_C128;
  check(admm_cmat_info(path.c_str(), &rows, &cols, &t));
  if (cols != 1)
    throw FormatError("read_cvec: " + path + " holds a " + std::to_string(rows) + "x" + std::to_string(cols) +
                          " matrix, expected a column vector",
                      12);
  CVector v(rows);
  check(admm_cmat_read(path.c_str(), v.data(), rows, ADMM_C128));
  return v;
}

}  // namespace admmgpu
