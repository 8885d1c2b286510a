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
#pragma once

#include <algorithm>
#include <cmath>
#include <complex>
#include <cstddef>
#include <cstdint>
#include <functional>
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
  admm_dtype dtype = ADMM_C128;
  int device = 0;
  bool trace_objective = true;
};

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
};

inline void observer_trampoline(const admm_snapshot* s, void* user) {
  auto* ctx = static_cast<ObserverCtx*>(user);
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
}

// Fills the ledger with the reference's per-iteration records (solvers.hpp:111,128,
// 219-224, 358-369, 400).
inline void fill_ledger(CommLedger& led, admm_method m, const std::vector<std::size_t>& rb,
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

inline SolveReport solve(admm_method method, const SensingProblem& problem, const SolverConfig& cfg,
                         std::size_t m, std::size_t n, const SolveOptions& opts) {
  cfg.validate();
  if (problem.h.empty()) throw DimensionError("SensingProblem: empty sensing matrix");
  if (problem.g.size() != problem.h.rows())
    throw DimensionError("SensingProblem: g length " + std::to_string(problem.g.size()) + " != H rows " +
                         std::to_string(problem.h.rows()));
  admm_plan_options o{};
  o.method = method;
  o.M = m;
  o.N = n;
  o.ragged = opts.ragged ? 1 : 0;
  o.dtype = opts.dtype;
  o.device = opts.device;
  o.trace_objective = opts.trace_objective ? 1 : 0;
  admm_solver_config c{cfg.rho, cfg.lambda, cfg.scl, cfg.max_iters, cfg.eps_pri, cfg.eps_dual, cfg.seed};
  admm_plan* plan = nullptr;
  check(admm_plan_create(&o, &c, problem.h.rows(), problem.h.cols(), problem.h.data(), ADMM_C128,
                         reinterpret_cast<const double*>(problem.g.data()), &plan));
  const std::size_t M = method == ADMM_CONSENSUS || method == ADMM_HYBRID ? m : 1;
  const std::size_t N = method == ADMM_SECTIONING || method == ADMM_HYBRID ? n : 1;
  const auto rb = split_bounds(problem.h.rows(), M, opts.ragged);
  const auto cb = split_bounds(problem.h.cols(), N, opts.ragged);
  SolveReport r;
  r.solution.assign(problem.h.cols(), Complex());
  std::vector<double> tr(cfg.max_iters * 3, 0.0);
  std::uint64_t it = 0;
  double obj = 0.0;
  ObserverCtx ctx{&opts.observer, cb};
  const admm_status st = admm_plan_solve(plan, reinterpret_cast<double*>(r.solution.data()), tr.data(), &it, &obj,
                                         opts.observer ? observer_trampoline : nullptr, &ctx);
  admm_plan_destroy(plan);
  check(st);
  for (std::size_t k = 0; k < it; ++k) r.trace.push(tr[3 * k], tr[3 * k + 1], tr[3 * k + 2]);
  r.iterations_run = it;
  r.objective = obj;
  fill_ledger(r.ledger, method, rb, cb, it);
  if (problem.truth) r.metrics = recovery_metrics(r.solution, *problem.truth);
  return r;
}

}  // namespace detail

inline SolveReport lasso_admm_reference(const SensingProblem& p, const SolverConfig& cfg,
                                        const SolveOptions& opts = {}) {
  return detail::solve(ADMM_REFERENCE, p, cfg, 1, 1, opts);
}
inline SolveReport consensus_solve(const SensingProblem& p, const SolverConfig& cfg, std::size_t m,
                                   const SolveOptions& opts = {}) {
  return detail::solve(ADMM_CONSENSUS, p, cfg, m, 1, opts);
}
inline SolveReport sectioning_solve(const SensingProblem& p, const SolverConfig& cfg, std::size_t n,
                                    const SolveOptions& opts = {}) {
  return detail::solve(ADMM_SECTIONING, p, cfg, 1, n, opts);
}
inline SolveReport hybrid_solve(const SensingProblem& p, const SolverConfig& cfg, std::size_t m, std::size_t n,
                                const SolveOptions& opts = {}) {
  return detail::solve(ADMM_HYBRID, p, cfg, m, n, opts);
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
class GramSolver {
 public:
  enum class Strategy { Direct, Woodbury };
  static Strategy strategy_for(std::size_t rows, std::size_t cols) {
    return rows < cols ? Strategy::Woodbury : Strategy::Direct;
  }
  GramSolver(CMatrix block, double rho, int device = 0) : h_(std::move(block)), rho_(rho), device_(device) {
    if (h_.empty()) throw ParameterError("GramSolver: empty block");
    if (!(rho > 0.0)) throw ParameterError("GramSolver: rho must be positive");
    for (std::size_t i = 0; i < h_.size(); ++i)
      if (!std::isfinite(h_.data()[i].real()) || !std::isfinite(h_.data()[i].imag()))
        throw NumericalError("GramSolver: non-finite entries in block");
    strategy_ = strategy_for(h_.rows(), h_.cols());
  }
  Strategy strategy() const { return strategy_; }
  double rho() const { return rho_; }
  std::size_t inner_dim() const { return strategy_ == Strategy::Woodbury ? h_.rows() : h_.cols(); }
  CVector solve(const CVector& rhs) const {
    if (rhs.size() != h_.cols()) throw DimensionError("GramSolver::solve: rhs length mismatch");
    CVector x(rhs.size());
    check(admm_gram_solve(reinterpret_cast<const double*>(h_.data()), h_.rows(), h_.cols(), rho_,
                          reinterpret_cast<const double*>(rhs.data()), reinterpret_cast<double*>(x.data()), device_));
    return x;
  }
 private:
  CMatrix h_;
  double rho_;
  int device_;
  Strategy strategy_;
};

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
