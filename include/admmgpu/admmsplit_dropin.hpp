// include/admmgpu/admmsplit_dropin.hpp — the B200 solvers behind the reference's OWN types.
//
// For a caller of the reference library (/root/reference/proj/include/admmsplit): the
// functions below have the reference's exact signatures (solvers.hpp:74/179/306,
// reference.hpp:27) and class shape (GramSolver, gram.hpp:26-128) and take and return
// admmsplit:: types -- SensingProblem, SolverConfig, SolveOptions (with its observer),
// SolveReport (solution, trace, CommLedger, metrics), admmsplit::CMatrix -- and throw the
// reference's exception classes (errors.hpp:10-81).  Switching a call site is a namespace
// change: admmsplit::hybrid_solve(...) -> admmgpu::ref::hybrid_solve(...).
//
// H is read in place from the reference's CMatrix (same row-major interleaved layout as the
// C ABI; no host copy).  Device knobs (GPU list, complex64 storage) come in an optional
// trailing DeviceOptions argument.  Requires the reference headers on the include path.
#pragma once

#include <exception>
#include <memory>
#include <optional>
#include <vector>

#include "admmgpu/admmgpu.hpp"
#include "admmsplit/admmsplit.hpp"

namespace admmgpu::ref {

struct DeviceOptions {
  admm_dtype dtype = ADMM_C128;
  int device = 0;
  std::vector<int> devices;  // non-empty: one shard per GPU (plan-owned NCCL)
  bool trace_objective = true;
};

namespace detail {

// admmgpu exceptions -> the reference's classes (same what(), same payloads).
template <class F>
auto rethrow_as_reference(F&& f) -> decltype(f()) {
  try {
    return f();
  } catch (const admmgpu::NumericalError& e) {
    throw admmsplit::NumericalError(e.what(), e.last_good_iteration());
  } catch (const admmgpu::DimensionError& e) {
    throw admmsplit::DimensionError(e.what());
  } catch (const admmgpu::IndexError& e) {
    throw admmsplit::IndexError(e.what());
  } catch (const admmgpu::SingularityError& e) {
    throw admmsplit::SingularityError(e.what());
  } catch (const admmgpu::PartitionError& e) {
    throw admmsplit::PartitionError(e.what());
  } catch (const admmgpu::ParameterError& e) {
    throw admmsplit::ParameterError(e.what());
  } catch (const admmgpu::FormatError& e) {
    throw admmsplit::FormatError(e.what(), e.byte_offset());
  } catch (const admmgpu::IoError& e) {
    throw admmsplit::IoError(e.what());
  } catch (const admmgpu::MetricsError& e) {
    throw admmsplit::MetricsError(e.what());
  } catch (const admmgpu::Error& e) {
    throw admmsplit::Error(e.what());  // device / NCCL failures: the reference's base class
  }
}

inline admmsplit::SolveReport solve(admm_method method, const admmsplit::SensingProblem& problem,
                                    const admmsplit::SolverConfig& cfg, std::size_t m, std::size_t n,
                                    const admmsplit::SolveOptions& opts, const DeviceOptions& dev) {
  cfg.validate();  // the reference's own validation first (admm_core.hpp:26-34)
  admmgpu::SolverConfig c;
  c.rho = cfg.rho;
  c.lambda = cfg.lambda;
  c.scl = cfg.scl;
  c.max_iters = cfg.max_iters;
  c.eps_pri = cfg.eps_pri;
  c.eps_dual = cfg.eps_dual;
  c.seed = cfg.seed;
  admmgpu::SolveOptions o;
  o.ragged = opts.ragged;
  o.dtype = dev.dtype;
  o.device = dev.device;
  o.devices = dev.devices;
  o.trace_objective = dev.trace_objective;
  if (opts.observer)
    o.observer = [&opts](const admmgpu::IterateSnapshot& s) {
      admmsplit::IterateSnapshot r;
      r.iteration = s.iteration;
      r.v = s.v;
      r.v_prev = s.v_prev;
      r.replica_u = s.replica_u;
      r.segment_v = s.segment_v;
      r.segment_v_prev = s.segment_v_prev;
      opts.observer(r);  // its exceptions propagate unchanged (solvers.hpp:150-160)
    };
  const admmgpu::SolveReport g = rethrow_as_reference([&] {
    return admmgpu::detail::solve(method, admmgpu::view(problem), c, m, n, o);  // H read in place
  });
  admmsplit::SolveReport r;
  r.solution = g.solution;
  for (std::size_t k = 0; k < g.trace.size(); ++k) r.trace.push(g.trace.primal[k], g.trace.dual[k], g.trace.objective[k]);
  r.iterations_run = g.iterations_run;
  r.objective = g.objective;
  const std::size_t M = method == ADMM_CONSENSUS || method == ADMM_HYBRID ? m : 1;
  const std::size_t N = method == ADMM_SECTIONING || method == ADMM_HYBRID ? n : 1;
  const auto rb = admmgpu::detail::split_bounds(problem.h.rows(), M, opts.ragged);
  const auto cb = admmgpu::detail::split_bounds(problem.h.cols(), N, opts.ragged);
  admmgpu::detail::fill_ledger(r.ledger, method, rb, cb, r.iterations_run);  // the reference's own CommLedger
  if (problem.truth) r.metrics = admmsplit::recovery_metrics(r.solution, *problem.truth);  // metrics.hpp:20-43
  return r;
}

}  // namespace detail

inline admmsplit::SolveReport lasso_admm_reference(const admmsplit::SensingProblem& p, const admmsplit::SolverConfig& cfg,
                                                   const admmsplit::SolveOptions& opts = {},
                                                   const DeviceOptions& dev = {}) {
  return detail::solve(ADMM_REFERENCE, p, cfg, 1, 1, opts, dev);
}
inline admmsplit::SolveReport consensus_solve(const admmsplit::SensingProblem& p, const admmsplit::SolverConfig& cfg,
                                              std::size_t m, const admmsplit::SolveOptions& opts = {},
                                              const DeviceOptions& dev = {}) {
  return detail::solve(ADMM_CONSENSUS, p, cfg, m, 1, opts, dev);
}
inline admmsplit::SolveReport sectioning_solve(const admmsplit::SensingProblem& p, const admmsplit::SolverConfig& cfg,
                                               std::size_t n, const admmsplit::SolveOptions& opts = {},
                                               const DeviceOptions& dev = {}) {
  return detail::solve(ADMM_SECTIONING, p, cfg, 1, n, opts, dev);
}
inline admmsplit::SolveReport hybrid_solve(const admmsplit::SensingProblem& p, const admmsplit::SolverConfig& cfg,
                                           std::size_t m, std::size_t n, const admmsplit::SolveOptions& opts = {},
                                           const DeviceOptions& dev = {}) {
  return detail::solve(ADMM_HYBRID, p, cfg, m, n, opts, dev);
}

// gram.hpp:26-128 over the reference's CMatrix (kept alive by the shared_ptr; read in place).
class GramSolver {
 public:
  using Strategy = admmsplit::GramSolver::Strategy;
  static Strategy strategy_for(std::size_t rows, std::size_t cols) {
    return admmsplit::GramSolver::strategy_for(rows, cols);
  }
  GramSolver(std::shared_ptr<const admmsplit::CMatrix> block, double rho)
      : GramSolver(std::move(block), rho, std::nullopt) {}
  GramSolver(admmsplit::CMatrix block, double rho)
      : GramSolver(std::make_shared<const admmsplit::CMatrix>(std::move(block)), rho) {}
  GramSolver(admmsplit::CMatrix block, double rho, Strategy strategy)
      : GramSolver(std::make_shared<const admmsplit::CMatrix>(std::move(block)), rho, strategy) {}
  GramSolver(std::shared_ptr<const admmsplit::CMatrix> block, double rho, std::optional<Strategy> strategy,
             int device = 0)
      : block_(std::move(block)), rho_(rho) {
    detail::rethrow_as_reference([&] {
      admm_gram* g = nullptr;
      const int s = strategy ? (*strategy == Strategy::Woodbury ? 1 : 0) : -1;
      admmgpu::check(admm_gram_create(reinterpret_cast<const double*>(block_->empty() ? nullptr : block_->data()),
                                      block_->empty() ? 0 : block_->rows(), block_->empty() ? 0 : block_->cols(), rho,
                                      s, device, &g));
      factor_.reset(g, admm_gram_destroy);
      int used = 1;
      std::uint64_t dim = 0;
      admmgpu::check(admm_gram_info(g, &used, &dim));
      strategy_ = used ? Strategy::Woodbury : Strategy::Direct;
      inner_ = dim;
      return 0;
    });
  }
  Strategy strategy() const { return strategy_; }
  double rho() const { return rho_; }
  const admmsplit::CMatrix& block() const { return *block_; }
  std::size_t inner_dim() const { return inner_; }
  admmsplit::CVector solve(const admmsplit::CVector& rhs) const {
    if (rhs.size() != block_->cols())
      throw admmsplit::DimensionError("GramSolver::solve: rhs length " + std::to_string(rhs.size()) +
                                      " != block cols " + std::to_string(block_->cols()));
    admmsplit::CVector x(rhs.size());
    detail::rethrow_as_reference([&] {
      admmgpu::check(admm_gram_apply(factor_.get(), reinterpret_cast<const double*>(rhs.data()),
                                     reinterpret_cast<double*>(x.data())));
      return 0;
    });
    return x;
  }

 private:
  std::shared_ptr<const admmsplit::CMatrix> block_;
  double rho_;
  Strategy strategy_ = Strategy::Woodbury;
  std::size_t inner_ = 0;
  std::shared_ptr<admm_gram> factor_;
};

}  // namespace admmgpu::ref
