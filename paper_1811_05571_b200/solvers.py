"""Reference-shaped host API over the B200 engine (the drop-in for admmsplit's hot path).

Mirrors, name for name, the reference entry points and types:
  lasso_admm_reference  reference.hpp:27        consensus_solve   solvers.hpp:74
  sectioning_solve      solvers.hpp:179         hybrid_solve      solvers.hpp:306
  SolverConfig admm_core.hpp:17, SensingProblem problem.hpp:25, SolveOptions report.hpp:42,
  SolveReport report.hpp:16, IterateSnapshot report.hpp:28, ResidualTrace admm_core.hpp:38,
  RecoveryMetrics metrics.hpp:10, GramSolver gram.hpp:26, matvec/adjoint_matvec linalg.hpp:97/114,
  soft_threshold_vec prox.hpp:21, make_partition partition.hpp:56.
Validation order and exception classes follow the reference.  All
arithmetic runs in libadmm_b200.so on the GPU; this module only marshals arrays.
"""
from __future__ import annotations

import ctypes
import dataclasses
import enum
from typing import Callable, Optional

import numpy as np

from . import _lib
from .comm import CommLedger
from .errors import (DimensionError, IndexError, MetricsError, NumericalError, ParameterError,
                     PartitionError, check)

_METHOD = {"reference": 0, "consensus": 1, "sectioning": 2, "hybrid": 3}
_DTYPE = {"c128": 0, "complex128": 0, "c64": 1, "complex64": 1}


class ProblemKind(enum.Enum):
    ComplexGaussian = "complex-gaussian"
    RandomPhase = "random-phase"
    FromFile = "from-file"


@dataclasses.dataclass
class SolverConfig:
    """admm_core.hpp:17-35 (lambda is spelled lambda_)."""
    rho: float = 1.0
    lambda_: float = 1.0
    scl: float = 1.0
    max_iters: int = 50
    eps_pri: float = 0.0
    eps_dual: float = 0.0
    seed: int = 0

    def validate(self) -> None:
        if not self.rho > 0.0:
            raise ParameterError("SolverConfig: rho must be positive")
        if not self.lambda_ > 0.0:
            raise ParameterError("SolverConfig: lambda must be positive")
        if not self.scl > 0.0:
            raise ParameterError("SolverConfig: scl must be positive")
        if self.max_iters < 1:
            raise ParameterError("SolverConfig: max_iters must be >= 1")
        if self.eps_pri < 0.0 or self.eps_dual < 0.0:
            raise ParameterError("SolverConfig: residual thresholds must be non-negative")

    def _c(self) -> _lib.SolverConfigC:
        return _lib.SolverConfigC(float(self.rho), float(self.lambda_), float(self.scl),
                                  int(self.max_iters), float(self.eps_pri), float(self.eps_dual),
                                  int(self.seed))


@dataclasses.dataclass
class SensingProblem:
    """problem.hpp:25-49.  h may be complex128 or complex64 (the latter is kept as-is)."""
    h: np.ndarray
    g: np.ndarray
    truth: Optional[np.ndarray] = None
    noise_sigma: float = 0.0
    kind: ProblemKind = ProblemKind.FromFile

    def n_meas(self) -> int:
        return int(self.h.shape[0])

    def n_pix(self) -> int:
        return int(self.h.shape[1])

    def validate(self) -> None:
        """problem.hpp:35-49, host part: shapes, then the truth's finiteness.  H and g are
        scanned for non-finite entries by the C side (multithreaded), which then checks
        noise_sigma -- the reference's order (NumericalError before ParameterError)."""
        if self.h.ndim != 2 or self.h.size == 0:
            raise DimensionError("SensingProblem: empty sensing matrix")
        if self.g.shape[0] != self.h.shape[0] or self.g.ndim not in (1, 2):
            raise DimensionError(f"SensingProblem: g length {self.g.shape[0]} != H rows {self.h.shape[0]}")
        if self.truth is not None and self.truth.shape != (self.h.shape[1],):
            raise DimensionError(f"SensingProblem: truth length {self.truth.size} != H cols "
                                 f"{self.h.shape[1]}")
        if self.truth is not None and not np.all(np.isfinite(np.asarray(self.truth).view(np.float64))):
            raise NumericalError("SensingProblem: non-finite entries")


@dataclasses.dataclass
class IterateSnapshot:
    """report.hpp:28-35."""
    iteration: int
    v: np.ndarray
    v_prev: np.ndarray
    replica_u: list
    segment_v: list
    segment_v_prev: list


IterateObserver = Callable[[IterateSnapshot], None]


@dataclasses.dataclass
class SolveOptions:
    """report.hpp:42-46 plus the device knobs (dtype of the streamed matrices, CUDA
    device, per-iteration objective)."""
    threads: int = 1
    ragged: bool = False
    observer: Optional[IterateObserver] = None
    dtype: str = "c128"
    device: int = 0
    trace_objective: bool = True
    schedule: str = "auto"  # "auto" | "twopass" | "sweep" | "resident" | "support"
    devices: Optional[list] = None  # GPUs of this process, one shard each (plan-owned NCCL);
    #                                 None: the single-GPU plan on `device`


@dataclasses.dataclass
class ResidualTrace:
    """admm_core.hpp:38-50."""
    primal: np.ndarray
    dual: np.ndarray
    objective: np.ndarray

    def size(self) -> int:
        return int(self.primal.size)


@dataclasses.dataclass
class RecoveryMetrics:
    nmse: float = 0.0
    support_precision: float = 0.0
    support_recall: float = 0.0


@dataclasses.dataclass
class SolveReport:
    """report.hpp:16-23."""
    solution: np.ndarray
    trace: ResidualTrace
    ledger: CommLedger
    iterations_run: int = 0
    objective: float = 0.0
    metrics: Optional[RecoveryMetrics] = None


@dataclasses.dataclass
class PartitionSpec:
    M: int
    N: int
    row_bounds: list
    col_bounds: list
    ragged: bool = False

    def n_meas(self) -> int:
        return self.row_bounds[-1]

    def n_pix(self) -> int:
        return self.col_bounds[-1]

    def row_size(self, i: int) -> int:
        return self.row_bounds[i + 1] - self.row_bounds[i]

    def col_size(self, j: int) -> int:
        return self.col_bounds[j + 1] - self.col_bounds[j]


def _split_bounds(total: int, parts: int, ragged: bool, axis: str) -> list:
    """partition.hpp:34-52."""
    if parts < 1 or parts > total:
        raise PartitionError(f"make_partition: {axis} division count {parts} not in [1, {total}]")
    if not ragged and total % parts != 0:
        raise PartitionError(f"make_partition: {parts} does not divide {total} {axis}s "
                             "(pass ragged=true to allow uneven blocks)")
    base, rem = divmod(total, parts)
    b = [0]
    for k in range(parts):
        b.append(b[-1] + base + (1 if k < rem else 0))
    return b


def make_partition(n_meas: int, n_pix: int, m: int, n: int, ragged: bool = False) -> PartitionSpec:
    """partition.hpp:56-65."""
    return PartitionSpec(m, n, _split_bounds(n_meas, m, ragged, "row"),
                         _split_bounds(n_pix, n, ragged, "column"), ragged)


def recovery_metrics(estimate: np.ndarray, truth: np.ndarray) -> RecoveryMetrics:
    """metrics.hpp:20-43 (host, once per solve)."""
    if estimate.shape != truth.shape:
        raise DimensionError("recovery_metrics: length mismatch")
    tsq = float(np.sum(truth.real ** 2 + truth.imag ** 2))
    if tsq == 0.0:
        raise MetricsError("recovery_metrics: truth is identically zero")
    d = estimate - truth
    nmse = float(np.sum(d.real ** 2 + d.imag ** 2)) / tsq
    thr = 1e-3 * float(np.max(np.abs(estimate))) if estimate.size else 0.0
    in_est = np.abs(estimate) > thr
    in_truth = truth != 0
    est_support = int(in_est.sum())
    hits = int((in_est & in_truth).sum())
    precision = 1.0 if est_support == 0 else hits / est_support
    recall = hits / int(in_truth.sum())
    return RecoveryMetrics(nmse, precision, recall)


def _as_c128(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.complex128)


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


class AdmmPlan:
    """A solve configuration resident on one GPU: the uploaded blocks, their Woodbury
    inverses and a captured CUDA graph of one iteration (admm_plan_* of the C ABI).

    The reference rebuilds its workers on every solve call; a plan lets a caller reuse
    the factorizations across measurement vectors (set_g) and lambdas (set_lambda)."""

    def __init__(self, problem: SensingProblem, cfg: SolverConfig, method: str, M: int = 1,
                 N: int = 1, opts: Optional[SolveOptions] = None, dist: Optional[tuple] = None):
        """dist = (nccl_id bytes, nranks, rank): this process's rank of a multi-process plan
        (see distributed.dist_plan); opts.devices = [d0, d1, ...]: one process driving
        several GPUs.  Either way the plan owns its NCCL communicators and is used exactly
        like a single-GPU plan."""
        opts = opts or SolveOptions()
        cfg.validate()                      # 1. SolverConfig::validate
        problem.validate()                  # 2. SensingProblem::validate (shapes; finiteness in C)
        h = problem.h
        if h.dtype == np.complex64:
            h_dtype = 1
            h = np.ascontiguousarray(h)
        else:
            h_dtype = 0
            h = _as_c128(h)
        g = _as_c128(problem.g)
        self.batch = int(g.shape[1]) if g.ndim == 2 else 1  # scenes (BASELINE config 5)
        self.method = method
        self.n_meas, self.n_pix = h.shape
        self.M = M if method in ("consensus", "hybrid") else 1
        self.N = N if method in ("sectioning", "hybrid") else 1
        self.cfg = dataclasses.replace(cfg)
        self.opts = opts
        o = _lib.PlanOptionsC(_METHOD[method], self.M, self.N, int(opts.ragged),
                              _DTYPE[opts.dtype], int(opts.device), int(opts.trace_objective),
                              {"auto": 0, "twopass": 1, "sweep": 2, "resident": 4, "support": 5}[opts.schedule], self.batch,
                              float(problem.noise_sigma))
        c = self.cfg._c()
        handle = ctypes.c_void_p()
        if dist is not None:
            nid, nranks, rank = dist
            check(_lib.lib.admm_plan_create_dist(ctypes.byref(o), ctypes.byref(c), self.n_meas, self.n_pix,
                                                 _ptr(h), h_dtype, _ptr(g), bytes(nid), int(nranks), int(rank),
                                                 ctypes.byref(handle)))
        elif opts.devices is not None:
            devs = (ctypes.c_int * len(opts.devices))(*[int(d) for d in opts.devices])
            check(_lib.lib.admm_plan_create_multi(ctypes.byref(o), ctypes.byref(c), self.n_meas, self.n_pix,
                                                  _ptr(h), h_dtype, _ptr(g), len(opts.devices), devs,
                                                  ctypes.byref(handle)))
        else:
            check(_lib.lib.admm_plan_create(ctypes.byref(o), ctypes.byref(c), self.n_meas, self.n_pix,
                                            _ptr(h), h_dtype, _ptr(g), ctypes.byref(handle)))
        # (the C side validated finiteness, then the partition, then the factors)
        self._h = handle
        self.spec = make_partition(self.n_meas, self.n_pix, self.M, self.N, opts.ragged)

    # -- lifecycle ----------------------------------------------------------------
    def close(self) -> None:
        if getattr(self, "_h", None):
            _lib.lib.admm_plan_destroy(self._h)
            self._h = None

    def __del__(self):
        self.close()

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    # -- configuration -------------------------------------------------------------
    def set_g(self, g: np.ndarray) -> None:
        g = _as_c128(g)
        if g.shape != ((self.n_meas,) if self.batch == 1 else (self.n_meas, self.batch)):
            raise DimensionError("set_g: length mismatch")
        check(_lib.lib.admm_plan_set_g(self._h, _ptr(g)))

    def set_lambda(self, lam: float) -> None:
        check(_lib.lib.admm_plan_set_lambda(self._h, float(lam)))
        self.cfg.lambda_ = float(lam)

    def set_lambdas(self, lams) -> None:
        """Per-scene lambda_b of a batched plan."""
        lams = np.ascontiguousarray(lams, dtype=np.float64)
        if lams.shape != (self.batch,):
            raise DimensionError("set_lambdas: one lambda per scene")
        check(_lib.lib.admm_plan_set_lambdas(self._h, _ptr(lams)))

    def max_abs_adjoint_batched(self) -> np.ndarray:
        out = np.zeros(self.batch)
        check(_lib.lib.admm_plan_max_abs_adjoint_batched(self._h, _ptr(out)))
        return out

    def max_abs_adjoint(self) -> float:
        out = ctypes.c_double()
        check(_lib.lib.admm_plan_max_abs_adjoint(self._h, ctypes.byref(out)))
        return out.value

    def info(self) -> dict:
        i = _lib.PlanInfoC()
        check(_lib.lib.admm_plan_get_info(self._h, ctypes.byref(i)))
        out = {f: getattr(i, f) for f, _ in _lib.PlanInfoC._fields_}
        out["setup_phase_s"] = dict(zip(("validate", "upload", "gram", "inverse"), list(i.setup_phase_s)))
        return out

    # -- running -------------------------------------------------------------------
    def solve(self, observer: Optional[IterateObserver] = None) -> SolveReport:
        iters = int(self.cfg.max_iters)
        B = self.batch
        sol = np.zeros(self.n_pix * B, np.complex128)
        trace = np.zeros((iters, 3 * B), np.float64)
        it = ctypes.c_uint64()
        obj = ctypes.c_double()
        cb = _lib.OBSERVER()
        raised = []
        if observer is not None:
            spec = self.spec

            def _cb(sp, _user):
                try:
                    _observe(sp)
                    return 0
                except BaseException as e:  # noqa: BLE001 -- re-raised after the C call returns
                    raised.append(e)
                    return 1

            def _observe(sp):
                s = sp.contents
                n = int(s.n_pix)
                v = np.ctypeslib.as_array(s.v, shape=(2 * n,)).view(np.complex128).copy()
                vp = np.ctypeslib.as_array(s.v_prev, shape=(2 * n,)).view(np.complex128).copy()
                us = []
                for w in range(int(s.n_workers)):
                    ln = int(s.replica_len[w])
                    us.append(np.ctypeslib.as_array(s.replica_u[w], shape=(2 * ln,))
                              .view(np.complex128).copy())
                segv = [v[spec.col_bounds[j]:spec.col_bounds[j + 1]] for j in range(spec.N)]
                segp = [vp[spec.col_bounds[j]:spec.col_bounds[j + 1]] for j in range(spec.N)]
                observer(IterateSnapshot(int(s.iteration), v, vp, us, segv, segp))

            cb = _lib.OBSERVER(_cb)
        st = _lib.lib.admm_plan_solve(self._h, _ptr(sol), _ptr(trace), ctypes.byref(it),
                                      ctypes.byref(obj), cb, None)
        if raised:  # the observer's exception propagates out of the solve (solvers.hpp:150-160)
            raise raised[0]
        check(st)
        k = int(it.value)
        ledger = CommLedger.for_solve(self.method, self.spec.row_bounds, self.spec.col_bounds, k)
        if B > 1:  # solution (n_pix, B), trace columns (iterations, B)
            tr = trace[:k].reshape(k, B, 3)
            return SolveReport(sol.reshape(self.n_pix, B), ResidualTrace(tr[:, :, 0].copy(), tr[:, :, 1].copy(),
                                                                         tr[:, :, 2].copy()), ledger, k,
                               float(obj.value))
        tr = trace[:k, :3]
        return SolveReport(sol, ResidualTrace(tr[:, 0].copy(), tr[:, 1].copy(), tr[:, 2].copy()),
                           ledger, k, float(obj.value))

    def reset(self) -> None:
        check(_lib.lib.admm_plan_reset(self._h))

    def enqueue(self, iters: int) -> None:
        check(_lib.lib.admm_plan_enqueue(self._h, int(iters)))

    def sync(self) -> None:
        check(_lib.lib.admm_plan_sync(self._h))

    def stream(self) -> int:
        return int(_lib.lib.admm_plan_stream(self._h) or 0)

    def profile(self, iters: int = 5) -> dict:
        n = _lib.lib.admm_plan_kernel_count(self._h)
        names = (ctypes.c_char_p * n)()
        ms = (ctypes.c_double * n)()
        check(_lib.lib.admm_plan_profile(self._h, int(iters), names, ms))
        return {names[k].decode(): ms[k] for k in range(n)}

    def support_stats(self) -> tuple:
        """Support schedule: (iterations since reset, support columns summed over them)."""
        out = np.zeros(2)
        check(_lib.lib.admm_plan_read(self._h, 5, _ptr(out), 2))
        return int(out[0]), int(out[1])

    def read(self, which: str) -> np.ndarray:
        w = {"v": 0, "v_prev": 1, "u": 2}[which]
        n = self.n_pix if w < 2 else self.n_pix * self.M  # u: every worker's, in worker order
        out = np.zeros(n, np.complex128)
        check(_lib.lib.admm_plan_read(self._h, w, _ptr(out), n))
        return out


def _solve(method: str, problem: SensingProblem, cfg: SolverConfig, M: int, N: int,
           opts: Optional[SolveOptions]) -> SolveReport:
    opts = opts or SolveOptions()
    with AdmmPlan(problem, cfg, method, M, N, opts) as plan:
        rep = plan.solve(opts.observer)
    if problem.truth is not None:  # finalize_report, solvers.hpp:58-61
        rep.metrics = recovery_metrics(rep.solution, _as_c128(problem.truth))
    return rep


def lasso_admm_reference(problem: SensingProblem, cfg: SolverConfig,
                         opts: Optional[SolveOptions] = None) -> SolveReport:
    """reference.hpp:27-90 (single node, kappa = lambda/rho, immediate dual update)."""
    return _solve("reference", problem, cfg, 1, 1, opts)


def consensus_solve(problem: SensingProblem, cfg: SolverConfig, m: int,
                    opts: Optional[SolveOptions] = None) -> SolveReport:
    """solvers.hpp:74-167 (row split, replica mean, kappa = lambda/(M rho))."""
    return _solve("consensus", problem, cfg, m, 1, opts)


def sectioning_solve(problem: SensingProblem, cfg: SolverConfig, n: int,
                     opts: Optional[SolveOptions] = None) -> SolveReport:
    """solvers.hpp:179-292 (column split, Jacobi ghat exchange, kappa = lambda/rho)."""
    return _solve("sectioning", problem, cfg, 1, n, opts)


def hybrid_solve(problem: SensingProblem, cfg: SolverConfig, m: int, n: int,
                 opts: Optional[SolveOptions] = None) -> SolveReport:
    """solvers.hpp:306-454 (M x N grid)."""
    return _solve("hybrid", problem, cfg, m, n, opts)


# ---- L0 / L1 operations on the device -------------------------------------------------

def matvec(a: np.ndarray, x: np.ndarray, device: int = 0) -> np.ndarray:
    """linalg.hpp:97-111."""
    a, x = _as_c128(a), _as_c128(x)
    if a.ndim != 2 or a.shape[1] != x.size:
        raise DimensionError(f"matvec: A is {a.shape[0]}x{a.shape[1]}, x has length {x.size}")
    y = np.zeros(a.shape[0], np.complex128)
    check(_lib.lib.admm_matvec(_ptr(a), a.shape[0], a.shape[1], _ptr(x), _ptr(y), device))
    return y


def adjoint_matvec(a: np.ndarray, x: np.ndarray, device: int = 0) -> np.ndarray:
    """linalg.hpp:114-127."""
    a, x = _as_c128(a), _as_c128(x)
    if a.ndim != 2 or a.shape[0] != x.size:
        raise DimensionError(f"adjoint_matvec: A is {a.shape[0]}x{a.shape[1]}, x has length {x.size}")
    y = np.zeros(a.shape[1], np.complex128)
    check(_lib.lib.admm_adjoint_matvec(_ptr(a), a.shape[0], a.shape[1], _ptr(x), _ptr(y), device))
    return y


def soft_threshold_vec(a: np.ndarray, kappa: float, device: int = 0) -> np.ndarray:
    """prox.hpp:21-25."""
    a = _as_c128(a)
    out = np.zeros_like(a)
    check(_lib.lib.admm_soft_threshold(_ptr(a), a.size, float(kappa), _ptr(out), device))
    return out


class GramSolver:
    """gram.hpp:26-128 on the device: validated and factored ONCE at construction
    (gram.hpp:48-53), solve() reuses the stored factor.  Woodbury (rows < cols, or on
    request): the rows x rows (rho I + H H^H)^-1 through the inversion lemma; Direct: the
    cols x cols (H^H H + rho I)^-1 applied to rhs."""

    class Strategy(enum.Enum):
        Direct = 0
        Woodbury = 1

    @staticmethod
    def strategy_for(rows: int, cols: int) -> "GramSolver.Strategy":
        """gram.hpp:32-34: Woodbury iff rows < cols."""
        return GramSolver.Strategy.Woodbury if rows < cols else GramSolver.Strategy.Direct

    def __init__(self, block: np.ndarray, rho: float, strategy: Optional["GramSolver.Strategy"] = None,
                 device: int = 0):
        block = _as_c128(block)
        self._block, self._rho = block, float(rho)
        handle = ctypes.c_void_p()
        rows, cols = (block.shape if block.ndim == 2 and block.size else (0, 0))
        s = -1 if strategy is None else strategy.value
        check(_lib.lib.admm_gram_create(_ptr(block) if block.size else None, rows, cols, float(rho), s, device,
                                        ctypes.byref(handle)))
        self._g = handle
        used, dim = ctypes.c_int(), ctypes.c_uint64()
        check(_lib.lib.admm_gram_info(handle, ctypes.byref(used), ctypes.byref(dim)))
        self._strategy = GramSolver.Strategy(used.value)
        self._inner = int(dim.value)

    def __del__(self):
        if getattr(self, "_g", None):
            _lib.lib.admm_gram_destroy(self._g)
            self._g = None

    def strategy(self) -> "GramSolver.Strategy":
        return self._strategy

    def rho(self) -> float:
        return self._rho

    def block(self) -> np.ndarray:
        return self._block

    def inner_dim(self) -> int:
        return self._inner

    def solve(self, rhs: np.ndarray) -> np.ndarray:
        rhs = _as_c128(rhs)
        if rhs.size != self._block.shape[1]:
            raise DimensionError(f"GramSolver::solve: rhs length {rhs.size} != block cols "
                                 f"{self._block.shape[1]}")
        x = np.zeros(self._block.shape[1], np.complex128)
        check(_lib.lib.admm_gram_apply(self._g, _ptr(rhs), _ptr(x)))
        return x
