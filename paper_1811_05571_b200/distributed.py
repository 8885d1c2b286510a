"""Multi-GPU consensus / sectioning / grid ADMM.

The M x N block grid is dealt to a Pr x Pc process grid (rank = pr*Pc + pc owns row blocks
[pr*M/Pr, ..) x column blocks [pc*N/Pc, ..)).  The plan of every rank owns its NCCL
communicators (world, and the row / column communicators split from it) and issues the
exchanges of the reference's simulated message layer itself, between its shard's phases,
on its own stream, inside its CUDA graph (libadmm_b200.so, admm_dist.inc):

  ghat   (solvers.hpp:218-225, 361-372)  row communicator    — every rank gets the
         peers' ghat_iq and subtracts them in ascending q, exactly as the reference;
  outbox (solvers.hpp:120-136, 389-415)  column communicator — every rank gets all
         replicas' u+s and forms the mean in ascending i;
  scal   (residuals and objective, solvers.hpp:141-146)  all ranks, summed in rank order.

All-gathers instead of all-reduces keep the reference's reduction order, so a solve is
bit-identical for any GPU count.  torch.distributed is only the plumbing that carries the
NCCL unique id from rank 0 to the other ranks (any backend).

ShardPlan is the lower-level "bring your own transport" surface of the same shard plans
(admm_plan_create_sharded + admm_plan_run_phase + attached exchange buffers): a caller
with its own collective layer drives the phase / exchange sequence of admm_b200.h.
"""
from __future__ import annotations

import ctypes
from typing import Sequence

import numpy as np

X_GHAT, X_OUTBOX, X_SCAL = 0, 1, 2
SCAL_DOUBLES = 8  # kScalDoubles: rp2, rd2, |v|_1, non-finite flag, objective rows, spare


def choose_grid(world: int, method: str, M: int, N: int) -> tuple:
    """Process grid Pr x Pc for `world` GPUs (admm_choose_grid).  Column sharding (Pr = 1)
    is preferred: then every replica of a segment is local and the single-HBM-pass sweep
    applies."""
    from . import _lib
    from .solvers import _METHOD
    pr, pc = ctypes.c_uint64(), ctypes.c_uint64()
    st = _lib.lib.admm_choose_grid(int(world), _METHOD[method], int(M), int(N), ctypes.byref(pr), ctypes.byref(pc))
    if st != 0:
        raise ValueError(_lib.lib.admm_last_error().decode())
    return int(pr.value), int(pc.value)


def nccl_unique_id() -> bytes:
    from . import _lib
    from .errors import check
    buf = ctypes.create_string_buffer(128)
    check(_lib.lib.admm_nccl_unique_id(buf))
    return buf.raw


def dist_plan(problem, cfg, method: str, M: int, N: int, opts=None, group=None):
    """This process's rank of a multi-process plan (call on every rank after
    torch.distributed.init_process_group; one process per GPU, opts.device = its GPU)."""
    from .solvers import AdmmPlan
    try:
        import torch.distributed as dist
        up = dist.is_available() and dist.is_initialized()
    except ImportError:  # pragma: no cover
        up = False
    if not up:  # a one-rank job (the NCCL path with a world of one)
        return AdmmPlan(problem, cfg, method, M, N, opts, dist=(nccl_unique_id(), 1, 0))
    world, rank = dist.get_world_size(group), dist.get_rank(group)
    box = [nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(box, src=0, group=group)
    return AdmmPlan(problem, cfg, method, M, N, opts, dist=(box[0], world, rank))


def distributed_solve(problem, cfg, method: str, M: int, N: int, opts=None):
    """consensus / sectioning / hybrid solve over the job's GPUs (one process per GPU).
    Same SolveReport on every rank; early stopping (stop_now), the observer and
    NumericalError(last_good_iteration) behave exactly as on one GPU."""
    from .solvers import SolveOptions, _as_c128, recovery_metrics
    opts = opts or SolveOptions()
    with dist_plan(problem, cfg, method, M, N, opts) as plan:
        rep = plan.solve(opts.observer)
    if problem.truth is not None:
        rep.metrics = recovery_metrics(rep.solution, _as_c128(problem.truth))
    return rep


class ShardPlan:
    """One rank's shard plan over its blocks plus its three exchange buffers (torch tensors
    on the plan's device; the plan computes straight into them).  The caller drives
    phase(1), exchange(ghat), [phase(2), exchange(outbox)], phase(3), [exchange(scal)],
    phase(4) per iteration (admm_b200.h)."""

    def __init__(self, problem, cfg, method: str, M: int, N: int, grid: tuple, coords: tuple,
                 opts=None):
        import torch

        from . import _lib
        from .errors import check
        from .solvers import _DTYPE, _METHOD, SolveOptions, _as_c128, _ptr, make_partition
        opts = opts or SolveOptions()
        cfg.validate()
        problem.validate()
        self.method, self.M, self.N = method, M, N
        self.Pr, self.Pc = grid
        self.pr, self.pc = coords
        self.rank = self.pr * self.Pc + self.pc
        self.device = opts.device
        h = problem.h
        h_dtype = 1 if h.dtype == np.complex64 else 0
        h = np.ascontiguousarray(h) if h_dtype else _as_c128(h)
        g = _as_c128(problem.g)
        o = _lib.PlanOptionsC(_METHOD[method], M, N, int(opts.ragged), _DTYPE[opts.dtype], int(opts.device),
                              int(opts.trace_objective), {"auto": 0, "twopass": 1, "sweep": 2, "support": 5}[opts.schedule], 1,
                              float(problem.noise_sigma))
        c = cfg._c()
        sh = _lib.ShardC(self.Pr, self.Pc, self.pr, self.pc)
        handle = ctypes.c_void_p()
        check(_lib.lib.admm_plan_create_sharded(ctypes.byref(o), ctypes.byref(c), h.shape[0], h.shape[1], _ptr(h),
                                                h_dtype, _ptr(g), ctypes.byref(sh), ctypes.byref(handle)))
        self._h = handle
        self._lib, self._check = _lib, check
        sched = ctypes.c_int()
        check(_lib.lib.admm_plan_schedule(handle, ctypes.byref(sched)))
        self.schedule = "sweep" if sched.value == 1 else "twopass"
        self.buffers, self.slots = {}, {}
        self.fused_scal = False
        dev = torch.device("cuda", self.device)
        for which in (X_GHAT, X_OUTBOX, X_SCAL):
            tot, off, nb = ctypes.c_uint64(), ctypes.c_uint64(), ctypes.c_uint64()
            check(_lib.lib.admm_plan_exchange_info(handle, which, ctypes.byref(tot), ctypes.byref(off),
                                                   ctypes.byref(nb)))
            if tot.value == 0:  # scalars fused into the ghat exchange (Pr == 1, Pc > 1)
                self.fused_scal = True
                continue
            buf = torch.zeros(tot.value // 8, dtype=torch.float64, device=dev)
            check(_lib.lib.admm_plan_attach(handle, which, ctypes.c_void_p(buf.data_ptr())))
            self.buffers[which] = buf
            self.slots[which] = (off.value // 8, nb.value // 8)
        self.n_meas, self.n_pix = problem.h.shape
        # the plan's own partition (ragged bounds honoured on a 1 x 1 grid; sharded plans
        # with more ranks require uniform blocks and say so at creation)
        self.col_bounds = make_partition(self.n_meas, self.n_pix, M if method in ("consensus", "hybrid") else 1,
                                         N if method in ("sectioning", "hybrid") else 1, opts.ragged).col_bounds
        self.cfg = cfg
        self.reset()

    def stream(self):
        import torch
        return torch.cuda.ExternalStream(self._lib.lib.admm_plan_stream(self._h), device=self.device)

    def reset(self) -> None:
        self._check(self._lib.lib.admm_plan_reset(self._h))

    def info(self) -> dict:
        i = self._lib.PlanInfoC()
        self._check(self._lib.lib.admm_plan_get_info(self._h, ctypes.byref(i)))
        return {f: getattr(i, f) for f, _ in self._lib.PlanInfoC._fields_ if f != "setup_phase_s"}

    def set_stream(self, stream) -> None:
        """Launch on `stream` (a torch.cuda.Stream; None: the plan's own stream)."""
        ptr = ctypes.c_void_p(stream.cuda_stream) if stream is not None else None
        self._check(self._lib.lib.admm_plan_set_stream(self._h, ptr))

    def phase(self, k: int) -> None:
        self._check(self._lib.lib.admm_plan_run_phase(self._h, k))

    def sync(self) -> None:
        self._check(self._lib.lib.admm_plan_sync(self._h))

    def buffer(self, which: int):
        full = self.buffers[which]
        off, n = self.slots[which]
        return full, full[off:off + n]

    def segment_v(self) -> dict:
        """{column block j: v_j} for this shard's column blocks (host copies)."""
        from .solvers import _ptr
        out = np.zeros(self.n_pix, np.complex128)
        self._check(self._lib.lib.admm_plan_read(self._h, 0, _ptr(out), self.n_pix))
        nc = self.N // self.Pc if self.method in ("sectioning", "hybrid") else 1
        return {j: out[self.col_bounds[j]:self.col_bounds[j + 1]].copy()
                for j in range(self.pc * nc, (self.pc + 1) * nc)}

    def state(self) -> tuple:
        """(iterations completed, first non-finite iteration or -1)."""
        from .solvers import _ptr
        out = np.zeros(2)
        self._check(self._lib.lib.admm_plan_read(self._h, 4, _ptr(out), 2))
        return int(out[0]), int(out[1])

    def trace(self) -> np.ndarray:
        """(iterations, 3): primal, dual, objective (two-pass: iteration k's objective is
        closed in iteration k + 1; NaN until then)."""
        from .solvers import _ptr
        n = self.state()[0]
        tr = np.zeros(3 * max(n, 1))
        self._check(self._lib.lib.admm_plan_read(self._h, 3, _ptr(tr), tr.size))
        return tr[:3 * n].reshape(n, 3)

    def close(self) -> None:
        if getattr(self, "_h", None):
            self._lib.lib.admm_plan_destroy(self._h)
            self._h = None

    def __del__(self):
        self.close()


def gather_solution(segments: Sequence[dict], n_pix: int, col_bounds: list) -> np.ndarray:
    v = np.zeros(n_pix, np.complex128)
    for seg in segments:
        for j, vj in seg.items():
            v[col_bounds[j]:col_bounds[j + 1]] = vj
    return v


def phase_program(schedule: str, fused_scal: bool) -> list:
    """The per-iteration sequence a transport must drive (admm_b200.h): ints are phases,
    strings exchanges."""
    prog = [1, "ghat"]
    if schedule == "twopass":
        prog += [2, "outbox"]
    prog.append(3)
    if not fused_scal:
        prog.append("scal")
    prog.append(4)
    return prog


def iterate(shards: Sequence, comm, iters: int, in_graph: bool = False) -> None:
    """Drive `iters` iterations of caller-transported shards (the ShardPlan surface)."""
    prog = phase_program(shards[0].schedule, getattr(shards[0], "fused_scal", False))
    names = {"ghat": X_GHAT, "outbox": X_OUTBOX, "scal": X_SCAL}
    for _ in range(iters):
        for step in prog:
            if isinstance(step, int):
                for sh in shards:
                    sh.phase(step)
            else:
                comm.exchange(names[step], shards, in_graph)


def run_iterations(shards: Sequence, comm, iters: int) -> None:
    """After reset the ghat slots hold ghat^0 (sweep prologue) or 0: exchange first."""
    comm.exchange(X_GHAT, shards)
    iterate(shards, comm, iters)


def prime(shards: Sequence, comm) -> None:
    comm.exchange(X_GHAT, shards)
