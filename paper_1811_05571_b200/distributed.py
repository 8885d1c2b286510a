"""Multi-GPU consensus / sectioning / grid ADMM.

One process per GPU.  The M x N block grid is dealt to a Pr x Pc process grid
(rank = pr*Pc + pc owns row blocks [pr*M/Pr, ..) x column blocks [pc*N/Pc, ..)).
Each rank runs a *shard plan* (libadmm_b200.so) over its blocks; between its phases
the exchanges of the reference's simulated message layer become all-gathers:

  ghat   (solvers.hpp:218-225, 361-372)  row communicator    — every rank gets the
         peers' ghat_iq and subtracts them in ascending q, exactly as the reference;
  outbox (solvers.hpp:120-136, 389-415)  column communicator — every rank gets all
         replicas' u+s and forms the mean in ascending i;
  scal   (residual norms, solvers.hpp:141-145)  all ranks, summed in rank order.

All-gather instead of all-reduce keeps the reference's reduction order, so the result
is bit-identical for any GPU count.  The orchestration below is backend-agnostic: the
same `run_iterations` drives
  * TorchComm  — torch.distributed (NCCL on B200; gloo in the CPU tests), one shard
                 per process, collectives on the shard plan's stream;
  * LoopbackComm — several shards in ONE process (tests: the real CUDA shard plans on a
                 single GPU, exchanges as device copies; no kernel waits on another).
"""
from __future__ import annotations

import ctypes
import math
from typing import List, Optional, Sequence

import numpy as np

X_GHAT, X_OUTBOX, X_SCAL = 0, 1, 2


def choose_grid(world: int, method: str, M: int, N: int) -> tuple:
    """Process grid Pr x Pc for `world` GPUs.  Column sharding (Pr = 1) is preferred:
    then every replica of a segment is local and the single-HBM-pass sweep applies."""
    if method == "consensus":
        if M % world:
            raise ValueError(f"consensus: {world} GPUs must divide M={M}")
        return world, 1
    if method in ("sectioning", "reference"):
        if N % world:
            raise ValueError(f"sectioning: {world} GPUs must divide N={N}")
        return 1, world
    for pc in sorted({d for d in range(1, world + 1) if world % d == 0}, reverse=True):
        pr = world // pc
        if N % pc == 0 and M % pr == 0:
            return pr, pc
    raise ValueError(f"no {world}-GPU grid divides the {M}x{N} block grid")


class ShardPlan:
    """One rank's B200 plan over its blocks plus its three exchange buffers (torch
    tensors on the plan's device; the plan computes straight into them)."""

    def __init__(self, problem, cfg, method: str, M: int, N: int, grid: tuple, coords: tuple,
                 opts=None):
        import torch

        from . import _lib
        from .errors import check
        from .solvers import _DTYPE, _METHOD, SolveOptions, _as_c128, _ptr
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
                              0, {"auto": 0, "twopass": 1, "sweep": 2}[opts.schedule])
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
            if tot.value == 0:  # scalars fused into the ghat exchange (Pr == 1)
                self.fused_scal = True
                continue
            buf = torch.zeros(tot.value // 8, dtype=torch.float64, device=dev)
            check(_lib.lib.admm_plan_attach(handle, which, ctypes.c_void_p(buf.data_ptr())))
            self.buffers[which] = buf
            self.slots[which] = (off.value // 8, nb.value // 8)
        self.n_meas, self.n_pix = problem.h.shape
        self.col_bounds = _bounds(self.n_pix, N)
        self.cfg = cfg
        self.reset()

    # engine interface used by run_iterations
    def stream(self):
        import torch
        return torch.cuda.ExternalStream(self._lib.lib.admm_plan_stream(self._h), device=self.device)

    def reset(self) -> None:
        self._check(self._lib.lib.admm_plan_reset(self._h))

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
        nc = self.N // self.Pc
        return {j: out[self.col_bounds[j]:self.col_bounds[j + 1]].copy()
                for j in range(self.pc * nc, (self.pc + 1) * nc)}

    def state(self) -> tuple:
        """(iterations completed, first non-finite iteration or -1)."""
        from .solvers import _ptr
        out = np.zeros(2)
        self._check(self._lib.lib.admm_plan_read(self._h, 4, _ptr(out), 2))
        return int(out[0]), int(out[1])

    def trace(self) -> np.ndarray:
        """(iterations, 3): primal, dual, objective (NaN: not computed when sharded)."""
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


def _bounds(total: int, parts: int) -> list:
    base = total // parts
    return [k * base for k in range(parts + 1)]


class TorchComm:
    """torch.distributed all-gathers (one shard per process).  Row/column
    sub-communicators are created collectively by every rank in the same order."""

    def __init__(self, Pr: int, Pc: int):
        import torch.distributed as dist
        self.dist = dist
        self.Pr, self.Pc = Pr, Pc
        self.rank = dist.get_rank()
        pr, pc = divmod(self.rank, Pc)
        self.row = self.col = None
        for r in range(Pr):  # row communicators: same pr, ordered by pc
            g = dist.new_group([r * Pc + c for c in range(Pc)])
            if r == pr:
                self.row = g
        for c in range(Pc):  # column communicators: same pc, ordered by pr
            g = dist.new_group([r * Pc + c for r in range(Pr)])
            if c == pc:
                self.col = g

    def exchange(self, which: int, shards: Sequence, in_graph: bool = False) -> None:
        (sh,) = shards
        full, mine = sh.buffer(which)
        group = {X_GHAT: self.row, X_OUTBOX: self.col, X_SCAL: None}[which]
        import contextlib
        ctx = contextlib.nullcontext() if in_graph else _stream_ctx(sh)  # capture: current stream
        with ctx:
            if full.is_cuda:  # in place: `mine` is this rank's slot of `full` (rank order = group order)
                self.dist.all_gather_into_tensor(full, mine, group=group)
            else:  # gloo: list form over views of the slots
                n = mine.numel()
                views = list(full.split(n))
                self.dist.all_gather(views, mine.clone(), group=group)


def _stream_ctx(sh):
    import contextlib
    s = sh.stream() if hasattr(sh, "stream") else None
    if s is None:
        return contextlib.nullcontext()
    import torch
    return torch.cuda.stream(s)


class LoopbackComm:
    """All-gathers among several shards living in one process (test harness).  Each
    group's slots are copied into every member's buffer, after synchronising the
    members' streams — no kernel ever waits for another."""

    def __init__(self, Pr: int, Pc: int):
        self.Pr, self.Pc = Pr, Pc

    def exchange(self, which: int, shards: Sequence, in_graph: bool = False) -> None:
        assert not in_graph, "LoopbackComm synchronises on the host: not capturable"
        for sh in shards:
            if hasattr(sh, "sync"):
                sh.sync()
        by_rank = {sh.rank: sh for sh in shards}
        for sh in shards:
            if which == X_GHAT:
                members = [by_rank[sh.pr * self.Pc + c] for c in range(self.Pc)]
            elif which == X_OUTBOX:
                members = [by_rank[r * self.Pc + sh.pc] for r in range(self.Pr)]
            else:
                members = [by_rank[k] for k in range(self.Pr * self.Pc)]
            full, _ = sh.buffer(which)
            for m in members:
                if m is sh:
                    continue
                _, slot = m.buffer(which)
                off = m.slots[which][0]
                full[off:off + slot.numel()].copy_(slot)
        for sh in shards:
            if hasattr(sh, "buffers") and sh.buffers[which].is_cuda:
                import torch
                torch.cuda.synchronize(sh.buffers[which].device)


def run_iterations(shards: List, comm, iters: int) -> None:
    """Drive `iters` ADMM iterations of every local shard (phase order in admm_b200.h).
    After reset the ghat slots hold ghat^0 (sweep prologue) or 0: exchange first."""
    comm.exchange(X_GHAT, shards)
    _iterate(shards, comm, iters)


def prime(shards, comm) -> None:
    """After reset: the ghat of iteration 0 (sweep prologue) must reach the peers."""
    comm.exchange(X_GHAT, shards)


class GraphedIterations:
    """`iters_per_graph` distributed iterations (shard phases + NCCL all-gathers) captured
    once in a CUDA graph on a side stream and replayed: no Python or launch overhead per
    iteration.  Requires TorchComm over NCCL (collectives are capturable once the
    communicators are initialised — run one eager iteration first)."""

    def __init__(self, shard, comm, iters_per_graph: int = 8):
        import torch
        self.shard, self.n = shard, iters_per_graph
        self.stream = torch.cuda.Stream(device=shard.device)
        self.graph = torch.cuda.CUDAGraph()
        shard.sync()
        torch.cuda.synchronize(shard.device)
        shard.set_stream(self.stream)
        try:
            with torch.cuda.graph(self.graph, stream=self.stream):
                _iterate([shard], comm, iters_per_graph, in_graph=True)
        finally:
            shard.set_stream(None)

    def run(self, iters: int) -> None:
        """Replay ceil(iters / iters_per_graph) graphs (whole graphs only) on the shard
        plan's own stream, ordered after its reset/prime and covered by its sync()."""
        import torch
        with torch.cuda.stream(self.shard.stream()):
            for _ in range(-(-iters // self.n)):
                self.graph.replay()


def _iterate(shards, comm, iters, in_graph=False):
    sched = shards[0].schedule
    for _ in range(iters):
        for sh in shards:
            sh.phase(1)
        comm.exchange(X_GHAT, shards, in_graph)
        if sched == "twopass":
            for sh in shards:
                sh.phase(2)
            comm.exchange(X_OUTBOX, shards, in_graph)
            for sh in shards:
                sh.phase(3)
        if not getattr(shards[0], "fused_scal", False):  # else the scalars rode with ghat
            comm.exchange(X_SCAL, shards, in_graph)
        for sh in shards:
            sh.phase(4)


def gather_solution(segments: Sequence[dict], n_pix: int, col_bounds: list) -> np.ndarray:
    v = np.zeros(n_pix, np.complex128)
    for seg in segments:
        for j, vj in seg.items():
            v[col_bounds[j]:col_bounds[j + 1]] = vj
    return v


def distributed_solve(problem, cfg, method: str, M: int, N: int, opts=None, iters: Optional[int] = None):
    """Run a sharded solve on this process's GPU (call on every rank; torch.distributed
    already initialised).  Returns the full solution v on every rank."""
    import torch.distributed as dist
    world = dist.get_world_size()
    Pr, Pc = choose_grid(world, method, M, N)
    rank = dist.get_rank()
    pr, pc = divmod(rank, Pc)
    sh = ShardPlan(problem, cfg, method, M, N, (Pr, Pc), (pr, pc), opts)
    comm = TorchComm(Pr, Pc)
    run_iterations([sh], comm, iters or cfg.max_iters)
    sh.sync()
    segs = [None] * world
    dist.all_gather_object(segs, sh.segment_v())
    return gather_solution(segs, problem.h.shape[1], sh.col_bounds)
