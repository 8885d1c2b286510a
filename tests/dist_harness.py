"""TEST-ONLY transports for the ShardPlan surface (paper_1811_05571_b200.distributed).

  TorchComm    — torch.distributed all-gathers (gloo in the CPU tests: one numpy shard per
                 process; NCCL for tools/dist_check.py), one shard per process;
  LoopbackComm — several CUDA shard plans in ONE process (the single-GPU test box): the
                 exchanges are device copies between phases, after a host sync, so no
                 kernel ever waits for another.
The product's multi-GPU path is the plan-owned NCCL driver (admm_dist.inc); these let the
tests drive the same phases and buffer layouts without it.
"""
from __future__ import annotations

import contextlib
from typing import Sequence

from paper_1811_05571_b200.distributed import X_GHAT, X_OUTBOX, X_SCAL, iterate


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
        ctx = contextlib.nullcontext() if in_graph or not full.is_cuda else _stream_ctx(sh)
        with ctx:
            if full.is_cuda:  # in place: `mine` is this rank's slot of `full` (rank order = group order)
                self.dist.all_gather_into_tensor(full, mine, group=group)
            else:  # gloo: list form over views of the slots
                n = mine.numel()
                views = list(full.split(n))
                self.dist.all_gather(views, mine.clone(), group=group)


def _stream_ctx(sh):
    s = sh.stream() if hasattr(sh, "stream") else None
    if s is None:
        return contextlib.nullcontext()
    import torch
    return torch.cuda.stream(s)


class LoopbackComm:
    """All-gathers among several shards living in one process.  Each group's slots are
    copied into every member's buffer, after synchronising the members' streams."""

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


class GraphedIterations:
    """`iters_per_graph` iterations of one shard (phases + NCCL all-gathers through
    TorchComm) captured in a torch CUDA graph and replayed (tools/dist_check.py)."""

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
                iterate([shard], comm, iters_per_graph, in_graph=True)
        finally:
            shard.set_stream(None)

    def run(self, iters: int) -> None:
        assert iters % self.n == 0, "whole graphs only"
        import torch
        with torch.cuda.stream(self.shard.stream()):
            for _ in range(iters // self.n):
                self.graph.replay()
