"""CPU, world size 2 (gloo): the production multi-GPU orchestration — process grid,
sub-communicators, exchange order and buffer layouts (paper_1811_05571_b200.distributed)
— drives numpy stand-ins of the shard plans; the gathered solution must equal the
bit-pinned oracle's single-process solve."""
import os
import socket
import sys

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
sys.path.insert(0, HERE)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, case, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import dist_harness as DH
        import oracle_lib as orc
        import shard_engine_np as se
        from paper_1811_05571_b200 import distributed as D
        method, M, N, shape, iters = case
        h, g, _, _ = orc.gen_problem(shape[0], shape[1], 6, 30.0, 31, "cg")
        lam = 0.05 * float(np.max(np.abs(orc.adjoint_matvec(h, g))))
        Pr, Pc = D.choose_grid(world, method, M, N)
        pr, pc = divmod(rank, Pc)
        sh = se.NumpyShard(h, g, 1.0, lam, method, M, N, (Pr, Pc), (pr, pc))
        D.run_iterations([sh], DH.TorchComm(Pr, Pc), iters)
        segs = [None] * world
        dist.all_gather_object(segs, sh.segment_v())
        v = D.gather_solution(segs, shape[1], sh.col_bounds)
        if rank == 0:
            ref = orc.solve(method, h, g, M=M, N=N, lam=lam, iters=iters)
            err = np.linalg.norm(v - ref["solution"]) / np.linalg.norm(ref["solution"])
            tr = np.array(sh.trace_rows)
            terr = np.max(np.abs(tr[:, 1] - ref["trace"][:, 1]) / np.maximum(np.abs(ref["trace"][:, 1]), 1e-300))
            # objective trace by the recurrence + gathered A regions; the two-pass schedule
            # closes iteration k's in k + 1 (its last entry comes from the final exact pass)
            n = iters if sh.schedule == "sweep" else iters - 1
            oerr = np.max(np.abs(tr[:n, 2] - ref["trace"][:n, 2]) / np.abs(ref["trace"][:n, 2]))
            out.put((err, terr, oerr, sh.schedule, (Pr, Pc)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("case", [
    ("sectioning", 1, 4, (24, 96), 12),   # 1 x 2 grid: sweep schedule, ghat all-gather
    ("consensus", 4, 1, (32, 64), 12),    # 2 x 1 grid: two-pass, outbox all-gather
    ("hybrid", 2, 2, (24, 80), 10),       # 1 x 2 grid (column sharding preferred)
    ("hybrid", 2, 1, (24, 80), 10),       # 2 x 1 grid: both exchanges
])
def test_two_rank_gloo_orchestration_matches_oracle(case):
    ctx = mp.get_context("spawn")
    out = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, case, out)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=240)
        assert p.exitcode == 0
    err, terr, oerr, sched, grid = out.get(timeout=5)
    assert err <= 1e-12, (err, sched, grid)
    assert terr <= 1e-10, (terr, sched, grid)
    assert oerr <= 1e-10, (oerr, sched, grid)


def test_phase_program():
    from paper_1811_05571_b200.distributed import phase_program
    assert phase_program("sweep", True) == [1, "ghat", 3, 4]
    assert phase_program("sweep", False) == [1, "ghat", 3, "scal", 4]
    assert phase_program("twopass", False) == [1, "ghat", 2, "outbox", 3, "scal", 4]


def test_choose_grid_prefers_column_sharding():
    from paper_1811_05571_b200.distributed import choose_grid
    assert choose_grid(8, "hybrid", 2, 4) == (2, 4)
    assert choose_grid(4, "hybrid", 2, 4) == (1, 4)
    assert choose_grid(2, "hybrid", 2, 4) == (1, 2)
    assert choose_grid(8, "sectioning", 1, 8) == (1, 8)
    assert choose_grid(8, "consensus", 8, 1) == (8, 1)
    with pytest.raises(ValueError):
        choose_grid(3, "consensus", 8, 1)
