#!/usr/bin/env python3
"""Run under torchrun (any world size): sharded solve of a small problem, eager vs
CUDA-graph-captured iterations (NCCL collectives inside the graph).  Prints one JSON line
on rank 0 with the max abs difference (expected 0: same kernels, same order)."""
import json
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
sys.path.insert(0, os.path.join(REPO, "tests"))
import dist_harness as DH  # noqa: E402  (test transport)
import paper_1811_05571_b200 as admm  # noqa: E402
from paper_1811_05571_b200 import distributed as D  # noqa: E402


def main():
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    ws, rank = dist.get_world_size(), dist.get_rank()
    out = {}
    for method, M, N, shape in [("sectioning", 1, 8, (64, 2048)), ("hybrid", 2, 4, (96, 1024)),
                                ("consensus", 4, 1, (128, 1024))]:
        p = admm.gen_problem(shape[0], shape[1], 8, 30.0, 23)
        lam = 0.05 * float(np.max(np.abs(p.h.conj().T @ p.g)))
        cfg = admm.SolverConfig(rho=1.0, lambda_=lam, max_iters=32)
        Pr, Pc = D.choose_grid(ws, method, M, N)
        sh = D.ShardPlan(p, cfg, method, M, N, (Pr, Pc), divmod(rank, Pc),
                         admm.SolveOptions(device=local, trace_objective=False))
        comm = DH.TorchComm(Pr, Pc)
        D.run_iterations([sh], comm, 16)
        sh.sync()
        eager = sh.segment_v()
        sh.reset()
        D.prime([sh], comm)
        g = DH.GraphedIterations(sh, comm, iters_per_graph=8)  # captured from the current state
        sh.reset()
        D.prime([sh], comm)
        g.run(16)
        sh.sync()
        graphed = sh.segment_v()
        diff = max(float(np.max(np.abs(eager[j] - graphed[j]))) for j in eager)
        ref = admm.hybrid_solve(p, admm.SolverConfig(rho=1.0, lambda_=lam, max_iters=16), M, N,
                                admm.SolveOptions(device=local, trace_objective=False)) if method == "hybrid" else None
        out[method] = {"eager_vs_graph_maxabs": diff, "grid": [Pr, Pc], "schedule": sh.schedule,
                       "iters": sh.state()[0]}
        if ref is not None:
            v = D.gather_solution([graphed], shape[1], sh.col_bounds) if ws == 1 else None
            if v is not None:
                out[method]["vs_single_plan_rel"] = float(np.linalg.norm(v - ref.solution) / np.linalg.norm(ref.solution))
        sh.close()
    if rank == 0:
        print(json.dumps(out))
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
