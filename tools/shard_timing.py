#!/usr/bin/env python3
"""Time one rank's phase-1 + phase-4 work of a column-sharded grid on ONE GPU, without
collectives (the other ranks' ghat slots stay as primed): the per-rank kernel cost of the
Pc-way sharded config, for the L2-residency decision (ADMM_B200_KEEP_L2).  Diagnostic
only; the numbers are not bench values."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1811_05571_b200 as admm  # noqa: E402
from paper_1811_05571_b200 import distributed as D  # noqa: E402


class NullComm:
    """No collectives: the other ranks' slots keep their primed values."""
    def exchange(self, which, shards, in_graph=False):
        pass


def main():
    pc_grid = int(sys.argv[1]) if len(sys.argv) > 1 else 8
    p = admm.gen_problem(1024, 32768, 64, 30.0, 2)
    cfg = admm.SolverConfig(rho=1.0, lambda_=0.05, max_iters=4000)
    sh = D.ShardPlan(p, cfg, "sectioning", 1, 8, (1, pc_grid), (0, 0),
                     admm.SolveOptions(device=0, trace_objective=False))
    comm = NullComm()
    D.prime([sh], comm)
    g = D.GraphedIterations(sh, comm, iters_per_graph=16)
    st = sh.stream()
    g.run(64)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    n = 512
    e0.record(st)
    g.run(n)
    e1.record(st)
    e1.synchronize()
    ms = e0.elapsed_time(e1) / n
    print(json.dumps({"grid": [1, pc_grid], "schedule": sh.schedule, "keep_l2": os.environ.get("ADMM_B200_KEEP_L2", "auto"),
                      "fused_scal": sh.fused_scal, "ms_per_iter": ms}))
    sh.close()


if __name__ == "__main__":
    main()
