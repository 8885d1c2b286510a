#!/usr/bin/env python3
"""ncu driver: config 1 on the resident schedule, one launch of 200 iterations."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_1811_05571_b200 as admm  # noqa: E402

cfg = bench.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "1"]
method, m, n, k, snr, seed, kind, M, N, lr, iters, dtype = cfg
p = bench.make_problem(cfg)
plan = admm.AdmmPlan(p, admm.SolverConfig(rho=1.0, lambda_=1.0, max_iters=iters), method, M, N,
                     admm.SolveOptions(dtype=dtype, schedule="resident"))
plan.set_lambda(lr * plan.max_abs_adjoint())
plan.reset()
plan.enqueue(iters)
plan.sync()
print("ok", plan.info()["schedule"])
