#!/usr/bin/env python3
"""ncu driver: one iteration of the config-5 batched plan (64 CRA scenes)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_1811_05571_b200 as admm  # noqa: E402

cfg = bench.CONFIGS["5"]
p = bench.make_problem(cfg)
plan = admm.AdmmPlan(p, admm.SolverConfig(rho=1.0, lambda_=1.0, max_iters=10), "hybrid", 2, 4,
                     admm.SolveOptions(dtype="c64", trace_objective=False))
plan.set_lambdas(0.03 * plan.max_abs_adjoint_batched())
plan.reset()
print(plan.profile(iters=2))
