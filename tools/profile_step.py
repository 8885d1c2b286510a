#!/usr/bin/env python3
"""Minimal driver for ncu: build the config-N plan, then run a few ADMM iterations as
individual (non-graph) launches so ncu can attribute them.  Usage:
  ncu ... python tools/profile_step.py --config 2 --iters 3
"""
import argparse
import os
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)

import bench  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="2")
    ap.add_argument("--iters", type=int, default=3)
    a = ap.parse_args()
    import paper_1811_05571_b200 as admm
    cfg = bench.CONFIGS[a.config]
    method, m, n, k, snr, seed, kind, M, N, lr, iters, dtype = cfg
    p = bench.make_problem(cfg)
    plan = admm.AdmmPlan(p, admm.SolverConfig(rho=1.0, lambda_=1.0, max_iters=iters), method, M, N,
                         admm.SolveOptions(dtype=dtype, trace_objective=False))
    plan.set_lambda(lr * plan.max_abs_adjoint())
    plan.reset()
    print(plan.profile(iters=a.iters))


if __name__ == "__main__":
    main()
