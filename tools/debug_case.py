#!/usr/bin/env python3
"""Run one golden case on the GPU with a chosen schedule (debugging aid)."""
import faulthandler
import os
import sys
import time

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
sys.path.insert(0, os.path.join(REPO, "tests"))
faulthandler.enable()

import numpy as np  # noqa: E402

import golden_cases as gc  # noqa: E402
import oracle_lib as orc  # noqa: E402
import paper_1811_05571_b200 as a  # noqa: E402

name, sched = sys.argv[1], sys.argv[2]
obj = len(sys.argv) > 3 and sys.argv[3] == "obj"
entry, ref = gc.load(name)
args = gc.solver_args(entry)
h, g, t = gc.problem(entry, orc.gen_problem)
p = a.SensingProblem(h, g, t)
cfg = a.SolverConfig(rho=args["rho"], lambda_=args["lam"], scl=args["scl"], max_iters=args["iters"],
                     eps_pri=args["eps_pri"], eps_dual=args["eps_dual"])
opts = a.SolveOptions(ragged=args["ragged"], schedule=sched, trace_objective=obj)
t0 = time.time()
with a.AdmmPlan(p, cfg, args["method"], args["M"], args["N"], opts) as plan:
    print("info", plan.info(), flush=True)
    r = plan.solve()
print("solve s", time.time() - t0, "iters", r.iterations_run, flush=True)
if "solution" in ref:
    s = np.max(np.abs(ref["solution"]))
    print("rel err", np.linalg.norm((r.solution - ref["solution"]) / s) / np.linalg.norm(ref["solution"] / s))
