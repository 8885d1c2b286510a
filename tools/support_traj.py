#!/usr/bin/env python3
"""Config 4: per-iteration support size of v and iteration time along the solve from zero
(support schedule).  usage: python tools/support_traj.py [iters] > gpurun_out/support_traj.json"""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
import paper_1811_05571_b200 as admm

iters = int(sys.argv[1]) if len(sys.argv) > 1 else 120
cfg = bench.CONFIGS["4"]
method, m, n, k, snr, seed, kind, M, N, lr, its, dtype = cfg
problem = bench.make_problem(cfg)
plan = admm.AdmmPlan(problem, admm.SolverConfig(rho=1.0, lambda_=1.0, max_iters=its), method, M, N,
                     admm.SolveOptions(dtype=dtype, device=0, trace_objective=True))
plan.set_lambda(lr * plan.max_abs_adjoint())
stream = torch.cuda.ExternalStream(plan.stream(), device=0)
plan.reset()
out = []
prev = 0
for it in range(iters):
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stream); plan.enqueue(1); e1.record(stream); e1.synchronize()
    done, cols = plan.support_stats()
    out.append({"it": it, "ms": e0.elapsed_time(e1), "support": cols - prev})
    prev = cols
print(json.dumps(out))
