#!/usr/bin/env python3
"""Diagnostics: per-phase clock64 timeline of the resident kernel (config 1, 16 iterations)."""
import ctypes
import os
import sys

import numpy as np

os.environ["ADMM_B200_RES_TRACE"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_1811_05571_b200 as admm  # noqa: E402
from paper_1811_05571_b200 import _lib  # noqa: E402

cfg = bench.CONFIGS["1"]
method, m, n, k, snr, seed, kind, M, N, lr, iters, dtype = cfg
p = bench.make_problem(cfg)
plan = admm.AdmmPlan(p, admm.SolverConfig(rho=1.0, lambda_=1.0, max_iters=iters), method, M, N,
                     admm.SolveOptions(dtype=dtype, schedule="resident"))
plan.set_lambda(lr * plan.max_abs_adjoint())
plan.reset()
plan.enqueue(16)
plan.sync()
P = 148
buf = np.zeros(P * 16 * 10, np.float64)
_lib.lib.admm_plan_read(plan._h, 9, buf.ctypes.data, buf.size)
t = buf.view(np.uint64).reshape(P, 16, 10).astype(np.int64)
used = np.nonzero(t[:, 2, 0])[0]
t = t[used]
base = t[:, 2, 0].min()
for it in (2, 3, 4):
    a = t[:, it] - base
    print(f"iter {it}: A start {a[:,0].min()}..{a[:,0].max()}  A end {a[:,1].min()}..{a[:,1].max()}  "
          f"after bar1 {a[:,2].min()}..{a[:,2].max()}  B end {a[:,3].min()}..{a[:,3].max()} (owners {a[:4,3]}) "
          f"after bar2 {a[:,4].min()}..{a[:,4].max()}")
d = t[:, 4]
for name, a, b in [("q load", 0, 5), ("objective rows", 5, 6), ("z", 6, 7), ("update+sums", 7, 8), ("w partial", 8, 1),
                   ("barrier 1", 1, 2), ("phase B", 2, 3), ("barrier 2", 3, 4)]:
    x = d[:, b] - d[:, a]
    print(f"{name:16s} min {x.min():8d} median {int(np.median(x)):8d} max {x.max():8d} cycles")
per = (t[:, 10, 0] - t[:, 2, 0]) / 8
print("cycles per iteration", per.mean(), "CTAs", len(used))
