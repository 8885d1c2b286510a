#!/usr/bin/env python3
"""Diagnostics of the slab sweep (admm_slab.cuh) on a BASELINE config: iteration time and
the per-strip clock64 timeline of the first CTAs (ADMM_B200_SLAB_TRACE).

  python tools/slab_diag.py --config 3 [--env ADMM_B200_SLAB_C=2 ...]

Timeline events per strip k (trace[(cta*64 + k)*8 + ev], compute warp 0 and the D warps):
  0 (C) start (stage landed)   1 (C) end (z partial published)
  2 (A) start (c of the strip landed)   3 (A) end
  4 D: local z partials complete   5 D: c published
"""
import argparse
import os
import sys
import tempfile

import numpy as np

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="3")
    ap.add_argument("--iters", type=int, default=100)
    ap.add_argument("--env", action="append", default=[])
    ap.add_argument("--trace", action="store_true")
    a = ap.parse_args()
    for kv in a.env:
        k, v = kv.split("=", 1)
        os.environ[k] = v
    tfile = None
    if a.trace:
        tfile = tempfile.mktemp(suffix=".bin")
        os.environ["ADMM_B200_SLAB_TRACE"] = tfile
    import torch

    import bench
    import paper_1811_05571_b200 as admm
    cfg = bench.CONFIGS[a.config]
    method, m, n, k, snr, seed, kind, M, N, lr, iters, dtype = cfg
    p = bench.make_problem(cfg)
    plan = admm.AdmmPlan(p, admm.SolverConfig(rho=1.0, lambda_=1.0, max_iters=iters), method, M, N,
                         admm.SolveOptions(dtype=dtype, trace_objective=False, schedule="sweep"))
    plan.set_lambda(lr * plan.max_abs_adjoint())
    info = plan.info()
    stream = torch.cuda.ExternalStream(plan.stream())
    plan.reset()
    plan.enqueue(8)
    plan.sync()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    plan.enqueue(a.iters)
    e1.record(stream)
    e1.synchronize()
    ms = e0.elapsed_time(e1) / a.iters
    kern = plan.profile(iters=5)
    print(f"config {a.config} env {a.env}: {1e3 / ms:.1f} it/s ({ms * 1e3:.1f} us/iter) "
          f"sweep C={info['slab_cluster']} RB={info['slab_row_bytes']} RPW={info['slab_rows']} grid={info['grid_sweep']}")
    print("  isolated launches (us):", {k: round(v * 1e3, 1) for k, v in kern.items()})
    if tfile:
        plan.close()
        t = np.fromfile(tfile, dtype=np.uint64).astype(np.float64).reshape(-1, 64, 8)
        ncta = t.shape[0]
        entry, exitt = t[:, 0, 6], t[:, 0, 7]
        print(f"  CTAs {ncta}: kernel duration (cycles) mean {np.mean(exitt - entry):.0f}")
        if int(info['slab_row_bytes']) == 16:  # fused loop: 0 loop top, 2 stage landed, 3 c landed, 1 end
            w = t[:, 32:48, :4]  # per compute warp: loop cycles, stage wait, c wait, fused strips
            n = np.maximum(w[:, :, 3], 1)
            print(f"  per compute warp, per fused strip (all CTAs): loop {np.mean(w[:, :, 0] / n):.0f} cyc | stage wait "
                  f"{np.mean(w[:, :, 1] / n):.0f} (warp 0: {np.mean(w[:, 0, 1] / n[:, 0]):.0f}, warp 15: "
                  f"{np.mean(w[:, 15, 1] / n[:, 15]):.0f}) | c wait {np.mean(w[:, :, 2] / n):.0f} (max warp "
                  f"{np.max(np.mean(w[:, :, 2] / n, axis=0)):.0f})")
            for cta in (0, 1, ncta // 2, ncta - 1):
                r = t[cta][:32]
                ks = np.nonzero((r[:, 0] > 0) & (r[:, 1] > 0) & (r[:, 3] > 0))[0]
                ks = ks[4:-2]
                per = np.diff(r[ks, 0])
                wf, wc, cmp_ = r[ks, 2] - r[ks, 0], r[ks, 3] - r[ks, 2], r[ks, 1] - r[ks, 3]
                top = r[ks[1:], 0] - r[ks[:-1], 1]
                dz = r[ks, 5] - r[ks, 4]
                zl = r[ks, 4] - r[ks, 1]  # D: all z partials of strip k in, after warp 0 published its own
                f = lambda x: f"{np.mean(x):.0f} (med {np.median(x):.0f}, p90 {np.percentile(x, 90):.0f})"
                print(f"  cta {cta}: strips {len(ks)} per strip {f(per)} | wait stage {f(wf)} | wait c {f(wc)} | "
                      f"compute {f(cmp_)} | loop end->top {f(top)} | D z->c {f(dz)} | warp0 z -> all z {f(zl)}")
            return
        for cta in (0, 1, ncta // 2):
            r = t[cta]
            ok = (r[:, 0] > 0) & (r[:, 3] > 0)
            ks = np.nonzero(ok)[0]
            if len(ks) < 4:
                continue
            ks = ks[2:-1]
            c = np.median(r[ks, 1] - r[ks, 0])
            per = np.median(np.diff(r[ks, 0]))
            await_ = np.median(r[ks, 2] - r[ks - 1, 1]) if len(ks) else 0
            a_ = np.median(r[ks, 3] - r[ks, 2])
            dz = np.median(r[ks, 5] - r[ks, 4]) if np.all(r[ks, 4] > 0) else -1
            print(f"  cta {cta}: per strip {per:.0f} cyc | C {c:.0f} | A {a_:.0f} | C->A gap {await_:.0f} | "
                  f"D z->c {dz:.0f} | first strip at {r[0, 0] - entry[cta]:.0f} cyc after entry")


if __name__ == "__main__":
    main()
