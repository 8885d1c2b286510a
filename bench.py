#!/usr/bin/env python3
"""Benchmark of the B200 ADMM hot path (BASELINE.json metric: ADMM iterations/s and
H-stream HBM GB/s, % of B200 peak, at 1/2/4/8 GPUs).

Workload (default, N=1): BASELINE config 4 -- consensus ADMM at scale, complex64 storage,
H 16384 x 262144 i.i.d. CN(0, 1/16384) (32 GiB), 1000-sparse unit-phase truth, 30 dB SNR,
M = 8 row blocks of 2048, rho = 1, lambda = 0.05 max|H^H g|, 1000 iterations, seed 4: the
largest configuration that fits one GPU (configs[1..4]; config 5 is the batched variant of
config 3).  `--config 1|2|3|5` selects another BASELINE config.  A "step" is one ADMM
iteration over the whole problem (both H products, the 8 Woodbury applies, the column
update, the residuals and the objective of the trace).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config 4]

Prints one JSON line (rank 0).  Timing: CUDA events on the plan's stream around K
graph-replayed iterations, after W warm-up iterations, with a barrier + synchronize on both
sides, max over ranks.  Every input is larger than L2 (config 4: 32 GiB of H; config 2:
512 MiB), so each iteration streams HBM; no flush is needed.  `e2e`: the public API
(AdmmPlan.set_g + solve) with the measurement vector copied from pinned host memory and the
solution + trace read back.

--gpus N > 1 outside torchrun re-executes itself under `torch.distributed.run
--nproc-per-node N` (one process per GPU); the plan of every rank owns its NCCL
communicators.

The reference arm (`--impl reference`) runs the UNMODIFIED reference solver
(oracle/_ref/admmsplit_ref, the reference headers compiled where they lie) on the host
cores, on inputs from the reference's own generator; it never imports this package.
"""
from __future__ import annotations

import argparse
import json
import os
import shutil
import socket
import subprocess
import sys
import tempfile
import threading
import time

import numpy as np

REPO = os.path.dirname(os.path.abspath(__file__))
REF_BIN = os.path.join(REPO, "oracle", "_ref", "admmsplit_ref")

CONFIGS = {
    # name: (method, rows, cols, k, snr, seed, kind, M, N, lambda_rel, iters, dtype)
    "1": ("consensus", 256, 2048, 16, 30.0, 1, "cg", 4, 1, 0.05, 200, "c128"),
    "2": ("sectioning", 1024, 32768, 64, 30.0, 2, "cg", 1, 8, 0.05, 300, "c128"),
    "3": ("hybrid", 3072, 32768, 300, 30.0, 3, "cra", 2, 4, 0.03, 500, "c64"),
    "4": ("consensus", 16384, 262144, 1000, 30.0, 4, "cg", 8, 1, 0.05, 1000, "c64"),
    "5": ("hybrid", 3072, 32768, 64, 30.0, 3, "cra_batch", 2, 4, 0.03, 500, "c64"),
}
DEFAULT_CONFIG = "4"


def describe(cfg):
    method, m, n, k, snr, seed, kind, M, N, lr, iters, dtype = cfg
    grid = f"M={M}" if method == "consensus" else f"N={N}" if method == "sectioning" else f"{M}x{N}"
    if kind == "cra":
        return (f"{method} ADMM {dtype} CRA-like H {m}x{n} (24 tx x 128 freq, 32^3 voxels), {k}-voxel "
                f"planar patch, {snr:g} dB seed {seed}, {grid}, rho=1, lambda={lr}*max|H^H g|, {iters} iterations")
    if kind == "cra_batch":
        return (f"{method} ADMM {dtype} CRA-like H {m}x{n} (config 3's generator and seed), {k} scenes of "
                f"100-400 planar-patch voxels, {snr:g} dB seed {seed}, {grid}, rho=1, "
                f"lambda_b={lr}*max|H^H g_b| per scene, {iters} iterations")
    return (f"{method} ADMM {dtype} H {m}x{n} CN(0,1/{m}) {k}-sparse {snr:g} dB seed {seed}, "
            f"{grid}, rho=1, lambda={lr}*max|H^H g|, {iters} iterations")


def config_dict(name):
    """The `config` object of BOTH arms (identical by construction)."""
    return {"workload": f"config {name}: {describe(CONFIGS[name])}"}


def peaks():
    p = os.path.join(REPO, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy)"
    return 6650.0, "fallback (B200_PROFILING.md)"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index=0):
        self.index = index
        self.rows = []
        self.proc = None

    def __enter__(self):
        if shutil.which("nvidia-smi"):
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def __exit__(self, *exc):
        if self.proc:
            time.sleep(0.25)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4)
                          if len(r) > 3 + i and r[3 + i].lower() == "active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons, "samples": len(self.rows)}


def dist_env():
    return (int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("RANK", "0")),
            int(os.environ.get("LOCAL_RANK", "0")))


# ----------------------------------------------------------------------------- reference
def reference_sample(name):
    """The bounded sample of config `name` the unmodified reference runs on (SURVEY §8d,
    BASELINE.md §4): the reference's own generator, the config's columns, blocks, method and
    lambda rule, with fewer rows where the full size is minutes of setup or does not fit
    host memory.  The reference's per-iteration cost is linear in the H bytes (3 FP64 passes
    over H: the two Woodbury products and the objective), so it/s scales by rows_sample /
    rows.  The CRA-like H of configs 3/5 has no reference generator: a random-phase H of
    the same shape stands in (the reference's timing does not depend on the values)."""
    method, m, n, k, snr, seed, kind, M, N, lr, iters, dtype = CONFIGS[name]
    rows = {"1": m, "2": m, "3": 768, "4": 256, "5": 768}[name]
    gkind = "rp" if kind.startswith("cra") else "cg"
    kk = min(k, n) if kind != "cra_batch" else 300
    scenes = k if kind == "cra_batch" else 1
    return dict(method=method, rows=rows, cols=n, k=kk, snr=snr, seed=seed, kind=gkind, M=M, N=N, lr=lr,
                scale=rows / m, scenes=scenes, full_rows=m)


def run_reference(name, iters, threads=None):
    """Time the unmodified reference on the host cores: generate the sample with the
    reference's gen_problem, solve with its solver (observer timestamps; setup excluded)."""
    if not os.path.exists(REF_BIN):
        return None
    s = reference_sample(name)
    threads = threads or max(1, min(s["M"] * s["N"], os.cpu_count() or 1))
    tmp = tempfile.mkdtemp(prefix="admm_ref_")
    try:
        d = os.path.join(tmp, "in")
        subprocess.run([REF_BIN, "gen", f"out={d}", f"m={s['rows']}", f"n={s['cols']}", f"k={s['k']}",
                        f"snr={s['snr']}", f"seed={s['seed']}", f"kind={s['kind']}"], check=True,
                       capture_output=True, timeout=1800)
        out = os.path.join(tmp, "out")
        subprocess.run([REF_BIN, "solve", f"in={d}", f"out={out}", f"method={s['method']}", f"M={s['M']}",
                        f"N={s['N']}", "rho=1", f"lambda={s['lr']}", "lambda_rel=1", f"iters={max(2, iters)}",
                        f"threads={threads}"], check=True, capture_output=True, timeout=3600)
        md = dict(line.split() for line in open(os.path.join(out, "meta.txt")))
        measured = float(md["it_per_s"])
        value = measured * s["scale"] / s["scenes"]
        what = (f"full workload" if s["scale"] == 1.0 else
                f"first {s['rows']} of {s['full_rows']} rows (reference gen_problem, kind {s['kind']}, all "
                f"{s['cols']} columns, M={s['M']} N={s['N']}), it/s x {s['scale']:g} (cost linear in H size)")
        if s["scenes"] > 1:
            what += f"; one scene per reference solve, it/s / {s['scenes']} scenes"
        return {"value": value, "measured": measured, "scale": s["scale"] / s["scenes"],
                "setup_s": float(md["setup_s"]), "threads": threads,
                "iters": max(2, iters),
                "sample": (f"unmodified reference ({s['method']}_solve, oracle/_ref) on {what}; {max(2, iters)} "
                           f"iterations after its serial setup ({float(md['setup_s']):.1f} s, excluded); it/s "
                           f"from observer timestamps ({measured:.4g} measured); includes the reference's "
                           f"per-iteration objective pass")}
    finally:
        shutil.rmtree(tmp, ignore_errors=True)


def bench_reference(args):
    ws, rank, _ = dist_env()
    if rank != 0:
        return
    iters = min(max(args.steps, 2), 20) + min(args.warmup, 3)
    r = run_reference(args.config, iters)
    if r is None:
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/admmsplit_ref not built"}))
        return
    v = r["value"]
    line = {"metric": "ADMM iterations/s", "value": v, "unit": "iterations/s", "impl": "reference",
            # a step = one reference iteration on the bounded sample (what was executed and timed);
            # `value` scales it to the whole workload (cpu_baseline.sample says how)
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1000.0 / r["measured"],
            "sample_scale": r["scale"],
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "c128",
            "data": "synthetic", "config": config_dict(args.config),
            "cpu_baseline": {"value": v, "unit": "iterations/s", "cores": r["threads"], "kind": "reference",
                             "sample": r["sample"]},
            "e2e": {"value": v, "unit": "iterations/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "setup_s": r["setup_s"]}
    print(json.dumps(line))


# ----------------------------------------------------------------------------- ours
def make_problem(cfg):
    import paper_1811_05571_b200 as admm
    method, m, n, k, snr, seed, kind, M, N, lr, iters, dtype = cfg
    if kind == "cra":  # BASELINE config 3: CRA-like structured H
        return admm.cra_problem(seed=seed, n_vox=k, snr_db=snr, dtype=dtype)
    if kind == "cra_batch":  # BASELINE config 5: config 3's H, k scenes of 100-400 voxels
        h = admm.cra_matrix(seed=seed, dtype=dtype)
        g, truth = admm.cra_scenes(h, k, seed=seed)
        return admm.SensingProblem(h, g, None)
    return admm.gen_problem(m, n, k, snr, seed, admm.ProblemKind.ComplexGaussian, dtype=dtype)


def kernel_roofline(plan, info, problem, name):
    """Dominant kernel of one iteration: per-kernel CUDA-event times of individually launched
    kernels on the plan's stream (`plan.profile`), algorithmic bytes per launch (SURVEY §8d:
    one pass over the stored H = rows x cols x sizeof(element); the packed K once)."""
    kern = plan.profile(iters=10)
    hb, kb = info["h_bytes"], info["k_bytes"]
    algo = {"gemv_n(H,c)": hb, "gemv_h(H,q)": hb, "gemv_n(K,r)": kb, "hemv(Kpacked,r)": kb, "sweep(H)": hb,
            "resident(iteration)": 2 * hb}
    algo = {k: v for k, v in algo.items() if k in kern}
    peak, peak_kind = peaks()
    if plan.batch > 1:  # config 5: FP64 SIMT compute-bound skinny GEMMs (8 flop per complex MAC)
        rows, cols = problem.h.shape
        algo = {"bgemm(H,C)": 8.0 * rows * cols * plan.batch, "bgemm_adj(H,Q)": 8.0 * rows * cols * plan.batch}
    dom = max(algo, key=lambda x: kern[x])
    achieved = algo[dom] / (kern[dom] / 1000.0) / 1e9
    traffic = None
    summ = os.path.join(REPO, "profiles", "ncu_traffic.json")
    if os.path.exists(summ):
        traffic = json.load(open(summ)).get(f"config{name}", {}).get(dom)
    if plan.batch > 1:
        roof = {"bound": "fp64-simt", "kernel": dom, "achieved": achieved / 1e3, "peak": 34.1,
                "peak_kind": "measured FP64 FMA peak (tools/fp_peak.cu; not in MEASURED_PEAKS.json)",
                "unit": "TFLOP/s", "frac": achieved / 1e3 / 34.1}
    else:
        roof = {"bound": "hbm", "kernel": dom, "achieved": achieved, "peak": peak, "peak_kind": peak_kind,
                "unit": "GB/s", "frac": achieved / peak,
                "peak_note": "copy bandwidth (read+write); read-only streams can exceed it"}
    roof.update({"traffic": traffic, "algorithmic_per_launch": algo[dom], "avg_launch_ms": kern[dom]})
    return roof, {"isolated_launch_ms": kern,
                  "note": "CUDA events around individually launched kernels of one iteration on the plan's "
                          "stream (not the graph-replayed chain: their sum exceeds ms_per_step)"}


def cpu_baseline(name):
    r = run_reference(name, 5)
    if not r:
        return None
    return {"value": r["value"], "unit": "iterations/s", "cores": r["threads"], "kind": "reference",
            "sample": r["sample"]}


def bench_ours(args):
    import torch

    import paper_1811_05571_b200 as admm
    from paper_1811_05571_b200 import distributed as D

    ws, rank, local = dist_env()
    cfg = CONFIGS[args.config]
    method, m, n, k, snr, seed, kind, M, N, lr, iters, dtype = cfg
    torch.cuda.set_device(local)
    # ws > 1: one process per GPU, the plan owns its NCCL communicators; BENCH_FORCE_DIST=1
    # runs that path with a world of one (schema check of the N > 1 line)
    sharded = ws > 1 or os.environ.get("BENCH_FORCE_DIST") == "1"
    if ws > 1:
        import torch.distributed as dist
        dist.init_process_group("gloo")  # plumbing only (NCCL id broadcast, timing max); data moves over NCCL
    problem = make_problem(cfg)
    scfg = admm.SolverConfig(rho=1.0, lambda_=1.0, max_iters=iters)
    opts = admm.SolveOptions(dtype=dtype, device=local, trace_objective=args.trace_objective)
    t_setup = time.perf_counter()
    plan = D.dist_plan(problem, scfg, method, M, N, opts) if sharded else admm.AdmmPlan(problem, scfg, method, M, N,
                                                                                         opts)
    if plan.batch > 1:  # per-scene lambda_b = c max|H^H g_b|
        lams = lr * plan.max_abs_adjoint_batched()
        plan.set_lambdas(lams)
    else:
        plan.set_lambda(lr * plan.max_abs_adjoint())
    setup_s = time.perf_counter() - t_setup
    info = plan.info()
    stream = torch.cuda.ExternalStream(plan.stream(), device=local)

    def barrier():
        torch.cuda.synchronize(local)
        if ws > 1:
            torch.distributed.barrier()
        torch.cuda.synchronize(local)

    # ---- device-resident throughput (value)
    plan.reset()
    # The support schedule's cost depends on the iterate: v's support is 97k of 262144 columns
    # at iteration 7 of config 4's solve from zero and the truth's 1000 from iteration ~100 on
    # (tools/support_traj.py).  The timed window is placed mid-solve (the state of iteration
    # iters/2, reached by running those iterations untimed), where 90% of the solve's
    # iterations are; the WHOLE solve from zero, dense early iterations included, is `e2e`
    # and `run.whole_solve`.  Schedules whose cost is data-independent are timed from zero.
    warm = max(args.warmup, 3)
    prime = 0
    if int(info["schedule"]) == 5:
        prime = iters // 2 if iters // 2 + warm + args.steps <= iters else max(0, iters - warm - args.steps)
        plan.enqueue(prime)
    plan.enqueue(warm)
    plan.sync()
    barrier()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    stats0 = plan.support_stats() if int(info["schedule"]) == 5 else None
    with ClockSampler(local) as clk:
        e0.record(stream)
        plan.enqueue(args.steps)
        e1.record(stream)
        e1.synchronize()
    barrier()
    ms = e0.elapsed_time(e1)
    if ws > 1:
        t = torch.tensor([ms], dtype=torch.float64)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        ms = float(t.item())
    ms_per_step = ms / args.steps
    value = args.steps / (ms / 1000.0)  # whole job: every rank runs its shard of the same iterations
    support = None
    if int(info["schedule"]) == 5:  # support schedule: the columns of v's support read per iteration
        done, cols = plan.support_stats()
        done0, cols0 = stats0
        mean_cols = (cols - cols0) / max(done - done0, 1)
        sbytes = mean_cols * m * (8 if dtype == "c64" else 16)
        support = {"mean_support_columns": mean_cols, "of_columns": n, "bytes_per_iter": sbytes,
                   "frac_of_H": sbytes / info["h_bytes"],
                   "note": "a' = H v' over the nonzero columns of the soft-thresholded v (exact: skipped terms "
                           "are exact zeros); w' = 2a' - a - G q (DESIGN.md §4); averaged over the timed "
                           "iterations"}

    whole = None
    if prime:  # the whole solve from zero on the device (no host copies): the dense early iterations included
        plan.reset()
        plan.enqueue(warm)  # clocks / graphs warm; then start over
        plan.reset()
        w0 = torch.cuda.Event(enable_timing=True)
        w1 = torch.cuda.Event(enable_timing=True)
        w0.record(stream)
        plan.enqueue(iters)
        w1.record(stream)
        w1.synchronize()
        wms = w0.elapsed_time(w1)
        if ws > 1:
            t = torch.tensor([wms], dtype=torch.float64)
            torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
            wms = float(t.item())
        whole = {"iterations": iters, "device_ms": wms, "iterations_per_s": iters / (wms / 1000.0),
                 "note": "all iterations of the config's solve from zero iterates, CUDA events on the plan's stream"}

    if not sharded:
        roof, kern = kernel_roofline(plan, info, problem, args.config)
    else:  # the plan's kernels are not launched one by one: whole-iteration HBM roofline
        peak, peak_kind = peaks()
        passes = 1 if int(info["schedule"]) in (2, 5) else 2  # sweep / support: one dense pass over this rank's H
        achieved = info["h_bytes"] * passes / (ms_per_step / 1000.0) / 1e9
        roof = {"bound": "hbm", "kernel": f"whole iteration ({passes} pass(es) over this rank's H)",
                "achieved": achieved, "peak": peak, "peak_kind": peak_kind, "unit": "GB/s", "frac": achieved / peak,
                "traffic": None, "algorithmic_per_launch": info["h_bytes"] * passes, "avg_launch_ms": ms_per_step}
        kern = None

    # ---- end to end through the public API: g from pinned memory, full solve, solution and
    # trace back to the host (AdmmPlan.set_g + solve)
    g_pinned = torch.from_numpy(np.ascontiguousarray(problem.g).view(np.float64)).pin_memory()
    g_host = g_pinned.numpy().view(np.complex128)
    plan.set_g(g_host)
    plan.solve()  # warm (graphs captured)
    barrier()
    e2e_solves = 1 if iters >= 1000 else max(1, min(3, args.steps // iters + 1))
    t0 = time.perf_counter()
    for _ in range(e2e_solves):
        plan.set_g(g_host)
        rep = plan.solve()
    t1 = time.perf_counter()
    dt = t1 - t0
    if ws > 1:
        t = torch.tensor([dt], dtype=torch.float64)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        dt = float(t.item())
    e2e_value = e2e_solves * iters / dt
    h2d = problem.g.nbytes
    d2h = rep.solution.nbytes + iters * 3 * 8 * plan.batch

    if rank != 0:
        return
    hb = info["h_bytes"]
    h_stream_gbs = info["h_stream_bytes_per_iter"] / (ms_per_step / 1000.0) / 1e9
    peak, peak_kind = peaks()
    sched = {1: "two-pass", 2: "single-HBM-pass sweep", 3: "batched scenes (FP64 SIMT GEMMs)",
             4: "resident (H in SMEM, one persistent cooperative kernel)",
             5: "support (one dense H pass + the columns of v's support)"}[int(info["schedule"])]
    line = {
        "metric": "ADMM iterations/s", "value": value, "unit": "iterations/s", "n_gpus": ws,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step,
        "higher_is_better": True, "scaling": "strong" if ws > 1 else "weak", "vs_baseline": None,
        "dtype": dtype, "data": "synthetic (seeded generator of the reference, generate.hpp)",
        "config": config_dict(args.config),
        "run": {"schedule": sched, "parallelism": (f"{info['grid_pr']}x{info['grid_pc']} process grid, NCCL owned "
                                                    f"by the plan" if sharded else "single GPU, all blocks"),
                "l2": f"inputs larger than L2 (H {hb * ws / 2**20:.0f} MiB over {ws} GPU(s)), no flush needed",
                "lambda": plan.cfg.lambda_, "trace_objective": bool(args.trace_objective),
                "setup_s": setup_s, "setup_phase_s": info["setup_phase_s"],
                "setup_gram": {"device_s": info["gram_device_s"],
                               "tflops_fp64": info["gram_flops"] / max(info["gram_device_s"], 1e-12) / 1e12,
                               "kernel": "gram_dmma_kernel (mma.sync m8n8k4 f64), launched per block under the upload"},
                "setup_inverse": {"device_s": info["inverse_device_s"],
                                  "tflops_fp64": info["inverse_flops"] / max(info["inverse_device_s"], 1e-12) / 1e12,
                                  "kernel": "blocked Gauss-Jordan, 64-wide panels, DMMA rank-64 updates"},
                "timing": "CUDA events on the plan's stream around K graph-replayed "
                                              "iterations, max over ranks",
                "window": (f"iterations {prime + warm}..{prime + warm + args.steps - 1} of the {iters}-iteration solve "
                           f"(first {prime} iterations run untimed to reach the mid-solve state: the support schedule's "
                           f"cost follows |supp v|, see run.whole_solve and e2e for the solve from zero)" if prime else
                           f"iterations {warm}..{warm + args.steps - 1} of the solve from zero (cost is data-independent)")},
        "h_stream_gbs": h_stream_gbs, "h_stream_frac_of_peak": h_stream_gbs / peak,
        "h_stream_note": "2 x |H| per iteration (SURVEY §8d's two-pass H-stream bytes) / time: a single-pass "
                         "schedule can exceed 1.0",
        "hbm_compulsory_gbs": (info["hbm_bytes_per_iter"] + (support["bytes_per_iter"] if support else 0))
                              / (ms_per_step / 1000.0) / 1e9,
        "hbm_compulsory_frac": (info["hbm_bytes_per_iter"] + (support["bytes_per_iter"] if support else 0))
                               / (ms_per_step / 1000.0) / 1e9 / peak,
        "e2e": {"value": e2e_value, "unit": "iterations/s", "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                "step": f"one full solve ({iters} iterations) via AdmmPlan.set_g + solve from pinned host memory"},
        "gpu_launches": int(info["launches_per_iter"]) * args.steps if int(info["schedule"]) != 4 else 1,
        "clocks": clk.summary(),
    }
    if whole:
        line["run"]["whole_solve"] = whole
    line["roofline"] = roof
    if support:
        line["support"] = support
    if kern:
        line["kernels"] = kern
    if sharded:
        xb = info["exchange_bytes_per_iter"]
        line["nccl"] = {"bytes_per_iter_per_rank": xb, "nvlink_term_us": xb / 900e9 * 1e6,
                        "peak_gbs": 900.0, "peak_kind": "nominal NVLink 5 per direction",
                        "frac_of_iteration": (xb / 900e9) / (ms_per_step / 1000.0)}
    if not args.no_cpu_baseline:  # rank 0 only, after the GPU work
        cb = cpu_baseline(args.config)
        if cb:
            line["cpu_baseline"] = cb
    print(json.dumps(line))


def relaunch_under_torchrun(args):
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def parse_args(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=300)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default=DEFAULT_CONFIG, choices=sorted(CONFIGS))
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-trace-objective", dest="trace_objective", action="store_false",
                    help="drop the per-iteration objective from the trace (default: on, as the "
                         "reference evaluates it every iteration, solvers.hpp:146; here by the "
                         "H-pass-free recurrence, DESIGN.md §2)")
    return ap.parse_args(argv)


def main():
    args = parse_args()
    ws = int(os.environ.get("WORLD_SIZE", "0"))
    if args.gpus > 1 and ws == 0:  # one process per GPU
        sys.exit(relaunch_under_torchrun(args))
    if ws and ws != args.gpus:
        sys.exit(f"bench.py: WORLD_SIZE={ws} but --gpus {args.gpus}")
    sys.path.insert(0, REPO)
    if args.impl == "reference":
        bench_reference(args)
    else:
        bench_ours(args)


if __name__ == "__main__":
    main()
