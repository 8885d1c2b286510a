"""GPU: multi-GPU plans.

* The plan-owned NCCL path (admm_plan_create_dist / _create_multi, admm_dist.inc) with a
  world of one -- the whole distributed driver (phases, grouped all-gathers, graph capture,
  gathered solution/trace/objective, early stop, observer, NumericalError) on the one GPU
  of the test box, against the oracle.
* The real CUDA shard plans of larger grids (1x2 ... 4x2) on the ONE GPU, exchanging
  through the test transport LoopbackComm (device copies between phases; no kernel ever
  waits for another): every shard kernel and buffer layout of the N > 1 path, including
  the sharded objective (A regions, gathered rows), against the oracle.
"""
import numpy as np
import pytest

import dist_harness as DH
import oracle_lib as orc

pytestmark = pytest.mark.gpu


def rel(a, b):
    s = float(np.max(np.abs(b)))
    return float(np.linalg.norm(a / s - b / s) / np.linalg.norm(b / s))


@pytest.mark.parametrize("method,M,N,shape,P,iters", [
    ("sectioning", 1, 8, (64, 2048), 2, 20),
    ("sectioning", 1, 8, (64, 2048), 4, 20),
    ("consensus", 4, 1, (256, 2048), 2, 30),
    ("consensus", 4, 1, (256, 2048), 4, 30),
    ("hybrid", 2, 4, (96, 1024), 2, 15),
    ("hybrid", 2, 4, (96, 1024), 8, 15),
    ("hybrid", 4, 2, (128, 512), 4, 15),
])
def test_sharded_plans_match_oracle(method, M, N, shape, P, iters):
    import paper_1811_05571_b200 as admm
    from paper_1811_05571_b200 import distributed as D
    p = admm.gen_problem(shape[0], shape[1], 8, 30.0, 23)
    lam = 0.05 * float(np.max(np.abs(orc.adjoint_matvec(p.h, p.g))))
    cfg = admm.SolverConfig(rho=1.0, lambda_=lam, max_iters=iters)
    Pr, Pc = D.choose_grid(P, method, M, N)
    shards = [D.ShardPlan(p, cfg, method, M, N, (Pr, Pc), divmod(r, Pc)) for r in range(P)]
    D.run_iterations(shards, DH.LoopbackComm(Pr, Pc), iters)
    for sh in shards:
        sh.sync()
    v = D.gather_solution([sh.segment_v() for sh in shards], shape[1], shards[0].col_bounds)
    ref = orc.solve(method, p.h, p.g, M=M, N=N, lam=lam, iters=iters)
    err = np.linalg.norm(v - ref["solution"]) / np.linalg.norm(ref["solution"])
    assert err <= 1e-9, (err, shards[0].schedule, (Pr, Pc))
    # every rank closed the same iterations with the same residual and objective trace
    trs = [sh.trace() for sh in shards]
    for tr in trs:
        assert tr.shape[0] == iters
        np.testing.assert_array_equal(tr, trs[0])
    rd = trs[0][:, 1]
    assert np.max(np.abs(rd - ref["trace"][:, 1]) / np.abs(ref["trace"][:, 1])) <= 1e-8
    # objective by the recurrence + gathered A regions (two-pass closes k-1 in iteration k)
    n = iters if shards[0].schedule == "sweep" else iters - 1
    ob = trs[0][:n, 2]
    assert np.max(np.abs(ob - ref["trace"][:n, 2]) / np.abs(ref["trace"][:n, 2])) <= 1e-9


@pytest.mark.parametrize("P,dtype", [(2, "c128"), (4, "c128"), (4, "c64")])
def test_sharded_support_schedule_matches_oracle(P, dtype):
    """Consensus shards on the support schedule (one dense H pass per rank and iteration: w = H c
    from the support of the v every rank holds after the replica-mean exchange, G q = r - rho q;
    admm_sparse.cuh) driven by the two-pass phase program, through the test transport."""
    import paper_1811_05571_b200 as admm
    from paper_1811_05571_b200 import distributed as D
    M, shape, iters = 4, (256, 2048), 60
    p = admm.gen_problem(shape[0], shape[1], 8, 30.0, 31, dtype=dtype)
    h128 = p.h.astype(np.complex128)
    lam = 0.05 * float(np.max(np.abs(orc.adjoint_matvec(h128, p.g))))
    cfg = admm.SolverConfig(rho=1.0, lambda_=lam, max_iters=iters)
    opts = admm.SolveOptions(dtype=dtype, schedule="support")
    shards = [D.ShardPlan(p, cfg, "consensus", M, 1, (P, 1), (r, 0), opts) for r in range(P)]
    assert all(sh.info()["schedule"] == 5 for sh in shards)
    D.run_iterations(shards, DH.LoopbackComm(P, 1), iters)
    for sh in shards:
        sh.sync()
    v = D.gather_solution([sh.segment_v() for sh in shards], shape[1], shards[0].col_bounds)
    ref = orc.solve("consensus", h128, p.g, M=M, N=1, lam=lam, iters=iters)
    assert rel(v, ref["solution"]) <= (1e-9 if dtype == "c128" else 1e-4)
    trs = [sh.trace() for sh in shards]
    for tr in trs:
        np.testing.assert_array_equal(tr, trs[0])
    tol = 1e-8 if dtype == "c128" else 1e-3
    assert np.max(np.abs(trs[0][:, 1] - ref["trace"][:, 1]) / np.abs(ref["trace"][:, 1])) <= tol
    ob = trs[0][:iters - 1, 2]  # the two-pass program closes iteration k-1's objective in iteration k
    assert np.max(np.abs(ob - ref["trace"][:iters - 1, 2]) / np.abs(ref["trace"][:iters - 1, 2])) <= (1e-9 if dtype == "c128" else 1e-4)


def test_plan_owned_nccl_support_schedule():
    """The plan-owned NCCL driver (graph-captured phases + collectives) on the support schedule."""
    import paper_1811_05571_b200 as admm
    from paper_1811_05571_b200 import distributed as D
    p = admm.gen_problem(256, 2048, 8, 30.0, 29)
    lam = 0.05 * float(np.max(np.abs(orc.adjoint_matvec(p.h, p.g))))
    cfg = admm.SolverConfig(rho=1.0, lambda_=lam, max_iters=40)
    with D.dist_plan(p, cfg, "consensus", 4, 1, admm.SolveOptions(schedule="support")) as plan:
        assert plan.info()["schedule"] == 5
        r = plan.solve()
        r2 = plan.solve()
    np.testing.assert_array_equal(r.solution, r2.solution)
    ref = orc.solve("consensus", p.h, p.g, M=4, N=1, lam=lam, iters=40)
    assert rel(r.solution, ref["solution"]) <= 1e-9
    tr = np.stack([r.trace.primal, r.trace.dual, r.trace.objective], 1)
    assert np.max(np.abs(tr[:, 1] - ref["trace"][:, 1]) / np.abs(ref["trace"][:, 1])) <= 1e-8
    assert np.max(np.abs(tr[:, 2] - ref["trace"][:, 2]) / np.abs(ref["trace"][:, 2])) <= 1e-9
    assert abs(r.objective - ref["objective"]) <= 1e-9 * abs(ref["objective"])


CASES = [("sectioning", 1, 8, (64, 2048), 25, "c128"), ("consensus", 4, 1, (256, 2048), 40, "c128"),
         ("hybrid", 2, 4, (96, 1024), 20, "c128"), ("consensus", 8, 1, (512, 4096), 30, "c64"),
         ("reference", 1, 1, (40, 120), 30, "c128")]


@pytest.mark.parametrize("how", ["dist", "multi"])
@pytest.mark.parametrize("method,M,N,shape,iters,dtype", CASES)
def test_plan_owned_nccl_world_of_one(how, method, M, N, shape, iters, dtype):
    """The plan-owned NCCL driver with one rank (multi-process API) / one device
    (single-process API): solution, trace and objective vs the oracle, and equal to the
    single-GPU plan up to summation order."""
    import paper_1811_05571_b200 as admm
    from paper_1811_05571_b200 import distributed as D
    p = admm.gen_problem(shape[0], shape[1], 8, 30.0, 29, dtype=dtype)
    h128 = p.h.astype(np.complex128)
    lam = 0.05 * float(np.max(np.abs(orc.adjoint_matvec(h128, p.g))))
    cfg = admm.SolverConfig(rho=1.0, lambda_=1.0, max_iters=iters)
    opts = admm.SolveOptions(dtype=dtype, devices=[0] if how == "multi" else None)
    plan = D.dist_plan(p, cfg, method, M, N, opts) if how == "dist" else admm.AdmmPlan(p, cfg, method, M, N, opts)
    with plan:
        info = plan.info()
        assert info["n_ranks"] == 1 and info["grid_pr"] == 1 and info["grid_pc"] == 1
        assert abs(plan.max_abs_adjoint() * 0.05 - lam) <= 1e-12 * lam  # lambda rule through the gathered path
        plan.set_lambda(lam)
        r = plan.solve()
        r2 = plan.solve()  # repeatable (graph replays after the first capture)
    np.testing.assert_array_equal(r.solution, r2.solution)
    ref = orc.solve(method, h128, p.g, M=M, N=N, lam=lam, iters=iters)
    tol = 1e-9 if dtype == "c128" else 1e-4
    assert rel(r.solution, ref["solution"]) <= tol
    assert r.iterations_run == iters
    tr = np.stack([r.trace.primal, r.trace.dual, r.trace.objective], 1)
    assert np.max(np.abs(tr[:, 1] - ref["trace"][:, 1]) / np.abs(ref["trace"][:, 1])) <= (1e-8 if dtype == "c128" else 1e-3)
    assert np.max(np.abs(tr[:, 2] - ref["trace"][:, 2]) / np.abs(ref["trace"][:, 2])) <= (1e-9 if dtype == "c128" else 1e-4)
    assert abs(r.objective - ref["objective"]) <= (1e-9 if dtype == "c128" else 1e-4) * abs(ref["objective"])
    single = admm.AdmmPlan(p, admm.SolverConfig(rho=1.0, lambda_=lam, max_iters=iters), method, M, N,
                           admm.SolveOptions(dtype=dtype)).solve()
    assert rel(r.solution, single.solution) <= 1e-12


def test_plan_owned_nccl_early_stop_observer_and_blowup():
    """stop_now (admm_core.hpp:52-57), the observer (solvers.hpp:150-160) and
    NumericalError(last_good_iteration) (solvers.hpp:47-56) on a distributed plan."""
    import paper_1811_05571_b200 as admm
    from paper_1811_05571_b200 import distributed as D
    p = admm.gen_problem(64, 256, 4, 30.0, 7)
    lam = 0.05 * float(np.max(np.abs(orc.adjoint_matvec(p.h, p.g))))
    cfg = admm.SolverConfig(rho=1.0, lambda_=lam, max_iters=400, eps_pri=1e-6, eps_dual=1e-6)
    ref = orc.solve("consensus", p.h, p.g, M=4, lam=lam, iters=400, eps_pri=1e-6, eps_dual=1e-6)
    single = admm.consensus_solve(p, cfg, 4)
    snaps = []
    opts = admm.SolveOptions(observer=lambda s: snaps.append(s))
    with D.dist_plan(p, cfg, "consensus", 4, 1, opts) as plan:
        r = plan.solve(opts.observer)
    assert r.iterations_run == single.iterations_run == ref["iterations_run"] < 400
    assert len(snaps) == r.iterations_run and len(snaps[-1].replica_u) == 4
    assert rel(r.solution, single.solution) <= 1e-12
    np.testing.assert_allclose(snaps[-1].v, r.solution, rtol=0, atol=0)

    def boom(_s):
        raise KeyError("from the observer")
    with D.dist_plan(p, cfg, "consensus", 4, 1) as plan, pytest.raises(KeyError):
        plan.solve(boom)  # the observer's exception propagates out of the solve
    q = admm.gen_problem(6, 9, 2, float("inf"), 1008, admm.ProblemKind.RandomPhase)
    huge = admm.SensingProblem(q.h * 1e300, q.g * 1e300)
    with pytest.raises(admm.NumericalError) as ei:  # (at setup or in the loop, as the reference)
        with D.dist_plan(huge, admm.SolverConfig(lambda_=1e-3, max_iters=5), "consensus", 3, 1) as plan:
            plan.solve()
    ref = orc.solve("consensus", huge.h, huge.g, M=3, lam=1e-3, iters=5)
    assert ref["error"] == "NumericalError" and ei.value.last_good_iteration() == ref["last_good"]


def test_graph_captured_torch_nccl_iterations_match_eager():
    """torchrun with one process (NCCL through torch.distributed, the ShardPlan surface with
    the test transport): graph-captured iterations reproduce the eager ones bit-for-bit."""
    import json
    import os
    import subprocess
    import sys
    repo = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "1",
                        "--master-addr", "127.0.0.1", "--master-port", "29533",
                        os.path.join(repo, "tools", "dist_check.py")], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-4000:]
    out = json.loads(r.stdout.strip().splitlines()[-1])
    for method, res in out.items():
        assert res["eager_vs_graph_maxabs"] == 0.0, (method, res)
        assert res["iters"] == 16
    assert out["hybrid"]["vs_single_plan_rel"] <= 1e-12


def test_bench_sharded_line_schema():
    """BENCH_FORCE_DIST=1: the N > 1 code path of bench.py at N = 1 prints a line with the
    N = 1 line's keys (objective trace on, e2e, roofline, cpu_baseline)."""
    import json
    import os
    import subprocess
    import sys
    repo = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, BENCH_FORCE_DIST="1")
    r = subprocess.run([sys.executable, os.path.join(repo, "bench.py"), "--config", "1", "--steps", "16",
                        "--warmup", "3"], capture_output=True, text=True, timeout=900, env=env)
    assert r.returncode == 0, r.stderr[-3000:]
    line = json.loads(r.stdout.strip().splitlines()[-1])
    for key in ("metric", "value", "e2e", "roofline", "clocks", "gpu_launches", "nccl", "config", "run"):
        assert key in line, key
    assert line["run"]["trace_objective"] is True and line["value"] > 0
    assert set(line["config"]) == {"workload"}
