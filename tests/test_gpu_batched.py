"""GPU: batched multi-scene plans (BASELINE config 5).  Each scene of a batched plan is
an independent reference solve: it must match a single-scene plan on that scene and the
oracle (c64-rounded H promoted), with per-scene lambda_b = 0.03 max|H^H g_b|."""
import numpy as np
import pytest

import oracle_lib as orc

pytestmark = pytest.mark.gpu


def rel(a, b):
    s = float(np.max(np.abs(b)))
    return float(np.linalg.norm(a / s - b / s) / np.linalg.norm(b / s))


def support(v):
    return np.abs(v) > 1e-3 * np.max(np.abs(v))


@pytest.mark.parametrize("dtype,B,split", [("c64", 8, None), ("c128", 5, None), ("c64", 64, None),
                                            ("c64", 8, "3,2,3"), ("c128", 3, "2,3,4")])
def test_batched_scenes_match_independent_solves(dtype, B, split, monkeypatch):
    """split: forced split-K counts "N,K,H" of the three skinny GEMMs (the automatic
    choice follows the wave count and is 1 at this size)."""
    import paper_1811_05571_b200 as admm
    if split:
        monkeypatch.setenv("ADMM_B200_BSPLIT", split)
    h = admm.cra_matrix(seed=5, dtype=dtype, n_tx=6, n_freq=32, grid=16)  # 192 x 4096
    g, truth = admm.cra_scenes(h, B, seed=5, lo=20, hi=60, grid=16)
    iters = 60
    p = admm.SensingProblem(h, g)
    cfg = admm.SolverConfig(rho=1.0, lambda_=1.0, max_iters=iters)
    opts = admm.SolveOptions(dtype=dtype, trace_objective=False)
    with admm.AdmmPlan(p, cfg, "hybrid", 2, 4, opts) as plan:
        assert plan.batch == B
        lams = 0.03 * plan.max_abs_adjoint_batched()
        h128 = h.astype(np.complex128)
        want = 0.03 * np.max(np.abs(h128.conj().T @ g), axis=0)
        np.testing.assert_allclose(lams, want, rtol=1e-12)
        plan.set_lambdas(lams)
        rep = plan.solve()
    assert rep.solution.shape == (h.shape[1], B) and rep.iterations_run == iters
    for b in ([0, B // 2, B - 1] if B > 8 else range(B)):
        single = admm.SensingProblem(h, g[:, b].copy())
        cfg1 = admm.SolverConfig(rho=1.0, lambda_=float(lams[b]), max_iters=iters)
        r1 = admm.hybrid_solve(single, cfg1, 2, 4, admm.SolveOptions(dtype=dtype, trace_objective=False))
        assert rel(rep.solution[:, b], r1.solution) <= 1e-12
        np.testing.assert_allclose(rep.trace.dual[:, b], r1.trace.dual, rtol=1e-10)
        ref = orc.solve("hybrid", h128, g[:, b], M=2, N=4, lam=float(lams[b]), iters=iters)
        err = rel(rep.solution[:, b], ref["solution"])
        assert err <= 1e-4 and np.array_equal(support(rep.solution[:, b]), support(ref["solution"]))


@pytest.mark.parametrize("dtype", ["c128", "c64"])
def test_batched_objective_trace(dtype):
    """Per-scene objective trace of a batched plan (the recurrence of the single-scene
    engine, per scene; the last entry from one extra w = H c) against the oracle."""
    import paper_1811_05571_b200 as admm
    h = admm.cra_matrix(seed=6, dtype=dtype, n_tx=6, n_freq=32, grid=16)  # 192 x 4096
    B = 6
    g, _ = admm.cra_scenes(h, B, seed=6, lo=20, hi=60, grid=16)
    iters = 40
    p = admm.SensingProblem(h, g)
    cfg = admm.SolverConfig(rho=1.0, lambda_=1.0, max_iters=iters)
    with admm.AdmmPlan(p, cfg, "hybrid", 2, 4, admm.SolveOptions(dtype=dtype, trace_objective=True)) as plan:
        lams = 0.03 * plan.max_abs_adjoint_batched()
        plan.set_lambdas(lams)
        rep = plan.solve()
    h128 = h.astype(np.complex128)
    for b in range(B):
        ref = orc.solve("hybrid", h128, g[:, b], M=2, N=4, lam=float(lams[b]), iters=iters)
        want = ref["trace"][:, 2]
        assert np.all(np.isfinite(rep.trace.objective[:, b]))
        np.testing.assert_allclose(rep.trace.objective[:, b], want, rtol=1e-9 if dtype == "c128" else 1e-5)
