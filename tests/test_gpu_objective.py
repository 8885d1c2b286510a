"""GPU: the per-iteration objective trace (objective_value, admm_core.hpp:60-64, pushed
every iteration at solvers.hpp:146/267/431) computed by the H-pass-free recurrence
(objective_rec_kernel) against (a) the extra-H-pass path
(ADMM_B200_OBJ=pass, the reference's own evaluation) and (b) the C oracle's trace.
Tolerance: 1e-9 relative per entry on converging runs (FP64 rounding of the recurrence,
which accumulates over the iterations), checked on both schedules and c128/c64."""
import numpy as np
import pytest

import oracle_lib as orc

pytestmark = pytest.mark.gpu

CASES = [("consensus", 4, 1), ("sectioning", 1, 4), ("hybrid", 2, 2), ("reference", 1, 1)]


def solve(p, method, M, N, lam, iters, dtype, schedule):
    import paper_1811_05571_b200 as admm
    cfg = admm.SolverConfig(rho=1.0, lambda_=lam, max_iters=iters)
    opts = admm.SolveOptions(dtype=dtype, schedule=schedule, trace_objective=True)
    with admm.AdmmPlan(p, cfg, method, M, N, opts) as plan:
        return plan.solve()


@pytest.mark.parametrize("schedule", ["auto", "twopass", "resident"])
@pytest.mark.parametrize("method,M,N", CASES)
def test_objective_recurrence_matches_pass_and_oracle(method, M, N, schedule, monkeypatch):
    import paper_1811_05571_b200 as admm
    p = admm.gen_problem(96, 512, 8, 30.0, 21)
    lam = 0.05 * float(np.max(np.abs(orc.adjoint_matvec(p.h, p.g))))
    iters = 150
    rec = solve(p, method, M, N, lam, iters, "c128", schedule)
    monkeypatch.setenv("ADMM_B200_OBJ", "pass")
    ps = solve(p, method, M, N, lam, iters, "c128", "auto" if schedule == "resident" else schedule)
    ref = orc.solve(method if method != "reference" else "reference", p.h, p.g, M=M, N=N, lam=lam, iters=iters)
    assert ref["error"] == "none"
    o_rec, o_pass, o_ref = rec.trace.objective, ps.trace.objective, ref["trace"][:, 2]
    assert np.all(np.isfinite(o_rec))
    np.testing.assert_allclose(o_pass, o_ref, rtol=1e-10)
    np.testing.assert_allclose(o_rec, o_ref, rtol=1e-9)
    # SolveReport.objective: one exact pass either way (ADMM_B200_OBJ=pass also moves small
    # problems off the resident schedule, so the iterates may differ in the last bit)
    assert abs(rec.objective - ps.objective) <= 1e-13 * abs(ps.objective)


def test_objective_recurrence_c64_and_ragged():
    import paper_1811_05571_b200 as admm
    p = admm.gen_problem(90, 500, 8, 30.0, 22)
    lam = 0.05 * float(np.max(np.abs(orc.adjoint_matvec(p.h, p.g))))
    cfg = admm.SolverConfig(rho=1.0, lambda_=lam, max_iters=120)
    r = admm.hybrid_solve(p, cfg, 4, 3, admm.SolveOptions(dtype="c128", ragged=True, trace_objective=True))
    ref = orc.solve("hybrid", p.h, p.g, M=4, N=3, lam=lam, iters=120, ragged=True)
    np.testing.assert_allclose(r.trace.objective, ref["trace"][:, 2], rtol=1e-9)
    h64 = p.h.astype(np.complex64)
    p64 = admm.SensingProblem(h64, p.g)
    r64 = admm.consensus_solve(p64, cfg, 3, admm.SolveOptions(dtype="c64", trace_objective=True))
    ref64 = orc.solve("consensus", h64.astype(np.complex128), p.g, M=3, N=1, lam=lam, iters=120)
    np.testing.assert_allclose(r64.trace.objective, ref64["trace"][:, 2], rtol=1e-6)
