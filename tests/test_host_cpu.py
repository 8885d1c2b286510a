"""CPU tests: the C ABI library loads and exports every declared symbol; the product's
input generator reproduces the reference bit-for-bit; host-side partition / ledger /
closed-form logic matches the reference (tests/test_partition.cpp, tests/test_comm.cpp,
tests/test_solvers.cpp:95-132)."""
import ctypes
import os
import re

import numpy as np
import pytest

import golden_cases as gc
import oracle_lib as orc

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    src = open(os.path.join(REPO, "include", "admm_b200.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(admm_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    lib = ctypes.CDLL(os.path.join(REPO, "paper_1811_05571_b200", "libadmm_b200.so"))
    syms = declared_symbols()
    assert len(syms) >= 20
    for s in syms:
        assert hasattr(lib, s), s
    assert lib.admm_abi_version() == 3


def test_python_binding_covers_the_header():
    from paper_1811_05571_b200 import _lib
    assert set(declared_symbols()) == set(_lib.EXPORTED)


def test_no_device_means_loud_failure_not_fallback():
    import torch
    if torch.cuda.is_available():
        pytest.skip("device present")
    import paper_1811_05571_b200 as admm
    with pytest.raises(admm.DeviceError):
        admm.matvec(np.eye(2), np.ones(2))
    p = admm.gen_problem(8, 16, 2, 30.0, 1)
    with pytest.raises(admm.DeviceError):
        admm.consensus_solve(p, admm.SolverConfig(lambda_=0.1), 2)


@pytest.mark.parametrize("name", gc.gen_cases())
def test_product_generator_matches_reference_bits(name):
    import paper_1811_05571_b200 as admm
    entry, _ = gc.load(name)
    m, n, k, snr, seed, kind = entry["problem"]
    p = admm.gen_problem(m, n, k, float(snr), seed,
                         admm.ProblemKind.ComplexGaussian if kind == "cg" else admm.ProblemKind.RandomPhase)
    assert f"{orc.fnv1a64(p.h, p.g, p.truth):016x}" == entry["fnv"]
    assert p.noise_sigma == entry["noise_sigma"]


def test_c64_generator_is_rounded_c128():
    import paper_1811_05571_b200 as admm
    a = admm.gen_problem(64, 300, 7, 30.0, 11)
    b = admm.gen_problem(64, 300, 7, 30.0, 11, dtype="c64")
    assert b.h.dtype == np.complex64
    np.testing.assert_array_equal(b.h, a.h.astype(np.complex64))
    np.testing.assert_array_equal(b.g, a.g)


def test_partition_rules_match_reference():
    import paper_1811_05571_b200 as admm
    s = admm.make_partition(2160, 22500, 4, 3)  # test_partition.cpp:21-27
    assert [s.row_size(i) for i in range(4)] == [540] * 4
    assert [s.col_size(j) for j in range(3)] == [7500] * 3
    s = admm.make_partition(10, 6, 4, 1, True)  # ragged leading-blocks rule
    assert [s.row_size(i) for i in range(4)] == [3, 3, 2, 2]
    for args in [(10, 6, 4, 1, False), (10, 6, 1, 4, False), (10, 6, 0, 1), (10, 6, 11, 1)]:
        with pytest.raises(admm.PartitionError):
            admm.make_partition(*args)


def test_closed_form_counts_match_reference():
    import paper_1811_05571_b200 as admm
    M = admm.Method
    assert admm.per_node_elements(M.Consensus, 22500, 2160, 4, 3) == 45000  # test_comm.cpp:10-15
    assert admm.per_node_elements(M.Sectioning, 22500, 2160, 4, 3) == 6480
    assert admm.per_node_elements(M.Hybrid, 22500, 2160, 4, 3) == 16620
    assert round(admm.reduction_vs_consensus(M.Sectioning, 22500, 2160, 4, 3), 1) == 85.6
    assert round(admm.reduction_vs_consensus(M.Hybrid, 22500, 2160, 4, 3), 1) == 63.1
    with pytest.raises(admm.PartitionError):
        admm.per_node_elements(M.Hybrid, 22500, 2160, 7, 3)
    with pytest.raises(admm.ParameterError):
        admm.per_node_elements(M.Consensus, 0, 1, 1, 1)


@pytest.mark.parametrize("name", [n for n in gc.solve_cases() if n.startswith(("ledger_", "lattice_"))])
def test_host_ledger_equals_reference_ledger(name):
    """The ledger a B200 solve reports is the reference's, cell for cell."""
    import paper_1811_05571_b200 as admm
    entry, ref = gc.load(name)
    if "ledger" not in ref:
        pytest.skip("error case")
    a = gc.solver_args(entry)
    m, n = entry["problem"][0], entry["problem"][1]
    spec = admm.make_partition(m, n, a["M"] if a["method"] in ("consensus", "hybrid") else 1,
                               a["N"] if a["method"] in ("sectioning", "hybrid") else 1, a["ragged"])
    led = admm.CommLedger.for_solve(a["method"], spec.row_bounds, spec.col_bounds,
                                    entry["iterations_run"])
    want = ref["ledger"]
    if a["method"] == "reference":
        assert led.empty() and want.size == 0
        return
    np.testing.assert_array_equal(led.as_array(), want)
    # ... and equals the closed form every iteration (test_solvers.cpp:95-119)
    meth = {"consensus": admm.Method.Consensus, "sectioning": admm.Method.Sectioning,
            "hybrid": admm.Method.Hybrid}[a["method"]]
    closed = admm.per_node_elements(meth, n, m, spec.M, spec.N)
    for node in range(led.node_count()):
        for k in range(led.iteration_count()):
            assert led.counts(node, k).total() == closed


def test_per_link_convention():
    import paper_1811_05571_b200 as admm
    led = admm.CommLedger()  # test_comm.cpp:83-107
    led.record_recv(0, 0, 100)
    led.record_send(0, 0, 40)
    led.record_broadcast(0, 0, 7, 3)
    led.record_broadcast(1, 0, 7, 0)
    assert led.counts(0, 0).total() == 147
    assert led.counts(0, 0, admm.Convention.PerLink).sent == 61
    assert led.counts(1, 0).sent == 7 and led.counts(1, 0, admm.Convention.PerLink).sent == 0
    assert led.counts(5, 9).total() == 0 and led.node_count() == 2 and led.iteration_count() == 1


def test_config_validation_matches_reference():
    import paper_1811_05571_b200 as admm
    for kw in [dict(rho=0.0), dict(lambda_=-1.0), dict(max_iters=0), dict(eps_pri=-1e-3), dict(scl=0.0)]:
        with pytest.raises(admm.ParameterError):
            admm.SolverConfig(**kw).validate()
