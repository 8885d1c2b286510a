"""CPU: pin the C restatement (oracle/liboracle.so) BIT-FOR-BIT to the unmodified reference.

The fixtures in tests/golden/ were produced by oracle/_ref (the reference library compiled
where it lies under /root/reference) via tests/golden/make_golden.py.  Every case restates a
reference Catch2 test or a BASELINE config; the oracle must reproduce the reference's
solution, residual trace, iteration count and error class exactly.
"""
import numpy as np
import pytest

import golden_cases as gc
import oracle_lib as orc


@pytest.mark.parametrize("name", gc.gen_cases())
def test_generator_hash_matches_reference(name):
    entry, _ = gc.load(name)
    m, n, k, snr, seed, kind = entry["problem"]
    h, g, t, ns = orc.gen_problem(m, n, k, snr, seed, kind)
    assert f"{orc.fnv1a64(h, g, t):016x}" == entry["fnv"]
    assert ns == entry["noise_sigma"]


@pytest.mark.parametrize("name", [c for c in gc.solve_cases() if not c.startswith("cfg2_")])
def test_oracle_bit_exact_vs_reference(name):
    entry, ref = gc.load(name)
    h, g, _ = gc.problem(entry, orc.gen_problem)
    if entry.get("prescale") is None:
        m, n, k, snr, seed, kind = entry["problem"]
        assert f"{orc.fnv1a64(*orc.gen_problem(m, n, k, snr, seed, kind)[:3]):016x}" == entry["fnv"]
    args = gc.solver_args(entry)
    out = orc.solve(h=h, g=g, snapshots="snapshots" in ref, **args)
    assert out["error"] == entry["error"]
    if entry["error"] != "none":
        assert out["last_good"] == entry["last_good"]
        return
    assert out["iterations_run"] == entry["iterations_run"]
    # bit-for-bit (same operation order, same libm, no FP contraction)
    np.testing.assert_array_equal(out["solution"], ref["solution"])
    np.testing.assert_array_equal(out["trace"], ref["trace"])
    if "snapshots" in ref:
        np.testing.assert_array_equal(out["snapshots"], ref["snapshots"])
    assert out["objective"] == entry["objective"]


def test_reference_known_answers_on_oracle():
    # prox KATs, tests/test_prox.cpp:8-20,42-54
    out = orc.soft_threshold_vec(np.array([5, -1, 2, -5, 3 + 4j]), 2.0)
    assert out[0] == 3 and out[1] == 0 and out[2] == 0 and out[3] == -3
    assert abs(out[4] - (1.8 + 2.4j)) < 1e-15
    # matvec KATs, tests/test_linalg.cpp:21-53
    a = np.array([[1, 1j], [0, 2]])
    assert np.array_equal(orc.matvec(a, np.array([1, 1])), np.array([1 + 1j, 2]))
    assert orc.adjoint_matvec(np.array([[1j]]), np.array([1]))[0] == -1j
    # gram KATs, tests/test_linalg.cpp:88-98
    x = orc.gram_solve(np.zeros((2, 2)), 2.0, np.array([4, 6]))
    assert np.allclose(x, [2, 3], atol=1e-12)
    x = orc.gram_solve(np.eye(2), 1.0, np.array([4, 4]))
    assert np.allclose(x, [2, 2], atol=1e-12)


def test_oracle_gram_vs_dense_solve():
    # tests/test_linalg.cpp:112-134: Woodbury vs dense oracle and vs Direct
    h = orc.random_gauss(40, 7).reshape(4, 10)
    rhs = orc.random_gauss(10, 8)
    got = orc.gram_solve(h, 0.5, rhs)
    want = np.linalg.solve(h.conj().T @ h + 0.5 * np.eye(10), rhs)
    assert np.linalg.norm(got - want) / np.linalg.norm(want) <= 1e-8
    direct = orc.gram_solve(h, 0.5, rhs, strategy=0)
    assert np.linalg.norm(got - direct) / np.linalg.norm(direct) <= 1e-8


def test_oracle_partition_rules():
    b = np.zeros(5, np.uint64)
    assert orc.lib().orc_split_bounds(10, 4, 1, orc._p(b)) == 0
    assert list(np.diff(b)) == [3, 3, 2, 2]  # ragged leading-blocks rule, partition.hpp:47-50
    assert orc.lib().orc_split_bounds(10, 4, 0, orc._p(b)) == 5  # PartitionError
    assert orc.lib().orc_split_bounds(10, 0, 0, orc._p(b)) == 5
    assert orc.lib().orc_split_bounds(10, 11, 0, orc._p(b)) == 5
