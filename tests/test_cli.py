"""tools/admmsplit_gpu: the reference's CLI surface (tools/admmsplit_main.cpp: gen :343, solve
:353-384, compare :577-665) with run_method (:296-303) on the device."""
import csv
import json
import os
import subprocess

import numpy as np
import pytest

import oracle_lib as orc

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CLI = os.path.join(REPO, "tools", "admmsplit_gpu")
REF = os.path.join(REPO, "oracle", "_ref", "admmsplit_ref")


def build():
    subprocess.run(["make", "-C", os.path.join(REPO, "tools"), "admmsplit_gpu"], check=True, capture_output=True)


def run(*args):
    return subprocess.run([CLI, *args], capture_output=True, text=True, timeout=600)


def test_cli_builds_and_generates_the_reference_problem_files(tmp_path):
    build()
    d = tmp_path / "p"
    r = run("gen", "--nm", "48", "--np", "160", "--k", "5", "--snr", "30", "--seed", "11", "--out", str(d))
    assert r.returncode == 0 and r.stdout.startswith(f"wrote {d}: H 48x160, k=5, kind=complex-gaussian, seed=11")
    man = json.load(open(d / "manifest.json"))
    assert list(man) == sorted(man) and man["schema_version"] == "1" and man["snr_db"] == 30.0
    h, g, t, sigma = orc.gen_problem(48, 160, 5, 30.0, 11)
    assert man["noise_sigma"] == sigma
    if os.path.exists(REF):  # byte-identical to the files the unmodified reference writes
        subprocess.run([REF, "gen", f"out={tmp_path / 'r'}", "m=48", "n=160", "k=5", "snr=30", "seed=11", "kind=cg"],
                       check=True, capture_output=True)
        for ours, theirs in (("H.cmat", "h.cmat"), ("g.cmat", "g.cmat"), ("truth.cmat", "truth.cmat")):
            assert open(d / ours, "rb").read() == open(tmp_path / "r" / theirs, "rb").read()


def test_cli_usage_and_validation_errors(tmp_path):
    build()
    assert run("solve", "--bogus").returncode == 2
    assert run().returncode == 2
    d = tmp_path / "p"
    assert run("gen", "--nm", "16", "--np", "32", "--k", "2", "--seed", "1", "--out", str(d)).returncode == 0
    assert json.load(open(d / "manifest.json"))["snr_db"] == "inf"
    out = str(tmp_path / "o")
    r = run("solve", "--method", "consensus", "--m", "4", "--n", "2", "--problem", str(d), "--out", out)
    assert r.returncode == 2 and "consensus takes --m only" in r.stderr
    r = run("solve", "--method", "hybrid", "--m", "2", "--problem", str(d), "--out", out)
    assert r.returncode == 2 and "hybrid takes both --m and --n" in r.stderr
    r = run("solve", "--method", "reference", "--problem", str(d), "--nm", "4", "--out", out)
    assert r.returncode == 2 and "not both" in r.stderr
    r = run("solve", "--method", "reference", "--nm", "8", "--np", "16", "--k", "2", "--out", out)
    assert r.returncode == 2 and "--seed is mandatory" in r.stderr
    r = run("solve", "--method", "reference", "--problem", str(d), "--rho", "-1", "--out", out)
    assert r.returncode == 2 and "rho must be positive" in r.stderr
    r = run("solve", "--method", "reference", "--problem", str(d), "--device", "cpu", "--out", out)
    assert r.returncode == 2 and "no CPU path" in r.stderr


def test_cli_reference_cases_without_a_device(tmp_path):
    """tests/test_cli.cpp:63-84, 105-117 restated: the cases that end before the device is needed."""
    build()
    d = tmp_path / "gen"
    r = run("gen", "--nm", "12", "--np", "30", "--k", "4", "--snr", "30", "--seed", "7", "--kind", "random-phase",
            "--out", str(d))
    assert r.returncode == 0, r.stderr
    for name in ("H.cmat", "g.cmat", "truth.cmat", "manifest.json"):
        assert (d / name).exists()
    import paper_1811_05571_b200 as admm
    h = admm.read_cmat(d / "H.cmat")
    assert h.shape == (12, 30) and np.allclose(np.abs(h), np.abs(h[0, 0]))  # random-phase: constant modulus
    bad = str(tmp_path / "gen_bad")
    assert run("gen", "--nm", "12", "--np", "30", "--k", "4", "--out", bad).returncode == 2      # no seed
    assert run("gen", "--nm", "12", "--np", "200", "--k", "300", "--seed", "1", "--out", bad).returncode == 2
    base = ["--nm", "12", "--np", "36", "--k", "3", "--seed", "5", "--out", str(tmp_path / "solve_bad")]
    assert run("solve", "--method", "consensus", *base).returncode == 2                 # missing --m
    assert run("solve", "--method", "sectioning", "--m", "3", *base).returncode == 2    # wrong division
    assert run("solve", "--method", "hybrid", "--m", "3", *base).returncode == 2        # missing --n
    assert run("solve", "--method", "reference", "--m", "2", *base).returncode == 2
    r = run("solve", "--method", "consensus", "--m", "5", *base)                        # non-divisible, no --ragged
    assert r.returncode == 2 and "error:" in r.stderr
    assert run("solve", "--method", "reference", "--problem", "/tmp/nowhere", *base).returncode == 2


@pytest.mark.gpu
def test_cli_reference_cases_on_device(tmp_path):
    """tests/test_cli.cpp:86-103, 119-165, 207-234 restated against tools/admmsplit_gpu."""
    build()
    d = tmp_path / "solve_ref"
    r = run("solve", "--method", "reference", "--nm", "12", "--np", "36", "--k", "3", "--seed", "5", "--rho", "1",
            "--lambda", "0.01", "--iters", "7", "--out", str(d))
    assert r.returncode == 0, r.stderr
    trace = open(d / "trace.csv").read()
    assert trace.count("\n") == 8 and trace.startswith("iteration,primal_norm,dual_norm,objective")
    met = open(d / "metrics.json").read()
    assert '"schema_version"' in met and '"nmse"' in met and (d / "solution.cmat").exists()
    assert open(d / "ledger.csv").read().count("\n") == 1  # single node: header only
    # hybrid ledger = closed form: 4 * (12 / 3) + 2 * (36 / 4) = 34 per node and iteration
    d = tmp_path / "solve_hybrid"
    r = run("solve", "--method", "hybrid", "--m", "3", "--n", "4", "--nm", "12", "--np", "36", "--k", "3", "--seed", "5",
            "--rho", "1", "--lambda", "0.01", "--iters", "3", "--out", str(d))
    assert r.returncode == 0, r.stderr
    rows = list(csv.reader(open(d / "ledger.csv")))[1:]
    assert len(rows) == 12 * 3
    for node, it, rec, sent, conv in rows:
        assert int(rec) + int(sent) == 34 and conv == "sender_once_broadcast"
    # byte-deterministic across runs and --threads values
    outs = []
    for k, threads in enumerate(("1", "2")):
        dk = tmp_path / f"det{k}"
        r = run("solve", "--method", "hybrid", "--m", "2", "--n", "3", "--nm", "12", "--np", "36", "--k", "3", "--seed",
                "11", "--rho", "1", "--lambda", "0.02", "--iters", "5", "--fingerprint", "--threads", threads, "--out",
                str(dk))
        assert r.returncode == 0, r.stderr
        outs.append((dk, r.stdout[r.stdout.index("fingerprint "):][:28]))
    for name in ("solution.cmat", "trace.csv", "ledger.csv", "metrics.json"):
        assert open(outs[0][0] / name, "rb").read() == open(outs[1][0] / name, "rb").read()
    assert outs[0][1] == outs[1][1]
    # compare: one entry per method spec; a single method is allowed
    out = tmp_path / "compare.json"
    r = run("compare", "--methods", "reference,consensus:3,sectioning:4,hybrid:3x4", "--nm", "12", "--np", "36", "--k",
            "3", "--seed", "5", "--rho", "1", "--lambda", "0.01", "--iters", "20", "--out", str(out))
    assert r.returncode == 0, r.stderr
    c = json.load(open(out))
    assert c["schema_version"] == "1" and len(c["entries"]) == 4 and "winners" in c
    assert run("compare", "--methods", "reference", "--nm", "12", "--np", "36", "--k", "3", "--seed", "5", "--iters", "5",
               "--rho", "1", "--out", str(tmp_path / "single.json")).returncode == 0
    # numerical blow-up: exit code 3 with the last good iteration
    r = run("solve", "--method", "consensus", "--m", "2", "--nm", "12", "--np", "36", "--k", "3", "--seed", "5", "--rho",
            "1", "--lambda", "0.01", "--scl", "1e300", "--iters", "3", "--out", str(tmp_path / "blowup"))
    assert r.returncode == 3 and "last good iteration" in r.stderr


@pytest.mark.gpu
def test_cli_solve_writes_the_reference_report_files(tmp_path):
    import paper_1811_05571_b200 as admm
    build()
    d, out = tmp_path / "p", tmp_path / "o"
    assert run("gen", "--nm", "64", "--np", "256", "--k", "6", "--snr", "30", "--seed", "7", "--out", str(d)).returncode == 0
    r = run("solve", "--method", "hybrid", "--m", "2", "--n", "2", "--problem", str(d), "--rho", "1", "--lambda", "0.05",
            "--iters", "40", "--out", str(out), "--fingerprint")
    assert r.returncode == 0, r.stderr
    assert r.stdout.startswith("method=hybrid iterations=40 objective=") and "fingerprint " in r.stdout
    h, g, t, _ = orc.gen_problem(64, 256, 6, 30.0, 7)
    ref = orc.solve("hybrid", h, g, M=2, N=2, lam=0.05, iters=40)
    sol = admm.read_cvec(out / "solution.cmat")
    assert np.linalg.norm(sol - ref["solution"]) <= 1e-9 * np.linalg.norm(ref["solution"])
    rows = list(csv.reader(open(out / "trace.csv")))
    assert rows[0] == ["iteration", "primal_norm", "dual_norm", "objective"] and len(rows) == 41
    tr = np.array(rows[1:], dtype=float)
    np.testing.assert_allclose(tr[:, 1:], ref["trace"], rtol=1e-8)
    led = list(csv.reader(open(out / "ledger.csv")))
    assert led[0] == ["node_id", "iteration", "received", "sent", "convention"] and len(led) == 1 + 4 * 40
    want = admm.CommLedger.for_solve("hybrid", [0, 32, 64], [0, 128, 256], 40).as_array()
    for node, it, rec, sent, conv in led[1:]:
        assert conv == "sender_once_broadcast"
        assert (int(rec), int(sent)) == tuple(want[int(node), int(it) - 1, :2])
    met = json.load(open(out / "metrics.json"))
    assert list(met) == sorted(met) and met["iterations_run"] == 40 and met["schema_version"] == "1"
    assert abs(met["objective"] - ref["objective"]) <= 1e-9 * abs(ref["objective"])
    m = admm.recovery_metrics(ref["solution"], t)
    assert abs(met["nmse"] - m.nmse) <= 1e-6 * m.nmse and met["support_recall"] == m.support_recall


@pytest.mark.gpu
def test_cli_compare_and_numerical_exit_code(tmp_path):
    build()
    out = tmp_path / "c.json"
    r = run("compare", "--methods", "reference,consensus:4,sectioning:2,hybrid:2x2", "--nm", "64", "--np", "256", "--k",
            "6", "--snr", "30", "--seed", "7", "--rho", "1", "--lambda", "0.05", "--iters", "30", "--out", str(out),
            "--fingerprint")
    assert r.returncode == 0, r.stderr
    c = json.load(open(out))
    assert [e["label"] for e in c["entries"]] == ["reference", "consensus:4", "sectioning:2", "hybrid:2x2"]
    assert c["entries"][0]["per_node_elements"] is None and c["entries"][1]["per_node_elements"] == 512
    assert c["entries"][3]["per_node_elements"] == 2 * 32 + 2 * 128
    assert c["winners"]["communication"] == "sectioning:2" and c["problem"] == {"nm": 64, "np": 256}
    h, g, t, _ = orc.gen_problem(64, 256, 6, 30.0, 7)
    for e, (meth, M, N) in zip(c["entries"], (("reference", 1, 1), ("consensus", 4, 1), ("sectioning", 1, 2),
                                              ("hybrid", 2, 2))):
        ref = orc.solve(meth, h, g, M=M, N=N, lam=0.05, iters=30)
        assert abs(e["objective"] - ref["objective"]) <= 1e-9 * abs(ref["objective"])
    # NumericalError -> exit code 3 with the last good iteration (admmsplit_main.cpp:745-748)
    r = run("solve", "--method", "sectioning", "--n", "8", "--nm", "32", "--np", "256", "--k", "4", "--seed", "3",
            "--rho", "1", "--lambda", "1e-3", "--iters", "4000", "--out", str(tmp_path / "x"))
    if r.returncode != 0:  # this Jacobi split diverges to overflow at rho = 1
        assert r.returncode == 3 and "last good iteration" in r.stderr
