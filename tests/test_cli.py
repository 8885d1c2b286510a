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
