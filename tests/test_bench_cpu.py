"""CPU: bench.py's launcher logic and the reference arm's line (no GPU, no import of the package).

* `--gpus N > 1` outside torchrun re-launches under torch.distributed.run with one process per GPU
  on 127.0.0.1; inside torchrun WORLD_SIZE must equal --gpus.
* the reference arm runs on rank 0 only, prints the contract's keys, and describes the same `config`
  as the product arm.
"""
import json
import os
import subprocess
import sys

import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
import bench  # noqa: E402

REF = os.path.join(REPO, "oracle", "_ref", "admmsplit_ref")


def test_relaunch_command(monkeypatch):
    seen = {}
    monkeypatch.setattr(bench.subprocess, "call", lambda cmd: seen.setdefault("cmd", cmd) and 0)
    monkeypatch.setattr(sys, "argv", ["bench.py", "--gpus", "4", "--steps", "7", "--warmup", "3"])
    args = bench.parse_args(sys.argv[1:])
    assert bench.relaunch_under_torchrun(args) == 0
    cmd = seen["cmd"]
    assert cmd[:3] == [sys.executable, "-m", "torch.distributed.run"]
    assert "--nnodes=1" in cmd and "--nproc-per-node=4" in cmd and "--master-addr=127.0.0.1" in cmd
    assert any(c.startswith("--master-port=") and int(c.split("=")[1]) > 0 for c in cmd)
    i = cmd.index(os.path.join(REPO, "bench.py"))
    assert cmd[i + 1:] == ["--gpus", "4", "--steps", "7", "--warmup", "3"]  # the caller's arguments, unchanged


def test_world_size_must_match_gpus():
    env = dict(os.environ, WORLD_SIZE="2", RANK="0", LOCAL_RANK="0")
    r = subprocess.run([sys.executable, os.path.join(REPO, "bench.py"), "--gpus", "4", "--impl", "reference"],
                       capture_output=True, text=True, env=env)
    assert r.returncode != 0 and "WORLD_SIZE=2 but --gpus 4" in r.stderr


def test_defaults_and_config_dicts():
    a = bench.parse_args([])
    assert (a.gpus, a.impl, a.config) == (1, "ours", "4") and a.warmup >= 3 and a.trace_objective
    for name in bench.CONFIGS:  # one `config` object for both arms, naming the BASELINE workload
        d = bench.config_dict(name)
        assert list(d) == ["workload"] and d["workload"].startswith(f"config {name}: ")
    s = bench.reference_sample("4")  # the bounded sample of the headline config and its scale
    assert (s["rows"], s["cols"], s["M"], s["full_rows"]) == (256, 262144, 8, 16384) and s["scale"] == 256 / 16384


@pytest.mark.skipif(not os.path.exists(REF), reason="oracle/_ref not built")
def test_reference_arm_line_and_rank_gating():
    base = [sys.executable, os.path.join(REPO, "bench.py"), "--impl", "reference", "--config", "1", "--steps", "4",
            "--warmup", "3"]
    r = subprocess.run(base, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr
    line = json.loads(r.stdout.strip().splitlines()[-1])
    assert line["impl"] == "reference" and line["metric"] == "ADMM iterations/s" and line["unit"] == "iterations/s"
    assert line["config"] == bench.config_dict("1") and line["higher_is_better"] is True
    assert line["steps"] == 4 and line["warmup"] == 3 and line["n_gpus"] == 1
    assert line["value"] > 0 and line["sample_scale"] == 1.0
    assert abs(line["ms_per_step"] * line["value"] / 1000.0 - 1.0) < 1e-9  # full workload: value = 1 / step time
    cb = line["cpu_baseline"]
    assert cb["kind"] == "reference" and cb["cores"] >= 1 and cb["value"] == line["value"] and cb["sample"]
    assert line["e2e"] == {"value": line["value"], "unit": "iterations/s", "h2d_bytes_per_step": 0,
                           "d2h_bytes_per_step": 0}
    # under torchrun only rank 0 runs and prints; the other ranks exit 0 without work
    env = dict(os.environ, WORLD_SIZE="2", RANK="1", LOCAL_RANK="1")
    r1 = subprocess.run(base[:2] + ["--gpus", "2"] + base[2:], capture_output=True, text=True, env=env, timeout=60)
    assert r1.returncode == 0 and r1.stdout.strip() == ""
