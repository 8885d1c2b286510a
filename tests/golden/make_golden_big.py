#!/usr/bin/env python3
"""Full-size BASELINE fixtures from the UNMODIFIED reference (oracle/_ref/admmsplit_ref).

Run in the build container (needs /root/reference for oracle/_ref; ~70 min on 8 cores):
    python tests/golden/make_golden_big.py [cfg2] [cfg3] [cfg4] [cfg5]

Writes tests/golden/big/<name>.npz + tests/golden/big/index.json.  These are the
north star's "oracle-matching solutions on all five configs" pins, consumed by
tests/test_gpu_full_configs.py:

  cfg2_sectioning8_it300  config 2 exactly: gen_problem(1024, 32768, 64, 30 dB, seed 2),
                          sectioning N=8, rho=1, lambda=0.05 max|H^H g|, 300 iterations.
  cfg3_hybrid24_it500     config 3 exactly: the CRA-like H (3072 x 32768, seed 3) rounded
                          to complex64 and promoted to c128 for the reference, one 300-voxel
                          scene; hybrid 2x4, lambda=0.03 max|H^H g|, 500 iterations.
  cfg4_rows256_it1000     config 4 at full width: gen_problem(256, 262144, 1000, 30 dB,
                          seed 4) -- the first 256 rows of config 4's H-stream (same
                          row-major draws; CN(0,1/256) instead of CN(0,1/16384)) -- rounded
                          to complex64, consensus M=8, lambda=0.05 max|H^H g|, 1000 iterations.
  cfg5_scene{0,1}_it500   config 5: scenes 0 and 1 of the 64-scene batch on the config-3 H,
                          each a reference hybrid_solve (the reference has no batched API).

Inputs the GPU side regenerates bit-exactly are pinned by FNV-1a hashes (the product's
generators, admm_gen_problem / admm_gen_cra); measurement vectors built with numpy
matmuls (BLAS results may differ across CPUs) are stored in the fixture instead.
"""
from __future__ import annotations

import json
import os
import shutil
import subprocess
import sys
import tempfile
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, REPO)
sys.path.insert(0, os.path.dirname(HERE))
from make_golden import meta, read_cmat, solve, write_cmat  # noqa: E402

BIG = os.path.join(HERE, "big")
REF = os.path.join(REPO, "oracle", "_ref", "admmsplit_ref")
THREADS = str(os.cpu_count() or 8)


def fnv(*arrays) -> str:
    import oracle_lib as orc
    return f"{orc.fnv1a64(*[np.ascontiguousarray(a) for a in arrays]):016x}"


def save(index: dict, name: str, entry: dict, res: dict, extra: dict | None = None) -> None:
    arrays = {k: v for k, v in res.items() if isinstance(v, np.ndarray)}
    arrays.update(extra or {})
    np.savez_compressed(os.path.join(BIG, f"{name}.npz"), **arrays)
    entry.update({k: v for k, v in res.items() if not isinstance(v, np.ndarray)})
    index[name] = entry
    with open(os.path.join(BIG, "index.json"), "w") as f:
        json.dump(index, f, indent=1, sort_keys=True)
    print(f"{name}: error={res['error']} iters={res['iterations_run']} obj={res['objective']:.6g}",
          flush=True)


def ref_gen(tmp: str, m, n, k, snr, seed, kind="cg") -> tuple[str, str]:
    d = os.path.join(tmp, f"gen_{m}_{n}")
    out = subprocess.run([REF, "gen", f"out={d}", f"m={m}", f"n={n}", f"k={k}", f"snr={snr}",
                          f"seed={seed}", f"kind={kind}"], check=True, capture_output=True, text=True)
    return d, out.stdout.split()[1]


def case_cfg2(tmp, index):
    d, h = ref_gen(tmp, 1024, 32768, 64, 30.0, 2)
    t0 = time.time()
    res = solve(d, os.path.join(tmp, "cfg2_out"), method="sectioning", N=8, rho=1, **{"lambda": 0.05},
                lambda_rel=1, iters=300, threads=THREADS)
    save(index, "cfg2_sectioning8_it300",
         {"problem": [1024, 32768, 64, 30.0, 2, "cg"], "fnv": h, "dtype": "c128",
          "solve": {"method": "sectioning", "N": 8, "rho": 1, "iters": 300}, "ref_seconds": time.time() - t0},
         res)


def promote_dir(src: str, dst: str, h64: np.ndarray | None = None, g: np.ndarray | None = None) -> None:
    """dst gets H rounded to complex64 and promoted back (what a c64 plan stores) + g."""
    os.makedirs(dst, exist_ok=True)
    if h64 is None:
        h64 = read_cmat(os.path.join(src, "h.cmat")).astype(np.complex64)
    write_cmat(os.path.join(dst, "h.cmat"), h64.astype(np.complex128))
    if g is None:
        shutil.copy(os.path.join(src, "g.cmat"), os.path.join(dst, "g.cmat"))
    else:
        write_cmat(os.path.join(dst, "g.cmat"), g)


def case_cfg4(tmp, index):
    d, h = ref_gen(tmp, 256, 262144, 1000, 30.0, 4)
    h64 = read_cmat(os.path.join(d, "h.cmat")).astype(np.complex64)
    g = read_cmat(os.path.join(d, "g.cmat")).ravel()
    fh64 = fnv(h64)
    d64 = os.path.join(tmp, "cfg4_c64")
    promote_dir(d, d64, h64)
    del h64
    t0 = time.time()
    res = solve(d64, os.path.join(tmp, "cfg4_out"), method="consensus", M=8, rho=1, **{"lambda": 0.05},
                lambda_rel=1, iters=1000, threads=THREADS)
    save(index, "cfg4_rows256_it1000",
         {"problem": [256, 262144, 1000, 30.0, 4, "cg"], "fnv": h, "fnv_h64": fh64, "dtype": "c64",
          "solve": {"method": "consensus", "M": 8, "rho": 1, "iters": 1000}, "ref_seconds": time.time() - t0},
         res)


def cra_inputs():
    import paper_1811_05571_b200 as admm
    p = admm.cra_problem(seed=3)  # config 3: H (c64), one 300-voxel scene
    return admm, p


def case_cfg3(tmp, index):
    admm, p = cra_inputs()
    d = os.path.join(tmp, "cfg3")
    promote_dir(None, d, p.h, p.g)
    t0 = time.time()
    res = solve(d, os.path.join(tmp, "cfg3_out"), method="hybrid", M=2, N=4, rho=1, **{"lambda": 0.03},
                lambda_rel=1, iters=500, threads=THREADS)
    save(index, "cfg3_hybrid24_it500",
         {"problem": "cra_matrix(seed=3, c64)", "fnv_h64": fnv(p.h), "dtype": "c64",
          "solve": {"method": "hybrid", "M": 2, "N": 4, "rho": 1, "iters": 500}, "ref_seconds": time.time() - t0},
         res, {"g": p.g, "truth": p.truth})


def case_cfg5(tmp, index, scenes=(0, 1)):
    admm, p = cra_inputs()
    g, truth = admm.cra_scenes(p.h, 64, seed=3)
    for b in scenes:
        d = os.path.join(tmp, f"cfg5_{b}")
        promote_dir(None, d, p.h, g[:, b])
        t0 = time.time()
        res = solve(d, os.path.join(tmp, f"cfg5_out{b}"), method="hybrid", M=2, N=4, rho=1,
                    **{"lambda": 0.03}, lambda_rel=1, iters=500, threads=THREADS)
        save(index, f"cfg5_scene{b}_it500",
             {"problem": "cra_matrix(seed=3, c64), cra_scenes(64, seed=3)", "scene": b, "fnv_h64": fnv(p.h),
              "dtype": "c64", "solve": {"method": "hybrid", "M": 2, "N": 4, "rho": 1, "iters": 500},
              "ref_seconds": time.time() - t0},
             res, {"g": g[:, b], "truth": truth[:, b]})
        shutil.rmtree(d, ignore_errors=True)


def main() -> None:
    if not os.path.exists(REF):
        sys.exit("build oracle/_ref first: make -C oracle")
    os.makedirs(BIG, exist_ok=True)
    want = sys.argv[1:] or ["cfg2", "cfg4", "cfg3", "cfg5"]
    p = os.path.join(BIG, "index.json")
    index = json.load(open(p)) if os.path.exists(p) else {}
    tmp = tempfile.mkdtemp(prefix="golden_big_", dir=os.environ.get("GOLDEN_TMP"))
    try:
        for w in want:
            t0 = time.time()
            {"cfg2": case_cfg2, "cfg3": case_cfg3, "cfg4": case_cfg4, "cfg5": case_cfg5}[w](tmp, index)
            print(f"{w} done in {time.time() - t0:.0f} s", flush=True)
            for e in os.listdir(tmp):
                shutil.rmtree(os.path.join(tmp, e), ignore_errors=True)
    finally:
        shutil.rmtree(tmp, ignore_errors=True)


if __name__ == "__main__":
    main()
