"""Access to the golden fixtures in tests/golden/ (made by tests/golden/make_golden.py from
the unmodified reference).  Inputs are regenerated with the seeded generator; the stored
FNV hash pins them."""
from __future__ import annotations

import json
import os

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def index() -> dict:
    with open(os.path.join(GOLDEN, "index.json")) as f:
        return json.load(f)


def solve_cases() -> list[str]:
    return sorted(k for k, v in index().items() if "solve" in v)


def gen_cases() -> list[str]:
    return sorted(k for k, v in index().items() if "solve" not in v)


def load(name: str) -> tuple[dict, dict]:
    entry = index()[name]
    path = os.path.join(GOLDEN, f"{name}.npz")
    arrays = dict(np.load(path)) if os.path.exists(path) else {}
    return entry, arrays


def solver_args(entry: dict) -> dict:
    """Keyword arguments (method, M, N, ragged, rho, lam, scl, iters, eps_*) of a case; lambda
    is the absolute value the reference actually used (relative rules already applied)."""
    s = entry["solve"]
    return dict(method=s["method"], M=int(s.get("M", 1)), N=int(s.get("N", 1)),
                ragged=bool(int(s.get("ragged", 0))), rho=float(s.get("rho", 1.0)),
                lam=float(entry["lambda"]), scl=float(s.get("scl", 1.0)),
                iters=int(s.get("iters", 50)), eps_pri=float(s.get("eps_pri", 0.0)),
                eps_dual=float(s.get("eps_dual", 0.0)))


def problem(entry: dict, gen) -> tuple[np.ndarray, np.ndarray, np.ndarray]:
    """(H, g, truth) for a case using generator `gen(m, n, k, snr, seed, kind)`."""
    m, n, k, snr, seed, kind = entry["problem"]
    h, g, t, _ = gen(m, n, k, snr, seed, kind)
    if entry.get("prescale") is not None:
        h = h * entry["prescale"]
        g = g * entry["prescale"]
    return h, g, t
