"""ctypes binding of the TEST-ONLY oracle (oracle/liboracle.so, the C restatement).

Importable only from tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ORACLE_DIR = os.path.join(REPO, "oracle")
LIB_PATH = os.path.join(ORACLE_DIR, "liboracle.so")
REF_BIN = os.path.join(ORACLE_DIR, "_ref", "admmsplit_ref")

ERRORS = {0: "none", 1: "DimensionError", 2: "IndexError", 3: "NumericalError",
          4: "SingularityError", 5: "PartitionError", 6: "ParameterError", 7: "AllocError"}
METHODS = {"reference": 0, "consensus": 1, "sectioning": 2, "hybrid": 3}

_lib = None


def lib() -> ctypes.CDLL:
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            subprocess.run(["make", "-C", ORACLE_DIR, "liboracle.so"], check=True,
                           capture_output=True)
        _lib = ctypes.CDLL(LIB_PATH)
        u64, dbl, ptr, i32 = ctypes.c_uint64, ctypes.c_double, ctypes.c_void_p, ctypes.c_int
        _lib.orc_gen_problem.argtypes = [u64, u64, u64, dbl, u64, i32, ptr, ptr, ptr, ptr]
        _lib.orc_fnv1a64.argtypes = [ptr, u64, u64]
        _lib.orc_fnv1a64.restype = u64
        _lib.orc_random_gauss.argtypes = [u64, u64, ptr]
        _lib.orc_matvec.argtypes = [ptr, u64, u64, ptr, ptr]
        _lib.orc_adjoint_matvec.argtypes = [ptr, u64, u64, ptr, ptr]
        _lib.orc_soft_threshold_vec.argtypes = [ptr, u64, dbl, ptr]
        _lib.orc_gram_solve.argtypes = [ptr, u64, u64, dbl, i32, ptr, ptr]
        _lib.orc_gram_solve.restype = i32
        _lib.orc_split_bounds.argtypes = [u64, u64, i32, ptr]
        _lib.orc_split_bounds.restype = i32
        _lib.orc_objective.argtypes = [ptr, u64, u64, ptr, ptr, dbl]
        _lib.orc_objective.restype = dbl
        _lib.orc_solve.argtypes = [i32, ptr, ptr, u64, u64, u64, u64, i32, dbl, dbl, dbl, u64,
                                   dbl, dbl, ptr, ptr, ptr, ptr, ptr, ptr]
        _lib.orc_solve.restype = i32
    return _lib


def _p(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


def gen_problem(m, n, k, snr, seed, kind="cg"):
    h = np.empty((m, n), np.complex128)
    g = np.empty(m, np.complex128)
    t = np.empty(n, np.complex128)
    ns = np.zeros(1, np.float64)
    snr = float("inf") if snr in ("inf", None) else float(snr)
    st = lib().orc_gen_problem(m, n, k, snr, seed, 0 if kind == "cg" else 1, _p(h), _p(g), _p(t),
                               _p(ns))
    if st:
        raise RuntimeError(ERRORS[st])
    return h, g, t, float(ns[0])


def random_gauss(count, seed):
    out = np.empty(count, np.complex128)
    lib().orc_random_gauss(count, seed, _p(out))
    return out


def matvec(a, x):
    a = np.ascontiguousarray(a, np.complex128)
    x = np.ascontiguousarray(x, np.complex128)
    y = np.empty(a.shape[0], np.complex128)
    lib().orc_matvec(_p(a), a.shape[0], a.shape[1], _p(x), _p(y))
    return y


def adjoint_matvec(a, x):
    a = np.ascontiguousarray(a, np.complex128)
    x = np.ascontiguousarray(x, np.complex128)
    y = np.empty(a.shape[1], np.complex128)
    lib().orc_adjoint_matvec(_p(a), a.shape[0], a.shape[1], _p(x), _p(y))
    return y


def soft_threshold_vec(a, kappa):
    a = np.ascontiguousarray(a, np.complex128)
    out = np.empty_like(a)
    lib().orc_soft_threshold_vec(_p(a), a.size, float(kappa), _p(out))
    return out


def gram_solve(h, rho, rhs, strategy=-1):
    h = np.ascontiguousarray(h, np.complex128)
    rhs = np.ascontiguousarray(rhs, np.complex128)
    x = np.empty(h.shape[1], np.complex128)
    st = lib().orc_gram_solve(_p(h), h.shape[0], h.shape[1], float(rho), strategy, _p(rhs), _p(x))
    if st:
        raise RuntimeError(ERRORS[st])
    return x


def objective(h, g, v, lam):
    h = np.ascontiguousarray(h, np.complex128)
    g = np.ascontiguousarray(g, np.complex128)
    v = np.ascontiguousarray(v, np.complex128)
    return lib().orc_objective(_p(h), h.shape[0], h.shape[1], _p(g), _p(v), float(lam))


def solve(method, h, g, M=1, N=1, ragged=False, rho=1.0, lam=1.0, scl=1.0, iters=50,
          eps_pri=0.0, eps_dual=0.0, snapshots=False):
    """Returns dict(error, last_good, iterations_run, objective, solution, trace, snapshots)."""
    h = np.ascontiguousarray(h, np.complex128)
    g = np.ascontiguousarray(g, np.complex128)
    m, n = h.shape
    sol = np.zeros(n, np.complex128)
    trace = np.zeros((iters, 3), np.float64)
    it = np.zeros(1, np.uint64)
    obj = np.zeros(1, np.float64)
    lg = np.zeros(1, np.uint64)
    snaps = np.zeros((iters, n), np.complex128) if snapshots else None
    st = lib().orc_solve(METHODS[method], _p(h), _p(g), m, n, M, N, int(ragged), float(rho),
                         float(lam), float(scl), iters, float(eps_pri), float(eps_dual), _p(sol),
                         _p(trace), _p(it), _p(obj), _p(lg),
                         _p(snaps) if snaps is not None else None)
    k = int(it[0])
    out = {"error": ERRORS[st], "last_good": int(lg[0]), "iterations_run": k,
           "objective": float(obj[0]), "solution": sol, "trace": trace[:k]}
    if snaps is not None:
        out["snapshots"] = snaps[:k]
    return out


def fnv1a64(*arrays, h=0xCBF29CE484222325):
    for a in arrays:
        a = np.ascontiguousarray(a)
        h = lib().orc_fnv1a64(_p(a), a.nbytes, h)
    return h
