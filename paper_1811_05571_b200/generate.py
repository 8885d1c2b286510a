"""Synthetic inputs for the BASELINE configs (input tooling, host side).

gen_problem restates generate.hpp:32-89 bit-for-bit (in libadmm_b200.so, pinned by
tests/test_generate.py against the reference's own output).  cra_problem builds the
CRA-like structured operator of configs 3 and 5 (no reference counterpart; the
paper's measured CRA matrix was never published) with its sparse planar-patch scenes.
"""
from __future__ import annotations

import ctypes
import math

import numpy as np

from . import _lib
from .errors import check
from .solvers import ProblemKind, SensingProblem


def _ptr(a):
    return a.ctypes.data_as(ctypes.c_void_p)


def gen_problem(n_meas: int, n_pix: int, sparsity_k: int, snr_db: float, seed: int,
                kind: ProblemKind = ProblemKind.ComplexGaussian, dtype: str = "c128") -> SensingProblem:
    """generate.hpp:32-89.  dtype="c64" returns H rounded to complex64 (g from FP64 H)."""
    c64 = dtype in ("c64", "complex64")
    h = np.empty((n_meas, n_pix), np.complex64 if c64 else np.complex128)
    g = np.empty(n_meas, np.complex128)
    t = np.empty(n_pix, np.complex128)
    ns = ctypes.c_double()
    k = 0 if kind in (ProblemKind.ComplexGaussian, "cg") else 1
    check(_lib.lib.admm_gen_problem(n_meas, n_pix, sparsity_k, float(snr_db), seed, k, _ptr(h),
                                    1 if c64 else 0, _ptr(g), _ptr(t), ctypes.byref(ns)))
    return SensingProblem(h, g, t, ns.value, ProblemKind.ComplexGaussian if k == 0 else ProblemKind.RandomPhase)


# BASELINE.json config 3: 24 transceivers on a 0.5 m aperture, 128 frequencies over
# 70-77 GHz, 32^3 voxels at 5 mm centred 0.6 m away, 64 reflector facets.
CRA = dict(n_tx=24, n_freq=128, grid=32, spacing=5e-3, z0=0.6, aperture=0.5, f0=70e9, f1=77e9,
           n_facets=64)


def cra_matrix(seed: int, dtype: str = "c64", **over) -> np.ndarray:
    p = dict(CRA, **over)
    rows = p["n_tx"] * p["n_freq"]
    cols = p["grid"] ** 3
    c64 = dtype in ("c64", "complex64")
    h = np.empty((rows, cols), np.complex64 if c64 else np.complex128)
    check(_lib.lib.admm_gen_cra(p["n_tx"], p["n_freq"], p["grid"], p["spacing"], p["z0"],
                                p["aperture"], p["f0"], p["f1"], p["n_facets"], seed, _ptr(h),
                                1 if c64 else 0))
    return h


def planar_patch(grid: int, n_vox: int, rng: np.random.Generator) -> np.ndarray:
    """Indices of n_vox voxels on a random tilted plane through the grid: the plane
    normal is drawn uniformly on the upper hemisphere (tilt < 60 degrees), the plane
    passes through a random point of the central half of the grid, and the voxels
    nearest to the plane and to that point are selected."""
    while True:
        nz = rng.uniform(0.5, 1.0)
        phi = rng.uniform(0.0, 2 * math.pi)
        s = math.sqrt(1 - nz * nz)
        n = np.array([s * math.cos(phi), s * math.sin(phi), nz])
        c = rng.uniform(grid * 0.25, grid * 0.75, size=3)
        ix, iy, iz = np.meshgrid(np.arange(grid), np.arange(grid), np.arange(grid), indexing="ij")
        pts = np.stack([ix.ravel(), iy.ravel(), iz.ravel()], 1).astype(np.float64)
        dist = np.abs((pts - c) @ n)
        near = np.nonzero(dist <= 0.5)[0]
        if near.size >= n_vox:
            r = np.linalg.norm(pts[near] - c, axis=1)
            return np.sort(near[np.argsort(r, kind="stable")[:n_vox]])


def add_noise(clean: np.ndarray, snr_db: float, rng: np.random.Generator) -> tuple:
    """Exact-SNR complex gaussian noise (the rule of generate.hpp:76-85)."""
    w = rng.standard_normal(clean.shape) + 1j * rng.standard_normal(clean.shape)
    alpha = np.linalg.norm(clean) / (np.linalg.norm(w) * 10 ** (snr_db / 20))
    return clean + alpha * w, float(alpha)


def cra_problem(seed: int = 3, n_vox: int = 300, snr_db: float = 30.0, dtype: str = "c64",
                **over) -> SensingProblem:
    """BASELINE config 3: CRA-like H, one planar-patch scene of unit reflectivity."""
    h = cra_matrix(seed, dtype, **over)
    grid = dict(CRA, **over)["grid"]
    rng = np.random.default_rng(seed + 1000)
    truth = np.zeros(h.shape[1], np.complex128)
    truth[planar_patch(grid, n_vox, rng)] = 1.0
    clean = h.astype(np.complex128) @ truth
    g, sigma = add_noise(clean, snr_db, rng)
    return SensingProblem(h, g, truth, sigma, ProblemKind.FromFile)


def cra_scenes(h: np.ndarray, n_scenes: int, seed: int, lo: int = 100, hi: int = 400,
               snr_db: float = 30.0, grid: int = 32):
    """BASELINE config 5: n_scenes independent planar-patch scenes (100-400 voxels)."""
    rng = np.random.default_rng(seed + 5000)
    truth = np.zeros((h.shape[1], n_scenes), np.complex128)
    for b in range(n_scenes):
        truth[planar_patch(grid, int(rng.integers(lo, hi + 1)), rng), b] = 1.0
    clean = h.astype(np.complex128) @ truth
    g = np.empty_like(clean)
    for b in range(n_scenes):
        g[:, b], _ = add_noise(clean[:, b], snr_db, rng)
    return g, truth
