"""CMAT file I/O (cmat_io.hpp) through libadmm_b200.so — the input side of the path.

Same functions and error behaviour as the reference (cmat_io.hpp:44-125): ``read_cmat``
/ ``write_cmat`` / ``read_cvec`` / ``write_cvec``, raising IoError, FormatError (with
``byte_offset()``), ParameterError and NumericalError exactly where the reference does.
Added: a complex64 file variant ("CMF1", half the bytes; ``dtype="c64"`` on write) and
conversion on read (``dtype="c64"`` rounds a CMX1 file straight into complex64 storage,
the layout a c64 plan uploads, without an FP64 host copy).
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

from . import _lib
from .errors import FormatError, check

_DT = {"c128": (0, np.complex128), "c64": (1, np.complex64)}


def _path(p) -> bytes:
    return os.fsencode(os.fspath(p))


def cmat_info(path) -> tuple:
    """(rows, cols, file dtype "c128" | "c64") from the validated header."""
    r, c, t = _lib._u64(), _lib._u64(), ctypes.c_int32()
    check(_lib.lib.admm_cmat_info(_path(path), ctypes.byref(r), ctypes.byref(c), ctypes.byref(t)))
    return int(r.value), int(c.value), ("c128", "c64")[t.value]


def read_cmat(path, dtype: str = "c128") -> np.ndarray:
    """read_cmat (cmat_io.hpp:57-105): rows x cols complex matrix of ``dtype``."""
    rows, cols, _ = cmat_info(path)
    code, npt = _DT[dtype]
    out = np.empty((rows, cols), dtype=npt)
    check(_lib.lib.admm_cmat_read(_path(path), out.ctypes.data, out.size, code))
    return out


def write_cmat(path, a, dtype: str = "c128") -> None:
    """write_cmat (cmat_io.hpp:44-55); ``dtype="c64"`` writes the CMF1 variant."""
    a = np.asarray(a)
    if a.ndim != 2:
        a = a.reshape(a.shape[0] if a.ndim else 0, -1) if a.size else np.zeros((0, 0), np.complex128)
    src = np.ascontiguousarray(a, dtype=np.complex64 if a.dtype == np.complex64 else np.complex128)
    sc = 1 if src.dtype == np.complex64 else 0
    check(_lib.lib.admm_cmat_write(_path(path), src.ctypes.data if src.size else None, src.shape[0],
                                   src.shape[1] if src.ndim == 2 else 0, sc, _DT[dtype][0]))


def write_cvec(path, v, dtype: str = "c128") -> None:
    """write_cvec (cmat_io.hpp:108-113): a cols == 1 file."""
    v = np.asarray(v).reshape(-1)
    write_cmat(path, v.reshape(v.size, 1) if v.size else np.zeros((0, 1), np.complex128), dtype)


def read_cvec(path, dtype: str = "c128") -> np.ndarray:
    """read_cvec (cmat_io.hpp:115-125): FormatError(offset 12) unless cols == 1."""
    rows, cols, _ = cmat_info(path)
    if cols != 1:
        raise FormatError(f"read_cvec: {os.fspath(path)} holds a {rows}x{cols} matrix, "
                          "expected a column vector", 12)
    return read_cmat(path, dtype).reshape(-1)
