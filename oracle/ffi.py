"""ctypes binding of oracle/build/liboracle.so — TEST INFRASTRUCTURE ONLY."""

from __future__ import annotations

import ctypes as C
import os
import subprocess
from pathlib import Path

import numpy as np

_HERE = Path(__file__).resolve().parent
_LIB_PATH = _HERE / "build" / "liboracle.so"
_lib = None


def build() -> Path:
    subprocess.run(["make", "-s", "-C", str(_HERE)], check=True)
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not _LIB_PATH.exists():
            build()
        _lib = C.CDLL(str(_LIB_PATH))
        dp = C.POINTER(C.c_double)
        ip = C.POINTER(C.c_int32)
        lp = C.POINTER(C.c_int64)
        up = C.POINTER(C.c_uint8)
        _lib.oracle_iso_pair.argtypes = [C.c_int, dp, C.c_int, dp, C.c_double, C.c_double, C.c_int,
                                         dp, dp, ip, dp, dp, ip, up]
        _lib.oracle_iso_batch.argtypes = [ip, lp, ip, lp, ip, dp, C.c_int64, ip, ip, C.c_double,
                                          C.c_double, C.c_int, C.c_int, dp, dp, ip, up]
    return _lib


def _p(a, t):
    return None if a is None else a.ctypes.data_as(C.POINTER(t))


def iso_pair(a, b, alpha=0.85, tol=1e-9, max_iter=1000, start=None):
    """normalize_pair + isorank_align + isorank_distance on dense inputs.

    Returns dict(X, matching, d, W, iterations, converged)."""
    a = np.ascontiguousarray(a, dtype=np.float64)
    b = np.ascontiguousarray(b, dtype=np.float64)
    n = max(a.shape[0], b.shape[0])
    x0 = None
    if start is not None:
        x0 = np.ascontiguousarray(np.asarray(start, dtype=float) / np.sum(start))
    X = np.empty((n, n))
    m = np.empty(n, np.int32)
    d = np.empty(1)
    w = np.empty(1)
    it = np.empty(1, np.int32)
    cv = np.empty(1, np.uint8)
    rc = lib().oracle_iso_pair(a.shape[0], _p(a, C.c_double), b.shape[0], _p(b, C.c_double), alpha,
                               tol, max_iter, _p(x0, C.c_double), _p(X, C.c_double),
                               _p(m, C.c_int32), _p(d, C.c_double), _p(w, C.c_double),
                               _p(it, C.c_int32), _p(cv, C.c_uint8))
    if rc:
        raise ValueError(f"oracle_iso_pair rc={rc}")
    return dict(X=X, matching=tuple(int(v) for v in m), d=float(d[0]), W=float(w[0]),
                iterations=int(it[0]), converged=bool(cv[0]))


def iso_batch(packed, ia, ib, alpha=0.85, tol=1e-9, max_iter=1000, threads=None):
    """Batch over a packed corpus (dict with n_nodes, rp_off, rowptr, nz_off, col, val)."""
    threads = threads or os.cpu_count() or 1
    ia = np.ascontiguousarray(ia, np.int32)
    ib = np.ascontiguousarray(ib, np.int32)
    n = len(ia)
    d = np.empty(n)
    w = np.empty(n)
    it = np.empty(n, np.int32)
    cv = np.empty(n, np.uint8)
    rc = lib().oracle_iso_batch(_p(packed["n_nodes"], C.c_int32), _p(packed["rp_off"], C.c_int64),
                                _p(packed["rowptr"], C.c_int32), _p(packed["nz_off"], C.c_int64),
                                _p(packed["col"], C.c_int32), _p(packed["val"], C.c_double), n,
                                _p(ia, C.c_int32), _p(ib, C.c_int32), alpha, tol, max_iter,
                                int(threads), _p(d, C.c_double), _p(w, C.c_double),
                                _p(it, C.c_int32), _p(cv, C.c_uint8))
    if rc:
        raise ValueError(f"oracle_iso_batch rc={rc}")
    return d, w, it, cv.astype(bool)
