"""ctypes binding of the sm_100a C-ABI library ``libcfgsim.so`` (include/cfgsim.h).

The library is built in-tree by ``__graft_entry__.build()``
(``csrc/Makefile``).  There is no CPU fallback: if the library is missing
this module raises on import, and every compute entry point raises
``DeviceError`` when no sm_100 GPU is visible.
"""

from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

import numpy as np

from .errors import BadOrder, DegenerateInput, DeviceError, DimMismatch

LIB_PATH = Path(__file__).resolve().parent / "libcfgsim.so"
if os.environ.get("CFGSIM_LIBRARY"):  # A/B runs of alternative builds of the same library
    LIB_PATH = Path(os.environ["CFGSIM_LIBRARY"]).resolve()

OK, ERR_ARG, ERR_DIM, ERR_CUDA, ERR_NOMEM, ERR_NODEVICE, ERR_DEGENERATE, ERR_ORDER = range(8)
(ERR_LISTING_SYNTAX, ERR_UNRESOLVED_LABEL, ERR_PROFILE_SYNTAX, ERR_DUPLICATE_KERNEL, ERR_EMPTY_GRAPH, ERR_CORPUS,
 ERR_VALUE, ERR_INDEX) = range(8, 16)
MODE_IDS = {"row_stochastic": 0, "global": 1, "raw_counts": 2}
FLAT_IDS = {"euc": 0, "man": 1, "min": 2, "jac": 3, "cos": 4}
FP64, FP32 = 0, 1

if not LIB_PATH.exists():
    raise ImportError(
        f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
        "(the IsoRank path runs only on sm_100a; there is no CPU fallback)"
    )

lib = C.CDLL(str(LIB_PATH))


class Params(C.Structure):
    _fields_ = [("alpha", C.c_double), ("tol", C.c_double), ("max_iter", C.c_int32),
                ("precision", C.c_int32), ("tol_fp32", C.c_double)]


_vp = C.c_void_p
_i32 = C.c_int32
_i64 = C.c_int64
_pp = C.POINTER(Params)

_SIGS = {
    "cfgsim_last_error": ([], C.c_char_p),
    "cfgsim_version": ([], C.c_int),
    "cfgsim_device_count": ([_vp], C.c_int),
    "cfgsim_corpus_create": ([_i32, _i32, _vp, _vp, _vp, _vp, _vp, _vp, C.POINTER(_vp)], C.c_int),
    "cfgsim_corpus_create_dense": ([_i32, _i32, _vp, _vp, C.POINTER(_vp)], C.c_int),
    "cfgsim_corpus_destroy": ([_vp], C.c_int),
    "cfgsim_corpus_info": ([_vp, _vp, _vp, _vp], C.c_int),
    "cfgsim_isorank_pairs": ([_vp, _vp, _i64, _vp, _vp, _pp, _vp, _vp, _vp, _vp, _vp], C.c_int),
    "cfgsim_allpairs_units": ([_vp, _vp], C.c_int),
    "cfgsim_allpairs_split": ([_vp, _i32, _vp], C.c_int),
    "cfgsim_allpairs_range": ([_vp, _i64, _i64, _i32, _pp, _vp, _vp, _vp], C.c_int),
    "cfgsim_allpairs_scatter": ([_vp, _i32, _vp, _vp, _vp, _vp, _vp], C.c_int),
    "cfgsim_allpairs": ([_vp, _i32, _pp, _vp, _vp, _vp], C.c_int),
    "cfgsim_isorank_single": ([_i32, _i32, _vp, _i32, _vp, _pp, _vp, _vp, _vp, _vp, _vp, _vp, _vp],
                              C.c_int),
    "cfgsim_nearest": ([_vp, _vp, _i32, _i32, _pp, _vp, _vp, _vp], C.c_int),
    "cfgsim_interpolate": ([_i32, _i32, _vp, _i32, _vp], C.c_int),
    "cfgsim_flat_single": ([_i32, _i32, _vp, _i32, _vp, _i32, C.c_double, _vp], C.c_int),
    "cfgsim_flat_pairs": ([_vp, _vp, _i64, _vp, _vp, _i32, C.c_double, _vp, _vp], C.c_int),
    "cfgsim_flat_allpairs": ([_vp, _i32, C.c_double, _vp, _vp], C.c_int),
    "cfgsim_flat_all_allpairs": ([_vp, C.c_double, _vp, _vp], C.c_int),
    "cfgsim_probe_fp64": ([_i32, _vp, _vp], C.c_int),
    "cfgsim_host_alloc": ([C.c_int64, C.POINTER(C.c_void_p)], C.c_int),
    "cfgsim_host_free": ([_vp], C.c_int),
    "cfgsim_heatmap_csv": ([_i32, _vp, _vp, _vp, _vp, _i64, _vp, _i32], C.c_int),
    "cfgsim_ward": ([_i32, _i32, _i32, _vp, _vp, _vp, _vp, _vp], C.c_int),
    "cfgsim_matrices_from_listings": ([_i32, _vp, _vp, _vp, _vp, _vp, _i32, _i32, C.POINTER(_vp)], C.c_int),
    "cfgsim_matrices_sizes": ([_vp, _vp, _vp], C.c_int),
    "cfgsim_matrices_read": ([_vp, _vp, _vp], C.c_int),
    "cfgsim_matrices_status": ([_vp, _i32, _vp, _vp, C.c_char_p, _i64], C.c_int),
    "cfgsim_matrices_destroy": ([_vp], None),
    "cfgsim_launch_count": ([], C.c_int64),
}
for _name, (_args, _res) in _SIGS.items():
    _f = getattr(lib, _name)
    _f.argtypes = _args
    _f.restype = _res

EXPORTED = tuple(_SIGS)


def check(rc: int) -> None:
    if rc == OK:
        return
    msg = (lib.cfgsim_last_error() or b"").decode(errors="replace")
    if rc == ERR_ARG:
        raise ValueError(msg)
    if rc == ERR_DIM:
        raise DimMismatch(msg)
    if rc == ERR_NOMEM:
        raise MemoryError(msg)
    if rc == ERR_DEGENERATE:
        raise DegenerateInput(msg)
    if rc == ERR_ORDER:
        raise BadOrder(msg)
    raise DeviceError(msg)


def ptr(a) -> int | None:
    """Raw address of a numpy array or torch tensor (None for None)."""
    if a is None:
        return None
    if isinstance(a, np.ndarray):
        return a.ctypes.data
    if hasattr(a, "data_ptr"):
        return a.data_ptr()
    if isinstance(a, int):
        return a
    raise TypeError(f"cannot take the address of {type(a)!r}")


def params(alpha=0.85, tol=1e-9, max_iter=1000, precision="fp64", tol_fp32=1e-7) -> Params:
    if precision not in ("fp64", "fp32"):
        raise ValueError(f"precision must be 'fp64' or 'fp32', got {precision!r}")
    return Params(float(alpha), float(tol), int(max_iter), FP64 if precision == "fp64" else FP32,
                  float(tol_fp32))


def device_count() -> int:
    n = np.zeros(1, np.int32)
    check(lib.cfgsim_device_count(ptr(n)))
    return int(n[0])


def default_device() -> int:
    return int(os.environ.get("LOCAL_RANK", "0")) if device_count() > 1 else 0


def launch_count() -> int:
    return int(lib.cfgsim_launch_count())


class _PinnedBuffer:
    """Page-locked host memory (cfgsim_host_alloc) exposed to numpy; freed
    when the last array viewing it is gone."""

    def __init__(self, nbytes: int):
        p = C.c_void_p()
        check(lib.cfgsim_host_alloc(int(nbytes), C.byref(p)))
        self.ptr = p.value
        self.nbytes = int(nbytes)
        self.__array_interface__ = {"shape": (self.nbytes,), "typestr": "|u1", "data": (self.ptr, False),
                                    "version": 3}

    def __del__(self):
        if getattr(self, "ptr", None):
            try:
                lib.cfgsim_host_free(self.ptr)
            except Exception:  # (interpreter shutdown: the module is already torn down)
                pass
            self.ptr = None


_PINNED: list = []  # [buffer, weakref of the array last handed out]


def pinned_array(shape, dtype=np.float64) -> np.ndarray:
    """An uninitialised array in page-locked memory for K x K results: a
    buffer is reused once no array handed out from it is alive, so repeated
    calls neither pin new memory nor fault fresh pages (device results land
    by DMA; the host scatter writes resident pages)."""
    import weakref
    dtype = np.dtype(dtype)
    nbytes = int(np.prod(shape)) * dtype.itemsize
    if nbytes < (1 << 20):
        return np.empty(shape, dtype)
    for ent in _PINNED:
        buf, ref = ent
        if buf.nbytes >= nbytes and (ref is None or ref() is None):
            a = np.asarray(buf)[:nbytes].view(dtype).reshape(shape)
            ent[1] = weakref.ref(a)
            return a
    try:
        buf = _PinnedBuffer(nbytes)
    except DeviceError:  # (no driver: plain host memory; the compute call itself will report it)
        return np.empty(shape, dtype)
    a = np.asarray(buf)[:nbytes].view(dtype).reshape(shape)
    _PINNED.append([buf, weakref.ref(a)])
    return a
