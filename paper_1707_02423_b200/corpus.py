"""CFG batching layer: pack transition matrices into CSR and keep them on the GPU.

Replaces the reference's ``list[TransitionMatrix]`` walked pair by pair
(``similarity.py:229-246``).  A corpus is packed once on the host
(``pack``), uploaded once per device (``DeviceCorpus``), and then every
all-pairs / query launch reads it from HBM.  The raw ``entries`` are packed
(not the row-normalised operator): bilinear size normalisation depends on
the partner's size, so it happens per pair inside the kernel prologue.
"""

from __future__ import annotations

import ctypes
from typing import Sequence

import numpy as np

from . import _native as nat
from .packing import _entries, pack, packed_bytes  # noqa: F401  (re-exported)



_read_ptr = ctypes.c_void_p.from_address
_DATA_OFFSET = 16  # PyArrayObject: PyObject_HEAD (refcount, type), then `char *data`


def _data_pointers(arrays: list) -> list:
    """Data addresses of ndarrays, read from each array object's `data` field
    (numpy's C ABI, PyArrayObject_fields) — ~5x cheaper per array than
    ``a.ctypes.data``, which matters on the per-call path of a 2k-matrix
    corpus.  Checked against ``__array_interface__`` on the first and last
    array; any mismatch falls back to the interface for every array."""
    if not arrays:
        return []
    ptrs = [_read_ptr(id(a) + _DATA_OFFSET).value for a in arrays]
    if (ptrs[0] != arrays[0].__array_interface__["data"][0]
            or ptrs[-1] != arrays[-1].__array_interface__["data"][0]):
        ptrs = [a.__array_interface__["data"][0] for a in arrays]
    return ptrs


class DeviceCorpus:
    """A packed corpus resident in one GPU's HBM (``cfgsim_corpus_create``)."""

    def __init__(self, matrices_or_packed, device: int | None = None):
        self.device = nat.default_device() if device is None else int(device)
        h = nat.C.c_void_p()
        if isinstance(matrices_or_packed, dict):
            packed = matrices_or_packed
            self.n_nodes = packed["n_nodes"]
            self.K = int(len(self.n_nodes))
            nat.check(nat.lib.cfgsim_corpus_create(
                self.device, self.K, nat.ptr(packed["n_nodes"]), nat.ptr(packed["rp_off"]),
                nat.ptr(packed["rowptr"]), nat.ptr(packed["nz_off"]), nat.ptr(packed["col"]),
                nat.ptr(packed["val"]), nat.C.byref(h)))
        else:  # dense entries: the CSR is built natively (cfgsim_corpus_create_dense)
            es = [np.ascontiguousarray(_entries(m)) for m in matrices_or_packed]
            for g, e in enumerate(es):
                if e.ndim != 2 or e.shape[0] != e.shape[1] or e.shape[0] < 1:
                    raise ValueError(f"matrix {g}: entries must be square and non-empty, got {e.shape}")
            self.n_nodes = np.array([e.shape[0] for e in es], np.int32)
            self.K = len(es)
            ptrs = (nat.C.c_void_p * self.K)(*_data_pointers(es))
            nat.check(nat.lib.cfgsim_corpus_create_dense(self.device, self.K, nat.ptr(self.n_nodes), ptrs,
                                                         nat.C.byref(h)))
        self._h = h
        info = np.zeros(1, np.int64)
        nat.check(nat.lib.cfgsim_corpus_info(h, None, None, nat.ptr(info)))
        self.h2d_bytes = int(info[0])

    @property
    def handle(self):
        return self._h

    def close(self):
        if getattr(self, "_h", None) is not None and self._h.value:
            nat.lib.cfgsim_corpus_destroy(self._h)
            self._h = nat.C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    # ---- all-pairs over the size-sorted upper triangle (include/cfgsim.h)
    def n_units(self) -> int:
        out = np.zeros(1, np.int64)
        nat.check(nat.lib.cfgsim_allpairs_units(self._h, nat.ptr(out)))
        return int(out[0])

    def split(self, world: int) -> np.ndarray:
        b = np.zeros(world + 1, np.int64)
        nat.check(nat.lib.cfgsim_allpairs_split(self._h, world, nat.ptr(b)))
        return b
