"""Host-side CSR packing of a corpus (no CUDA, no libcfgsim.so).

Kept apart from ``corpus.py`` so that test infrastructure and the CPU
reference arm of ``bench.py`` can pack matrices without loading the GPU
library.  Layout: include/cfgsim.h ("Packed corpus").
"""

from __future__ import annotations

from typing import Sequence

import numpy as np


def _entries(m) -> np.ndarray:
    e = getattr(m, "entries", m)
    return np.asarray(e, dtype=np.float64)


def pack(matrices: Sequence) -> dict[str, np.ndarray]:
    """CSR of every matrix (TransitionMatrix or square ndarray), concatenated.

    Layout (include/cfgsim.h): graph g's row pointer is
    ``rowptr[rp_off[g] : rp_off[g] + n + 1]`` (local offsets), its entries
    ``col/val[nz_off[g] : nz_off[g] + nnz_g]`` in row-major order."""
    k = len(matrices)
    n_nodes = np.empty(k, np.int32)
    rp_off = np.empty(k, np.int64)
    nz_off = np.empty(k, np.int64)
    rowptrs, cols, vals = [], [], []
    rp_at = nz_at = 0
    for g, m in enumerate(matrices):
        e = _entries(m)
        if e.ndim != 2 or e.shape[0] != e.shape[1] or e.shape[0] < 1:
            raise ValueError(f"matrix {g}: entries must be square and non-empty, got {e.shape}")
        n = e.shape[0]
        r, c = np.nonzero(e)
        rp = np.zeros(n + 1, np.int32)
        np.cumsum(np.bincount(r, minlength=n), out=rp[1:])
        n_nodes[g] = n
        rp_off[g] = rp_at
        nz_off[g] = nz_at
        rowptrs.append(rp)
        cols.append(c.astype(np.int32))
        vals.append(e[r, c])
        rp_at += n + 1
        nz_at += len(r)
    cat = lambda xs, dt: np.ascontiguousarray(np.concatenate(xs) if xs else np.zeros(0, dt), dt)
    return dict(n_nodes=n_nodes, rp_off=rp_off, rowptr=cat(rowptrs, np.int32),
                nz_off=nz_off, col=cat(cols, np.int32), val=cat(vals, np.float64))


def packed_bytes(packed: dict) -> int:
    return int(sum(a.nbytes for a in packed.values()))
