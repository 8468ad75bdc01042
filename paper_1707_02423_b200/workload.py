"""Algorithmic work accounting for the roofline; host-side numpy.

Per pair and per sweep the algorithmic FLOP count is
    2N(S_A + S_B) + N(z_A + z_B) + 8N^2
S = nonzeros of the size-normalised, row-normalised operator outside its
uniform rows (= nonzeros of the interpolated matrix), z = uniform
(all-zero) rows, N = max(n_a, n_b).  Shared-memory bytes per sweep are
2 N^2 w (w = 8 fp64 / 4 fp32).  Multiplied by the pair's iteration count.
These figures are implementation-independent; they are what
``roofline.achieved`` divides by the measured kernel time.
"""

from __future__ import annotations

import numpy as np


def _interp_pattern(e: np.ndarray, N: int) -> np.ndarray:
    n = e.shape[0]
    if N == n:
        return e
    if n == 1:
        return np.full((N, N), e[0, 0])
    pos = (np.arange(N) * (n - 1)) / (N - 1)
    lo = np.minimum(np.floor(pos).astype(int), n - 2)
    fr = (pos - lo)
    rows = (1 - fr)[:, None] * e[lo] + fr[:, None] * e[lo + 1]
    return (1 - fr)[None, :] * rows[:, lo] + fr[None, :] * rows[:, lo + 1]


def operator_stats(mats, nmax: int) -> tuple[np.ndarray, np.ndarray]:
    """S[g, N], Z[g, N] for every graph g and every N in [n_g, nmax]."""
    k = len(mats)
    S = np.zeros((k, nmax + 1), np.int64)
    Z = np.zeros((k, nmax + 1), np.int64)
    for g, m in enumerate(mats):
        e = np.asarray(getattr(m, "entries", m), float)
        for N in range(e.shape[0], nmax + 1):
            a = _interp_pattern(e, N) != 0
            S[g, N] = int(a.sum())
            Z[g, N] = int((~a.any(axis=1)).sum())
    return S, Z


def pair_flops(N, Sa, Sb, Za, Zb, iters) -> np.ndarray:
    N = np.asarray(N, np.float64)
    per_sweep = 2.0 * N * (Sa + Sb) + N * (Za + Zb) + 8.0 * N * N
    return per_sweep * np.asarray(iters, np.float64)


def pair_smem_bytes(N, iters, word: int = 8) -> np.ndarray:
    N = np.asarray(N, np.float64)
    return 2.0 * N * N * word * np.asarray(iters, np.float64)


def triangle_units(n_nodes: np.ndarray):
    """Units of the size-sorted upper triangle, as the library enumerates them
    (sorted by n descending, stable): returns (perm, a_idx, b_idx)."""
    n_nodes = np.asarray(n_nodes)
    perm = np.argsort(-n_nodes, kind="stable")
    k = len(n_nodes)
    a = np.repeat(np.arange(k), np.arange(k, 0, -1))
    row_start = np.concatenate([[0], np.cumsum(np.arange(k, 0, -1))])
    b = a + (np.arange(len(a)) - row_start[a])
    return perm, a, b


def side_stats(m, N: int) -> tuple[int, int]:
    """(S, z) of one graph at common size N: nonzeros outside uniform rows and
    the number of uniform (all-zero) rows of interpolate_to(m, N)."""
    e = np.asarray(getattr(m, "entries", m), float)
    a = _interp_pattern(e, N) != 0
    return int(a.sum()), int((~a.any(axis=1)).sum())
