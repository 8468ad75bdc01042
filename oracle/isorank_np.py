"""numpy restatement of the reference IsoRank path — TEST INFRASTRUCTURE ONLY.

Follows ``/root/reference/pkg/src/sasscfg`` operation by operation; the only
change is the Kronecker mat-vec (``similarity.py:133,140``), replaced by the
mathematically identical two-product form ``A'^T X B'``.  Inputs are plain
square float64 arrays (the ``TransitionMatrix.entries`` of the reference,
``matrix.py:24-42``).
"""

from __future__ import annotations

import numpy as np


def interpolate_to(src: np.ndarray, target_n: int) -> np.ndarray:
    """Bilinear upscale; ``matrix.py:74-106`` (identity when n == target)."""
    n = src.shape[0]
    if target_n < n:
        raise ValueError("target smaller than source")
    if target_n == n:
        return src
    if n == 1:  # matrix.py:87-89
        return np.full((target_n, target_n), float(src[0, 0]))
    pos = (np.arange(target_n) * (n - 1)) / (target_n - 1)  # matrix.py:93
    lo = np.minimum(np.floor(pos).astype(int), n - 2)  # :94
    frac = pos - lo  # :95
    v00 = src[np.ix_(lo, lo)]
    v01 = src[np.ix_(lo, lo + 1)]
    v10 = src[np.ix_(lo + 1, lo)]
    v11 = src[np.ix_(lo + 1, lo + 1)]
    fr = frac[:, None]
    fc = frac[None, :]
    return (1 - fr) * ((1 - fc) * v00 + fc * v01) + fr * ((1 - fc) * v10 + fc * v11)  # :104


def normalize_pair(a: np.ndarray, b: np.ndarray) -> tuple[np.ndarray, np.ndarray]:
    """``matrix.py:109-114``."""
    if a.shape[0] == b.shape[0]:
        return a, b
    target = max(a.shape[0], b.shape[0])
    return interpolate_to(a, target), interpolate_to(b, target)


def row_normalized(entries: np.ndarray) -> np.ndarray:
    """``similarity.py:85-93``: row-stochastic copy, zero rows -> 1/n."""
    n = entries.shape[0]
    out = np.array(entries, dtype=float)
    sums = out.sum(axis=1)
    zero = sums == 0
    out[zero] = 1.0 / n
    out[~zero] = out[~zero] / sums[~zero, None]
    return out


def greedy_matching(matrix: np.ndarray) -> tuple[int, ...]:
    """``similarity.py:96-108``: repeated global argmax, ties -> lowest
    row-major index; the taken row and column are set to -1."""
    n = matrix.shape[0]
    work = matrix.copy()
    match: dict[int, int] = {}
    for _ in range(n):
        flat = int(np.argmax(work))
        row, col = divmod(flat, n)
        match[row] = col
        work[row, :] = -1.0
        work[:, col] = -1.0
    return tuple(match[i] for i in range(n))


def isorank_align(a, b, alpha=0.85, tol=1e-9, max_iter=1000, start=None):
    """``similarity.py:111-157`` with ``kron_t @ x`` -> ``A'^T X B'``.

    Returns (matrix, matching, matched_weight, iterations, converged).
    """
    a = np.asarray(a, dtype=float)
    b = np.asarray(b, dtype=float)
    if a.shape[0] != b.shape[0]:
        raise ValueError("dimension mismatch")
    if not 0.0 < alpha < 1.0:
        raise ValueError("alpha out of range")
    n = a.shape[0]
    ap = row_normalized(a)
    bp = row_normalized(b)
    uniform = np.full(n * n, 1.0 / (n * n))  # :134
    x = uniform.copy() if start is None else np.asarray(start, dtype=float) / np.sum(start)  # :135
    converged = False
    iterations = 0
    for iterations in range(1, max_iter + 1):  # :139
        kx = (ap.T @ x.reshape(n, n) @ bp).ravel()  # == kron(ap, bp).T @ x
        fresh = alpha * kx + (1.0 - alpha) * uniform  # :140
        fresh /= fresh.sum()  # :141
        delta = float(np.abs(fresh - x).sum())  # :142
        x = fresh
        if delta < tol:  # :144
            converged = True
            break
    matrix = x.reshape(n, n)
    matching = greedy_matching(matrix)
    weight = float(sum(matrix[i, matching[i]] for i in range(n)))  # :150
    return matrix, matching, weight, iterations, converged


def isorank_distance_from(weight: float, n: int) -> float:
    """``similarity.py:160-173``."""
    if n == 1:
        concentration = 1.0
    else:
        concentration = (weight - 1.0 / n) / (1.0 - 1.0 / n)
        concentration = min(1.0, max(0.0, concentration))
    return 1.0 + (1.0 - concentration)


def measure_iso(a, b, alpha=0.85, tol=1e-9, max_iter=1000):
    """``similarity.py:176-189`` ISO branch: returns (d, W, iterations, converged)."""
    a, b = normalize_pair(np.asarray(a, float), np.asarray(b, float))
    _, _, w, it, conv = isorank_align(a, b, alpha, tol, max_iter)
    return isorank_distance_from(w, a.shape[0]), w, it, conv
