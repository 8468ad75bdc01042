"""IsoRank pair similarity — drop-in for the reference's ISO path.

Same names, signatures, defaults and error behaviour as
``pkg/src/sasscfg/similarity.py``; every alignment runs in the sm_100a
kernel (``csrc/isorank.cuh``) through the C ABI (``include/cfgsim.h``).

Additions (keyword-only, defaults reproduce the reference):
  precision="fp64"|"fp32"   fp64 reproduces the reference; fp32 stops on
                            delta < max(tol, tol_fp32)
  symmetric=True            pairwise ISO: one alignment per unordered pair,
                            d(j,i) := d(i,j) (ISO is symmetric);
                            False runs both directions like the reference
  device=None               GPU ordinal (default: LOCAL_RANK or 0)
and ``nearest`` (query-vs-corpus best match, no reference equivalent).

The five flat measures (euc/man/min/jac/cos, similarity.py:29-66) run on the
GPU too (``csrc/flat.cuh``): same values up to summation
order, same errors (DimMismatch, BadOrder, DegenerateInput; NaN inside
``pairwise``).
"""

from __future__ import annotations

from dataclasses import dataclass
from enum import Enum
from typing import Sequence

import numpy as np

from . import _native as nat
from .corpus import DeviceCorpus, pack
from .errors import BadOrder, DegenerateInput, DimMismatch, DuplicateKernel
from .matrix import TransitionMatrix


class MeasureId(str, Enum):
    EUC = "euc"
    ISO = "iso"
    MAN = "man"
    MIN = "min"
    JAC = "jac"
    COS = "cos"


@dataclass(frozen=True)
class AlignmentResult:
    """Node-pair alignment between two equal-size graphs (``similarity.py:69-82``)."""

    matrix: np.ndarray
    matching: tuple[int, ...]
    matched_weight: float
    iterations: int
    converged: bool


@dataclass(frozen=True)
class PairwiseMatrix:
    measure: MeasureId
    kernel_ids: tuple[str, ...]
    scores: np.ndarray
    scaled: bool = False


def _dev(device):
    return nat.default_device() if device is None else int(device)


def _check_alpha(alpha: float) -> None:
    if not 0.0 < alpha < 1.0:  # similarity.py:129-130
        raise ValueError(f"alpha must be in (0, 1), got {alpha}")


def _flat(a: TransitionMatrix, b: TransitionMatrix, measure: str, p: float = 3.0, device=None) -> float:
    """One flat measure on the GPU after normalize_pair (measure_distance's order)."""
    A = np.ascontiguousarray(a.entries, dtype=np.float64)
    B = np.ascontiguousarray(b.entries, dtype=np.float64)
    out = np.empty(1)
    nat.check(nat.lib.cfgsim_flat_single(_dev(device), a.n, nat.ptr(A), b.n, nat.ptr(B), nat.FLAT_IDS[measure],
                                         float(p), nat.ptr(out)))
    return float(out[0])


def _same_size(a: TransitionMatrix, b: TransitionMatrix) -> None:
    if a.n != b.n:  # similarity.py:29-32
        raise DimMismatch(f"matrix dimensions differ: {a.n} vs {b.n}")


def euclidean(a: TransitionMatrix, b: TransitionMatrix) -> float:
    """``sqrt(sum |x - y|^2)`` over the flattened entries (similarity.py:35-37)."""
    _same_size(a, b)
    return _flat(a, b, "euc")


def manhattan(a: TransitionMatrix, b: TransitionMatrix) -> float:
    """``sum |x - y|`` (similarity.py:40-42)."""
    _same_size(a, b)
    return _flat(a, b, "man")


def minkowski(a: TransitionMatrix, b: TransitionMatrix, p: float = 3.0) -> float:
    """``(sum |x - y|^p)^(1/p)``, p >= 1 else BadOrder (similarity.py:45-49)."""
    if p < 1:
        raise BadOrder(f"order p must be >= 1, got {p}")
    _same_size(a, b)
    return _flat(a, b, "min", p)


def jaccard(a: TransitionMatrix, b: TransitionMatrix) -> float:
    """``sum (x-y)^2 / (x.x + y.y - x.y)``; DegenerateInput for two zero matrices (similarity.py:52-57)."""
    _same_size(a, b)
    return _flat(a, b, "jac")


def cosine(a: TransitionMatrix, b: TransitionMatrix) -> float:
    """``1 - x.y / (|x| |y|)``; DegenerateInput for a zero matrix (similarity.py:60-66)."""
    _same_size(a, b)
    return _flat(a, b, "cos")


def isorank_align(a: TransitionMatrix, b: TransitionMatrix, alpha: float = 0.85, tol: float = 1e-9,
                  max_iter: int = 1000, start: np.ndarray | None = None, *, precision: str = "fp64",
                  device: int | None = None) -> AlignmentResult:
    """Damped power iteration on the Kronecker product (``similarity.py:111-157``)."""
    if a.n != b.n:
        raise DimMismatch(f"matrix dimensions differ: {a.n} vs {b.n}")
    _check_alpha(alpha)
    n = a.n
    x0 = None
    if start is not None:  # similarity.py:135
        x0 = np.ascontiguousarray(np.asarray(start, dtype=float) / np.sum(start), dtype=np.float64)
        if x0.size != n * n:
            raise DimMismatch(f"start vector has {x0.size} entries, expected {n * n}")
    A = np.ascontiguousarray(a.entries, dtype=np.float64)
    B = np.ascontiguousarray(b.entries, dtype=np.float64)
    X = np.empty((n, n))
    m = np.empty(n, np.int32)
    d = np.empty(1)
    w = np.empty(1)
    it = np.empty(1, np.int32)
    cv = np.empty(1, np.uint8)
    prm = nat.params(alpha, tol, max_iter, precision)
    nat.check(nat.lib.cfgsim_isorank_single(_dev(device), n, nat.ptr(A), n, nat.ptr(B), nat.C.byref(prm),
                                            nat.ptr(x0), nat.ptr(X), nat.ptr(m), nat.ptr(d), nat.ptr(w),
                                            nat.ptr(it), nat.ptr(cv)))
    return AlignmentResult(matrix=X, matching=tuple(int(v) for v in m), matched_weight=float(w[0]),
                           iterations=int(it[0]), converged=bool(cv[0]))


def isorank_distance(alignment: AlignmentResult) -> float:
    """Distance in [1, 2] from the matched weight (``similarity.py:160-173``)."""
    n = alignment.matrix.shape[0]
    if n == 1:
        return 1.0
    conc = (alignment.matched_weight - 1.0 / n) / (1.0 - 1.0 / n)
    conc = min(1.0, max(0.0, conc))
    return 1.0 + (1.0 - conc)


def measure_distance(a: TransitionMatrix, b: TransitionMatrix, measure: MeasureId, *, p: float = 3.0,
                     alpha: float = 0.85, tol: float = 1e-9, max_iter: int = 1000,
                     precision: str = "fp64", device: int | None = None) -> float:
    """Size-normalise a pair and apply one measure (``similarity.py:176-200``).

    For ISO the size normalisation (``normalize_pair``) is fused into the
    kernel prologue."""
    if measure is not MeasureId.ISO:
        if measure not in tuple(MeasureId):
            raise ValueError(f"unknown measure {measure!r}")
        if measure is MeasureId.MIN and p < 1:
            raise BadOrder(f"order p must be >= 1, got {p}")
        return _flat(a, b, measure.value, p, device)  # normalize_pair fused (similarity.py:187-199)
    _check_alpha(alpha)
    A = np.ascontiguousarray(a.entries, dtype=np.float64)
    B = np.ascontiguousarray(b.entries, dtype=np.float64)
    d = np.empty(1)
    prm = nat.params(alpha, tol, max_iter, precision)
    nat.check(nat.lib.cfgsim_isorank_single(_dev(device), a.n, nat.ptr(A), b.n, nat.ptr(B), nat.C.byref(prm),
                                            None, None, None, nat.ptr(d), None, None, None))
    return float(d[0])


def pairwise(matrices: list[TransitionMatrix], measure: MeasureId, *, p: float = 3.0, alpha: float = 0.85,
             tol: float = 1e-9, max_iter: int = 1000, precision: str = "fp64", symmetric: bool = True,
             device: int | None = None, return_iterations: bool = False):
    """All-pairs scores ordered by kernel_id (``similarity.py:211-257``).

    ISO fills the diagonal and both directions.  The whole corpus is packed
    and uploaded once; all alignments run in persistent sm_100a kernels.

    ``symmetric=True`` (default) aligns each unordered pair once, in the
    (lower kernel index, higher) direction, and mirrors it; the reference
    aligns both directions (similarity.py:240-246), which agree to 4.4e-16
    relative with identical iteration counts (pinned on the
    bundled corpus by tests/test_gpu_parity.py).  ``symmetric=False``
    evaluates every ordered pair exactly as the reference does (2x work)."""
    if len(matrices) < 2:
        raise ValueError("pairwise comparison needs at least 2 kernels")
    ordered = sorted(matrices, key=lambda m: m.kernel_id)
    ids = tuple(m.kernel_id for m in ordered)
    if len(set(ids)) != len(ids):
        raise DuplicateKernel("duplicate kernel_id in pairwise input")
    if measure not in tuple(MeasureId):
        raise ValueError(f"unknown measure {measure!r}")
    k = len(ordered)
    if measure is not MeasureId.ISO:
        # symmetric, zero diagonal, NaN where the measure fails (similarity.py:247-255)
        scores = np.empty((k, k))
        with DeviceCorpus(ordered, _dev(device)) as corpus:
            nat.check(nat.lib.cfgsim_flat_allpairs(corpus.handle, nat.FLAT_IDS[measure.value], float(p),
                                                   nat.ptr(scores), None))
        pm = PairwiseMatrix(measure=measure, kernel_ids=ids, scores=scores, scaled=False)
        return (pm, None) if return_iterations else pm
    _check_alpha(alpha)
    scores = nat.pinned_array((k, k))
    iters = np.empty((k, k), np.int32) if return_iterations else None
    prm = nat.params(alpha, tol, max_iter, precision)
    with DeviceCorpus(ordered, _dev(device)) as corpus:
        nat.check(nat.lib.cfgsim_allpairs(corpus.handle, 0 if symmetric else 1, nat.C.byref(prm),
                                          nat.ptr(scores), nat.ptr(iters), None))
    pm = PairwiseMatrix(measure=measure, kernel_ids=ids, scores=scores, scaled=False)
    return (pm, iters) if return_iterations else pm


def pairwise_all(matrices: list[TransitionMatrix], measures=None, *, p: float = 3.0, alpha: float = 0.85,
                 tol: float = 1e-9, max_iter: int = 1000, precision: str = "fp64", symmetric: bool = True,
                 device: int | None = None) -> dict:
    """``pairwise`` for several measures at once — what ``sasscfg compare
    --measure all`` computes (cli.py:150-165: one ``pairwise`` per measure).
    Returns {MeasureId: PairwiseMatrix}, each equal to ``pairwise(matrices,
    measure, ...)``.  The corpus is packed and uploaded once; the five flat
    measures come from ONE kernel pass over each pair's size-normalised
    entries (``cfgsim_flat_all_allpairs``) instead of five; ISO runs the
    IsoRank kernels on the same device corpus."""
    if measures is None:
        measures = tuple(MeasureId)
    measures = tuple(MeasureId(m) for m in measures)
    if len(matrices) < 2:
        raise ValueError("pairwise comparison needs at least 2 kernels")
    ordered = sorted(matrices, key=lambda m: m.kernel_id)
    ids = tuple(m.kernel_id for m in ordered)
    if len(set(ids)) != len(ids):
        raise DuplicateKernel("duplicate kernel_id in pairwise input")
    k = len(ordered)
    out = {}
    flat = [m for m in measures if m is not MeasureId.ISO]
    with DeviceCorpus(ordered, _dev(device)) as corpus:
        if flat:
            mats5 = np.empty((5, k, k))
            nat.check(nat.lib.cfgsim_flat_all_allpairs(corpus.handle, float(p), nat.ptr(mats5), None))
            for m in flat:
                out[m] = PairwiseMatrix(measure=m, kernel_ids=ids, scores=mats5[nat.FLAT_IDS[m.value]].copy(),
                                        scaled=False)
        if MeasureId.ISO in measures:
            _check_alpha(alpha)
            scores = np.empty((k, k))
            prm = nat.params(alpha, tol, max_iter, precision)
            nat.check(nat.lib.cfgsim_allpairs(corpus.handle, 0 if symmetric else 1, nat.C.byref(prm),
                                              nat.ptr(scores), None, None))
            out[MeasureId.ISO] = PairwiseMatrix(measure=MeasureId.ISO, kernel_ids=ids, scores=scores, scaled=False)
    return {m: out[m] for m in measures}


def minmax_scale(pm: PairwiseMatrix) -> PairwiseMatrix:
    """Affine rescale to [0, 1] over finite entries (``similarity.py:260-284``);
    ISO's diagonal takes part, the flat measures' zero diagonal does not."""
    k = pm.scores.shape[0]
    mask = np.isfinite(pm.scores)
    if pm.measure is not MeasureId.ISO:
        mask &= ~np.eye(k, dtype=bool)
    picked = pm.scores[mask]
    if picked.size == 0:
        raise DegenerateInput("no finite entries to scale")
    lo, hi = float(picked.min()), float(picked.max())
    out = pm.scores.copy()
    out[mask] = 0.0 if hi == lo else (pm.scores[mask] - lo) / (hi - lo)
    return PairwiseMatrix(measure=pm.measure, kernel_ids=pm.kernel_ids, scores=out, scaled=True)


def export_heatmap_csv(pm: PairwiseMatrix, *, native: bool | None = None) -> str:
    """CSV, kernel_id header row/column, 6 decimals, ``nan`` (``similarity.py:287-293``).

    Large matrices (K >= 64, or native=True) are formatted by the library's
    multi-threaded writer (``cfgsim_heatmap_csv``), byte-identical to the
    Python formatting below."""
    k = len(pm.kernel_ids)
    if native or (native is None and k >= 64):
        enc = [kid.encode() for kid in pm.kernel_ids]
        ids = np.frombuffer(b"".join(enc), np.uint8) if enc else np.zeros(0, np.uint8)
        off = np.zeros(k + 1, np.int64)
        off[1:] = np.cumsum([len(e) for e in enc])
        sc = np.ascontiguousarray(pm.scores, dtype=np.float64)
        n = np.zeros(1, np.int64)
        nat.check(nat.lib.cfgsim_heatmap_csv(k, nat.ptr(ids), nat.ptr(off), nat.ptr(sc), None, 0, nat.ptr(n), 0))
        buf = np.empty(int(n[0]), np.uint8)
        nat.check(nat.lib.cfgsim_heatmap_csv(k, nat.ptr(ids), nat.ptr(off), nat.ptr(sc), nat.ptr(buf), int(n[0]),
                                             nat.ptr(n), 0))
        return buf.tobytes().decode()
    header = "," + ",".join(pm.kernel_ids)
    body = [
        kid + "," + ",".join(f"{v:.6f}" if np.isfinite(v) else "nan" for v in row)
        for kid, row in zip(pm.kernel_ids, pm.scores)
    ]
    return "\n".join([header, *body]) + "\n"


def nearest(queries: Sequence[TransitionMatrix], corpus: Sequence[TransitionMatrix], *, alpha: float = 0.85,
            tol: float = 1e-9, max_iter: int = 1000, precision: str = "fp64",
            device: int | None = None) -> tuple[np.ndarray, np.ndarray]:
    """Best match of every query in ``corpus``: ``argmin_j measure_distance(q,
    corpus[j], ISO)``, ties to the lowest j.  Returns (best_d, best_index)."""
    _check_alpha(alpha)
    dev = _dev(device)
    nq = len(queries)
    best_d = np.empty(nq)
    best_i = np.empty(nq, np.int64)
    prm = nat.params(alpha, tol, max_iter, precision)
    with DeviceCorpus(queries, dev) as Q, DeviceCorpus(corpus, dev) as Cc:
        nat.check(nat.lib.cfgsim_nearest(Q.handle, Cc.handle, 0, Cc.K, nat.C.byref(prm), nat.ptr(best_d),
                                         nat.ptr(best_i), None))
    return best_d, best_i


def isorank_pairs(A: DeviceCorpus, B: DeviceCorpus, ia, ib, *, alpha: float = 0.85, tol: float = 1e-9,
                  max_iter: int = 1000, precision: str = "fp64", stream=None):
    """Batched ``measure_distance(A[ia[p]], B[ib[p]], ISO)``: returns (d, W, iters, converged)."""
    _check_alpha(alpha)
    ia = np.ascontiguousarray(ia, np.int32)
    ib = np.ascontiguousarray(ib, np.int32)
    n = len(ia)
    d = np.empty(n)
    w = np.empty(n)
    it = np.empty(n, np.int32)
    cv = np.empty(n, np.uint8)
    prm = nat.params(alpha, tol, max_iter, precision)
    nat.check(nat.lib.cfgsim_isorank_pairs(A.handle, B.handle, n, nat.ptr(ia), nat.ptr(ib), nat.C.byref(prm),
                                           nat.ptr(d), nat.ptr(w), nat.ptr(it), nat.ptr(cv), stream))
    return d, w, it, cv.astype(bool)
