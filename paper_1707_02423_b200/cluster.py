"""Ward-linkage clustering downstream of the distances.

Same names and behaviour as ``pkg/src/sasscfg/cluster.py``: ``FeatureVector``,
``Linkage``, ``ward_linkage`` (on the GPU: ``csrc/ward.cuh``, exact — the
reference's double arithmetic and tie rule, O(K^2) instead of O(K^3)),
``cut_clusters`` and the CSV exports (host).  Feature values are fp64 (the
reference also accepts exact ``Fraction`` inputs; here they are converted).
"""

from __future__ import annotations

import math
from dataclasses import dataclass
from typing import Sequence

import numpy as np

from . import _native as nat
from .errors import BadK, DimMismatch


@dataclass(frozen=True)
class FeatureVector:
    """Fixed-order grouping features for one kernel (cluster.py:21-37)."""

    kernel_id: str
    values: tuple[float, ...]
    norms: tuple[int, int] = (1, 1)

    def __post_init__(self) -> None:
        for v in self.values:
            if not math.isfinite(float(v)):
                raise ValueError(f"non-finite feature value {v!r} for {self.kernel_id}")


@dataclass(frozen=True)
class Linkage:
    """Merge history: leaves 0..n-1, merged clusters n..2n-2; rows
    (cluster_a, cluster_b, distance, size) with cluster_a < cluster_b
    (cluster.py:66-84)."""

    merges: tuple[tuple[int, int, float, int], ...]
    n_leaves: int

    def __post_init__(self) -> None:
        if len(self.merges) != self.n_leaves - 1:
            raise ValueError(f"expected {self.n_leaves - 1} merges, got {len(self.merges)}")
        used: set[int] = set()
        for a, b, dist, size in self.merges:
            if dist < 0:
                raise ValueError(f"negative merge distance {dist}")
            if a in used or b in used:
                raise ValueError(f"cluster {a if a in used else b} merged twice")
            used.update((a, b))


def ward_linkage(vectors: Sequence[FeatureVector], *, device: int | None = None) -> Linkage:
    """Ward's minimum-variance agglomeration (cluster.py:88-134): squared
    Euclidean start, Lance-Williams updates, ties to the smallest (id_a, id_b)."""
    n = len(vectors)
    if n < 2:
        raise ValueError("clustering needs at least 2 vectors")
    dim = len(vectors[0].values)
    for v in vectors:
        if len(v.values) != dim:
            raise DimMismatch(f"feature length {len(v.values)} != {dim} for {v.kernel_id}")
    F = np.ascontiguousarray(np.array([[float(x) for x in v.values] for v in vectors], dtype=np.float64)
                             .reshape(n, dim))
    a = np.empty(n - 1, np.int64)
    b = np.empty(n - 1, np.int64)
    d = np.empty(n - 1)
    s = np.empty(n - 1, np.int64)
    dev = nat.default_device() if device is None else int(device)
    nat.check(nat.lib.cfgsim_ward(dev, n, dim, nat.ptr(F), nat.ptr(a), nat.ptr(b), nat.ptr(d), nat.ptr(s)))
    merges = tuple((int(a[i]), int(b[i]), float(d[i]), int(s[i])) for i in range(n - 1))
    return Linkage(merges=merges, n_leaves=n)


def cut_clusters(linkage: Linkage, k: int, ids: Sequence[str]) -> dict[str, int]:
    """Flat clustering after the first n - k merges (cluster.py:130-145):
    cluster indices are assigned in increasing order of each cluster's
    smallest leaf.

    Union-find over the leaves: merged cluster n + s owns the representative
    of its two parts, so each merge is two finds and one link."""
    n = linkage.n_leaves
    if not 1 <= k <= n:
        raise BadK(f"cluster count {k} outside 1..{n}")
    if len(ids) != n:
        raise DimMismatch(f"{len(ids)} ids for {n} leaves")
    parent = list(range(n))
    rep = list(range(n)) + [0] * (n - 1)  # cluster id -> one leaf of it

    def find(x: int) -> int:
        while parent[x] != x:
            parent[x] = parent[parent[x]]
            x = parent[x]
        return x

    for s in range(n - k):
        a, b = linkage.merges[s][0], linkage.merges[s][1]
        ra, rb = find(rep[a]), find(rep[b])
        lo, hi = (ra, rb) if ra < rb else (rb, ra)
        parent[hi] = lo  # the root is always the smallest leaf of its cluster
        rep[n + s] = lo
    roots = sorted({find(x) for x in range(n)})
    index = {r: i for i, r in enumerate(roots)}
    return {ids[x]: index[find(x)] for x in range(n)}


def export_linkage_csv(linkage: Linkage) -> str:
    """``a,b,distance,size`` rows, distance as %.6g (cluster.py:201-205)."""
    rows = ["a,b,distance,size"] + [f"{a},{b},{float(d):.6g},{s}" for a, b, d, s in linkage.merges]
    return "\n".join(rows) + "\n"


def export_clusters_csv(assignment: dict[str, int]) -> str:
    """``kernel_id,cluster`` rows sorted by kernel_id (cluster.py:208-212)."""
    rows = ["kernel_id,cluster"] + [f"{kid},{assignment[kid]}" for kid in sorted(assignment)]
    return "\n".join(rows) + "\n"
