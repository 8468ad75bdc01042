"""Golden vectors for the flat measures from the
reference itself.  Run in the build container:

    python tests/golden/make_flat.py

Writes tests/golden/flat.npz: for each of euc/man/min(p=3)/jac/cos, the
reference's pairwise() scores over the bundled corpus (kernel_id order, from
bundled_corpus.npz) and measure_distance() over random raw matrices of
unequal sizes 1..12 (incl. all-zero ones: NaN where the reference raises
DegenerateInput), plus minkowski at p = 1, 1.5, 7.
"""

from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, "/root/reference/pkg/src")

from sasscfg import similarity as S  # noqa: E402
from sasscfg.errors import SasscfgError  # noqa: E402
from sasscfg.matrix import RAW_COUNTS, ROW_STOCHASTIC, TransitionMatrix  # noqa: E402

MEASURES = [("euc", S.MeasureId.EUC, 3.0), ("man", S.MeasureId.MAN, 3.0), ("min", S.MeasureId.MIN, 3.0),
            ("jac", S.MeasureId.JAC, 3.0), ("cos", S.MeasureId.COS, 3.0), ("min1", S.MeasureId.MIN, 1.0),
            ("min15", S.MeasureId.MIN, 1.5), ("min7", S.MeasureId.MIN, 7.0)]


def main():
    g = np.load(HERE / "bundled_corpus.npz")
    sizes, flat, ids = g["sizes"], g["flat"], g["ids"]
    mats, o = [], 0
    for n in sizes:
        n = int(n)
        mats.append(flat[o:o + n * n].reshape(n, n))
        o += n * n
    tms = [TransitionMatrix(str(k), m, tuple(range(len(m))), ROW_STOCHASTIC) for k, m in zip(ids, mats)]
    out = {}
    for name, mid, p in MEASURES:
        out[f"bundled_{name}"] = S.pairwise(tms, mid, p=p).scores
    rng = np.random.default_rng(1707)
    A, B = [], []
    for t in range(160):
        na, nb = int(rng.integers(1, 13)), int(rng.integers(1, 13))
        a = rng.random((na, na)) * (rng.random((na, na)) < 0.6)
        b = rng.random((nb, nb)) * (rng.random((nb, nb)) < 0.6)
        if t % 23 == 0:
            a[:] = 0.0
        if t % 31 == 0:
            b[:] = 0.0
        A.append(a)
        B.append(b)
    for name, mid, p in MEASURES:
        vals = []
        for a, b in zip(A, B):
            ta = TransitionMatrix("a.x.y.z", a, tuple(range(len(a))), RAW_COUNTS)
            tb = TransitionMatrix("b.x.y.z", b, tuple(range(len(b))), RAW_COUNTS)
            try:
                vals.append(S.measure_distance(ta, tb, mid, p=p))
            except SasscfgError:
                vals.append(np.nan)
        out[f"pairs_{name}"] = np.array(vals)
    out["sa"] = np.array([len(a) for a in A], np.int32)
    out["fa"] = np.concatenate([a.ravel() for a in A])
    out["sb"] = np.array([len(b) for b in B], np.int32)
    out["fb"] = np.concatenate([b.ravel() for b in B])
    np.savez_compressed(HERE / "flat.npz", **out)
    print({k: v.shape for k, v in out.items()})


if __name__ == "__main__":
    main()
