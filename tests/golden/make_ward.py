"""Golden vectors for Ward linkage from the reference
itself (cluster.py:88-134).  Run in the build container:

    python tests/golden/make_ward.py

Writes tests/golden/ward.npz: float feature sets (random spreads, integer
grids that provoke distance ties, duplicated points) and the reference's
merges (a, b, distance, size).
"""

from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, "/root/reference/pkg/src")

from sasscfg.cluster import FeatureVector, ward_linkage  # noqa: E402


def main():
    rng = np.random.default_rng(88)
    sets = []
    for t in range(40):
        k = int(rng.integers(2, 60)) if t < 36 else int(rng.integers(150, 260))
        dim = int(rng.integers(1, 12))
        if t % 3 == 0:
            x = rng.integers(0, 4, (k, dim)).astype(float)  # ties
        elif t % 3 == 1:
            x = rng.random((k, dim)) * 10
        else:
            x = rng.random((k, dim))
            x[rng.integers(0, k, k // 4)] = x[0]  # duplicates
        sets.append(x)
    sizes, dims, flat, merges, offs = [], [], [], [], [0]
    for x in sets:
        vs = [FeatureVector(f"k{i:04d}.w.t.x", tuple(float(v) for v in row)) for i, row in enumerate(x)]
        lk = ward_linkage(vs)
        sizes.append(x.shape[0])
        dims.append(x.shape[1])
        flat.append(x.ravel())
        merges.extend(lk.merges)
        offs.append(len(merges))
    m = np.array(merges, dtype=object)
    np.savez_compressed(HERE / "ward.npz", sizes=np.array(sizes, np.int32), dims=np.array(dims, np.int32),
                        flat=np.concatenate(flat), ma=np.array([r[0] for r in merges], np.int64),
                        mb=np.array([r[1] for r in merges], np.int64), md=np.array([r[2] for r in merges]),
                        ms=np.array([r[3] for r in merges], np.int64), offs=np.array(offs, np.int64))
    print(len(sets), "sets,", len(merges), "merges")


if __name__ == "__main__":
    main()
