"""Ward linkage on the GPU (cluster.py:88-134) against
the reference's own merges (tests/golden/make_ward.py): identical merge
order, ids and sizes, bitwise-equal distances (same double arithmetic)."""

from __future__ import annotations

import numpy as np
import pytest

from conftest import load_golden

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def C(gpu):
    from paper_1707_02423_b200 import cluster as C
    return C


def test_ward_matches_reference(C):
    g = load_golden("ward.npz")
    off = 0
    for t, (k, dim) in enumerate(zip(g["sizes"], g["dims"])):
        x = g["flat"][off:off + k * dim].reshape(k, dim)
        off += k * dim
        vs = [C.FeatureVector(f"k{i:04d}.w.t.x", tuple(row)) for i, row in enumerate(x)]
        lk = C.ward_linkage(vs)
        lo, hi = g["offs"][t], g["offs"][t + 1]
        ref = list(zip(g["ma"][lo:hi].tolist(), g["mb"][lo:hi].tolist(), g["md"][lo:hi].tolist(),
                       g["ms"][lo:hi].tolist()))
        assert list(lk.merges) == ref, t


def test_ward_errors_and_cuts(C):  # test_cluster.py pinned behaviour
    with pytest.raises(ValueError):
        C.ward_linkage([C.FeatureVector("a.w.t.x", (0.0,))])
    with pytest.raises(C.DimMismatch if hasattr(C, "DimMismatch") else Exception):
        C.ward_linkage([C.FeatureVector("a.w.t.x", (0.0, 1.0)), C.FeatureVector("b.w.t.x", (0.0,))])
    line = [C.FeatureVector(f"p{i}.w.t.x", (float(v),)) for i, v in enumerate((0, 1, 5))]
    lk = C.ward_linkage(line)
    assert lk.merges[0][:2] == (0, 1) and lk.merges[0][2] == 1.0
    ids = [v.kernel_id for v in line]
    assert C.cut_clusters(lk, 2, ids) == {"p0.w.t.x": 0, "p1.w.t.x": 0, "p2.w.t.x": 1}
    with pytest.raises(C.BadK):
        C.cut_clusters(lk, 0, ids)
    assert C.export_linkage_csv(lk).startswith("a,b,distance,size\n0,1,1,2\n")


def test_ward_large_is_fast_and_valid(C):
    rng = np.random.default_rng(5)
    x = rng.random((3000, 8))
    lk = C.ward_linkage([C.FeatureVector(f"k{i:05d}.w.t.x", tuple(r)) for i, r in enumerate(x)])
    d = np.array([m[2] for m in lk.merges])
    assert len(lk.merges) == 2999 and lk.merges[-1][3] == 3000
    assert (np.diff(d) >= -1e-12 * d[1:]).all()  # Ward merge distances are monotone (reducible linkage)
