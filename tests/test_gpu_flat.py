"""Flat measures (similarity.py:29-66) on the GPU against
the reference's own outputs (tests/golden/make_flat.py) and its pinned cases
(test_similarity.py:43-129).  Values agree up to summation order (1e-12
relative); errors map to the reference's exception types.
"""

from __future__ import annotations

import numpy as np
import pytest

from conftest import load_golden, unravel

pytestmark = pytest.mark.gpu

NAMES = {"euc": ("euc", 3.0), "man": ("man", 3.0), "min": ("min", 3.0), "jac": ("jac", 3.0), "cos": ("cos", 3.0),
         "min1": ("min", 1.0), "min15": ("min", 1.5), "min7": ("min", 7.0)}


@pytest.fixture(scope="module")
def P(gpu):
    import paper_1707_02423_b200 as P
    return P


def mat(P, e):
    e = np.asarray(e, float)
    return P.TransitionMatrix("x.f.t.m", e, tuple(range(len(e))), P.RAW_COUNTS)


@pytest.mark.parametrize("name", list(NAMES))
def test_flat_pairs_against_reference(P, name):
    g = load_golden("flat.npz")
    A, B = unravel(g["sa"], g["fa"]), unravel(g["sb"], g["fb"])
    mid, p = NAMES[name]
    ref = g[f"pairs_{name}"]
    for i, (a, b) in enumerate(zip(A, B)):
        if np.isnan(ref[i]):
            with pytest.raises(P.DegenerateInput):
                P.measure_distance(mat(P, a), mat(P, b), P.MeasureId(mid), p=p)
        else:
            got = P.measure_distance(mat(P, a), mat(P, b), P.MeasureId(mid), p=p)
            assert got == pytest.approx(ref[i], rel=1e-12, abs=1e-13), (i, a.shape, b.shape)


@pytest.mark.parametrize("name", list(NAMES))
def test_flat_pairwise_bundled_corpus(P, name):
    g = load_golden("bundled_corpus.npz")
    f = load_golden("flat.npz")
    mats = unravel(g["sizes"], g["flat"])
    tms = [P.TransitionMatrix(str(k), m, tuple(range(len(m))), P.ROW_STOCHASTIC) for k, m in zip(g["ids"], mats)]
    mid, p = NAMES[name]
    pm = P.pairwise(tms[::-1], P.MeasureId(mid), p=p)
    assert pm.kernel_ids == tuple(str(x) for x in g["ids"])
    np.testing.assert_allclose(pm.scores, f[f"bundled_{name}"], rtol=1e-12, atol=1e-14)
    assert (np.diag(pm.scores) == 0).all()


def test_flat_pinned_cases(P):  # test_similarity.py:43-129
    ca, cb = mat(P, [[1.0, 0.0], [0.0, 1.0]]), mat(P, [[0.0, 1.0], [1.0, 0.0]])
    assert P.euclidean(ca, cb) == 2.0
    assert P.manhattan(ca, cb) == 4.0
    assert P.minkowski(ca, cb, 3.0) == pytest.approx(4.0 ** (1.0 / 3.0))
    assert P.manhattan(mat(P, [[0.3]]), mat(P, [[0.8]])) == pytest.approx(0.5, abs=1e-12)
    for p in (0.99, 0.0, -3.0):
        with pytest.raises(P.BadOrder):
            P.minkowski(ca, cb, p)
    assert P.jaccard(mat(P, [[1.0]]), mat(P, [[1.0]])) == 0.0
    assert P.jaccard(ca, cb) == pytest.approx(1.0)
    assert P.jaccard(mat(P, [[2.0]]), mat(P, [[1.0]])) == pytest.approx(1.0 / 3.0)
    with pytest.raises(P.DegenerateInput):
        P.jaccard(mat(P, [[0.0]]), mat(P, [[0.0]]))
    assert P.jaccard(mat(P, [[0.0]]), mat(P, [[2.0]])) == pytest.approx(1.0)
    a = mat(P, [[1.0, 2.0], [0.0, 1.0]])
    assert P.cosine(a, a) == pytest.approx(0.0, abs=1e-12)
    assert P.cosine(a, mat(P, 2.0 * np.asarray(a.entries))) == pytest.approx(0.0, abs=1e-12)
    assert P.cosine(ca, cb) == pytest.approx(1.0)
    with pytest.raises(P.DegenerateInput):
        P.cosine(mat(P, [[0.0]]), mat(P, [[1.0]]))
    for f in (P.euclidean, P.manhattan, P.minkowski, P.jaccard, P.cosine):
        with pytest.raises(P.DimMismatch):
            f(mat(P, [[1.0]]), ca)


def test_flat_pairwise_nan_and_large(P):
    """Undefined pairs become NaN inside pairwise (similarity.py:243-254);
    sizes past the on-chip tiers (N up to 600) against an fp64 numpy restatement."""
    from oracle.isorank_np import normalize_pair
    rng = np.random.default_rng(9)
    ms = [np.zeros((3, 3)), rng.random((40, 40)), rng.random((5, 5)) * (rng.random((5, 5)) < 0.5),
          rng.random((600, 600)) * (rng.random((600, 600)) < 0.01), np.zeros((7, 7))]
    tms = [P.TransitionMatrix(f"g{i}.f.t.x", m, tuple(range(len(m))), P.RAW_COUNTS) for i, m in enumerate(ms)]
    pm = P.pairwise(tms, P.MeasureId.COS)
    assert np.isnan(pm.scores[0, 1]) and np.isnan(pm.scores[1, 4])  # cosine with an all-zero side
    pj = P.pairwise(tms, P.MeasureId.JAC)
    assert np.isnan(pj.scores[0, 4]) and np.isfinite(pj.scores[0, 1])  # two all-zero matrices
    pe = P.pairwise(tms, P.MeasureId.EUC)
    for i in range(len(ms)):
        for j in range(len(ms)):
            if i == j:
                continue
            x, y = normalize_pair(ms[i], ms[j])
            assert pe.scores[i, j] == pytest.approx(np.sqrt(np.sum((x - y) ** 2)), rel=1e-12)
    pn = P.pairwise(tms, P.MeasureId.MIN, p=0.5)
    assert np.isnan(pn.scores[~np.eye(len(ms), dtype=bool)]).all()


@pytest.mark.parametrize("p", [3.0, 1.5, 0.5])
def test_pairwise_all_one_pass_equals_per_measure(P, p):
    """`compare --measure all` (cli.py:150-165) through pairwise_all: the five
    flat matrices from one kernel pass are bitwise the per-measure pairwise()
    outputs (same sums, same order), ISO equals pairwise(ISO); the bundled
    corpus also matches the reference's own matrices (p = 3)."""
    from paper_1707_02423_b200 import synth
    g = load_golden("bundled_corpus.npz")
    mats = unravel(g["sizes"], g["flat"]) + synth.random_corpus(30, 3, 90, seed=4)
    tms = [P.TransitionMatrix(f"k{i:03d}.a.b", m, tuple(range(len(m))), P.ROW_STOCHASTIC) for i, m in enumerate(mats)]
    allm = P.pairwise_all(tms, p=p)
    assert list(allm) == list(P.MeasureId)
    for m, pm in allm.items():
        ref = P.pairwise(tms, m, p=p)
        assert pm.kernel_ids == ref.kernel_ids and pm.measure is m
        np.testing.assert_array_equal(pm.scores, ref.scores)
    if p == 3.0:
        f = load_golden("flat.npz")
        six = P.pairwise_all(tms[:len(g["ids"])], measures=["euc", "man", "min", "jac", "cos"])
        for mid in ("euc", "man", "min", "jac", "cos"):
            tm = [P.TransitionMatrix(str(k), m, tuple(range(len(m))), P.ROW_STOCHASTIC)
                  for k, m in zip(g["ids"], unravel(g["sizes"], g["flat"]))]
            np.testing.assert_allclose(P.pairwise_all(tm, measures=[mid])[P.MeasureId(mid)].scores,
                                       f[f"bundled_{mid}"], rtol=1e-12, atol=1e-14)
        assert len(six) == 5
