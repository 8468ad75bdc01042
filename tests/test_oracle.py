"""The CPU oracle is pinned against vectors produced by the reference itself.

tests/golden/*.npz come from tests/golden/make_golden.py (imports sasscfg
from /root/reference).  Both restatements (numpy, C) must reproduce the
reference's iteration counts exactly and its distances to rounding.
"""

from __future__ import annotations

import numpy as np
import pytest

from conftest import load_golden, unravel
from oracle import ffi
from oracle import isorank_np as onp


@pytest.fixture(scope="module")
def small():
    g = load_golden("small_pairs.npz")
    return g, unravel(g["sa"], g["fa"]), unravel(g["sb"], g["fb"])


def test_numpy_oracle_small_pairs(small):
    g, A, B = small
    for i, (a, b) in enumerate(zip(A, B)):
        d, w, it, cv = onp.measure_iso(a, b)
        assert it == g["iters"][i]
        assert cv == g["converged"][i]
        assert d == pytest.approx(g["d"][i], rel=1e-13, abs=1e-13)
        assert w == pytest.approx(g["W"][i], rel=1e-12, abs=1e-14)


def test_c_oracle_small_pairs_full_outputs(small):
    g, A, B = small
    X = unravel(g["sx"], g["fx"])
    moff = 0
    for i, (a, b) in enumerate(zip(A, B)):
        r = ffi.iso_pair(a, b)
        n = X[i].shape[0]
        assert r["iterations"] == g["iters"][i]
        assert r["converged"] == g["converged"][i]
        assert r["d"] == pytest.approx(g["d"][i], rel=1e-13, abs=1e-13)
        np.testing.assert_allclose(r["X"], X[i], rtol=1e-11, atol=1e-15)
        assert sorted(r["matching"]) == list(range(n))
        moff += n


def test_c_oracle_synthetic_cfg_pairs():
    g = load_golden("synth_pairs.npz")
    A, B = unravel(g["sa"], g["fa"]), unravel(g["sb"], g["fb"])
    for i, (a, b) in enumerate(zip(A, B)):
        r = ffi.iso_pair(a, b)
        assert r["iterations"] == g["iters"][i], i
        assert r["d"] == pytest.approx(g["d"][i], rel=1e-12)
        assert r["W"] == pytest.approx(g["W"][i], rel=1e-10)


def test_c_oracle_bundled_corpus_matrix():
    g = load_golden("bundled_corpus.npz")
    mats = unravel(g["sizes"], g["flat"])
    k = len(mats)
    for i in range(k):
        for j in range(k):
            r = ffi.iso_pair(mats[i], mats[j])
            assert r["iterations"] == g["iters"][i, j]
            assert r["d"] == pytest.approx(g["scores"][i, j], rel=1e-13)


def test_survey_golden_row():
    """first row and diagonal of the bundled ISO matrix."""
    g = load_golden("bundled_corpus.npz")
    first = [1.397629669, 1.872506457, 1.681899622, 1.872646839, 1.422185389, 1.879503139]
    diag = [1.397629669, 1.883695058, 1.399621565, 1.883326303, 1.440593526, 1.886062611]
    np.testing.assert_allclose(g["scores"][0], first, atol=1e-9)
    np.testing.assert_allclose(np.diag(g["scores"]), diag, atol=1e-9)


def test_c_oracle_batch_matches_single():
    g = load_golden("synth_pairs.npz")
    mats = unravel(g["sa"], g["fa"])[:8] + unravel(g["sb"], g["fb"])[:8]
    from paper_1707_02423_b200.packing import pack
    packed = pack(mats)
    ia = np.arange(8, dtype=np.int32)
    ib = ia + 8
    d, w, it, cv = ffi.iso_batch(packed, ia, ib, threads=4)
    np.testing.assert_array_equal(it, g["iters"][:8])
    np.testing.assert_allclose(d, g["d"][:8], rtol=1e-12)


def test_oracle_special_cases():
    s = load_golden("special.npz")
    r = ffi.iso_pair(np.zeros((1, 1)), np.zeros((1, 1)))
    np.testing.assert_array_equal(r["X"], s["singleton_X"])
    assert r["iterations"] == s["singleton_iters"] == 1
    r = ffi.iso_pair(np.zeros((3, 3)), np.zeros((3, 3)))
    assert r["matching"] == tuple(s["zeros_match"]) == (0, 1, 2)
    r = ffi.iso_pair(s["start_a"], s["start_b"], start=s["start_vec"])
    np.testing.assert_allclose(r["X"], s["start_X"], rtol=1e-11)
    assert r["iterations"] == s["start_iters"]
    for c in range(1, 8):
        r = ffi.iso_pair(s["cut_a"], s["cut_b"], max_iter=c)
        assert r["iterations"] == c
        np.testing.assert_allclose(r["X"], s["cut_X"][c - 1], rtol=1e-12)


def test_oracle_interpolation_bit_exact():
    g = load_golden("interp.npz")
    srcs, outs = unravel(g["ss"], g["fs"]), unravel(g["so"], g["fo"])
    for src, t, out in zip(srcs, g["targets"], outs):
        np.testing.assert_array_equal(onp.interpolate_to(src, int(t)), out)
