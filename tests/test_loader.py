"""Native corpus loader (csrc/loader.cpp) against the
reference's own outputs (tests/golden/make_loader.py): identical entries
(bitwise) and ordering for every synthetic listing/profile/mode case, and the
reference's exception class, line number and message for every malformed
input.  Host code only: runs in the CPU suite.
"""

from __future__ import annotations

import gzip
import json
from pathlib import Path

import numpy as np
import pytest

GOLDEN = Path(__file__).resolve().parent / "golden" / "loader.json.gz"
REF_CORPUS = Path("/root/reference/pkg/corpus/manifest.txt")


@pytest.fixture(scope="module")
def L():
    from paper_1707_02423_b200 import loader
    return loader


@pytest.fixture(scope="module")
def cases():
    with gzip.open(GOLDEN, "rt") as f:
        return json.load(f)


def dense(exp):
    n = exp["n"]
    m = np.zeros((n, n))
    for i, j, h in exp["nz"]:
        m[i, j] = float.fromhex(h)
    return m


def check_case(L, c, got=None, err=None):
    exp = c["expect"]
    if "error" in exp:
        assert err is not None, (c["listing"][:200], c["profile"])
        assert type(err).__name__ == exp["error"], (type(err), err, exp)
        assert getattr(err, "line_no", 0) == exp["line"]
        assert (getattr(err, "reason", None) or str(err)) == exp["msg"]
    else:
        assert err is None, (err, c["listing"][:300], c["profile"])
        assert got.ordering == tuple(exp["ordering"])
        want = dense(exp)
        assert got.entries.shape == want.shape
        assert np.array_equal(got.entries.view(np.int64), want.view(np.int64)), c["kernel_id"]
        assert got.mode == c["mode"] and got.kernel_id == c["kernel_id"]


def test_loader_cases_one_by_one(L, cases):
    for c in cases:
        got = err = None
        try:
            (got,) = L.matrices_from_listings([(c["kernel_id"], c["listing"], c["profile"])], c["mode"], threads=1)
        except Exception as e:  # noqa: BLE001
            err = e
        check_case(L, c, got, err)


@pytest.mark.parametrize("mode", ["row_stochastic", "global", "raw_counts"])
def test_loader_batch_multithreaded(L, cases, mode):
    """All well-formed cases of one mode in one multi-threaded call."""
    good = [c for c in cases if "n" in c["expect"] and c["mode"] == mode]
    mats = L.matrices_from_listings([(c["kernel_id"], c["listing"], c["profile"]) for c in good], mode, threads=8)
    assert len(mats) == len(good)
    for c, m in zip(good, mats):
        check_case(L, c, m)


def test_loader_first_failure_in_input_order(L, cases):
    good = next(c for c in cases if "n" in c["expect"])
    bad = [c for c in cases if c["expect"].get("error") == "ListingSyntaxError"][:2]
    ks = [(good["kernel_id"], good["listing"], good["profile"])] + \
         [(c["kernel_id"], c["listing"], c["profile"]) for c in bad]
    with pytest.raises(Exception) as ei:
        L.matrices_from_listings(ks, good["mode"])
    check_case(L, bad[0], err=ei.value)


def test_loader_unknown_mode(L):
    with pytest.raises(ValueError):
        L.matrices_from_listings([("k", "/*0008*/ EXIT ;\n", None)], "interpolated")


def test_loader_manifest(L, tmp_path):
    """load_manifest / load_corpus_matrices (corpus.py:32-79, cli.py:77-89):
    paths relative to the manifest, sorted by kernel id, shared profile files."""
    (tmp_path / "l").mkdir()
    (tmp_path / "l" / "b.sass").write_text(".L_0:\n/*0008*/ @P0 BRA `(.L_0) ;\n/*0010*/ EXIT ;\n")
    (tmp_path / "l" / "a.sass").write_text("/*0008*/ NOP ;\n/*0010*/ EXIT ;\n")
    (tmp_path / "p.prof").write_text("kernel b.x\nedge .L_0 .L_0 3\nedge .L_0 B1 1\nkernel a.x\n")
    (tmp_path / "m.txt").write_text("# corpus\nb.x l/b.sass p.prof sm_100\na.x l/a.sass sm_100  # no profile\n")
    mats = L.load_corpus_matrices(tmp_path / "m.txt")
    assert [m.kernel_id for m in mats] == ["a.x", "b.x"]
    assert np.array_equal(mats[0].entries, [[0.0]])  # one block, its only edge goes to STOP
    assert np.array_equal(mats[1].entries, [[0.75, 0.25], [0.0, 0.0]])
    (tmp_path / "m2.txt").write_text("c.x l/missing.sass sm_100\n")
    from paper_1707_02423_b200.errors import CorpusError
    with pytest.raises(CorpusError, match="listing not readable"):
        L.load_corpus_matrices(tmp_path / "m2.txt")
    (tmp_path / "m3.txt").write_text("c.x l/a.sass p.prof sm_100\n")
    with pytest.raises(CorpusError, match=r"p\.prof has no profile for kernel 'c\.x'"):
        L.load_corpus_matrices(tmp_path / "m3.txt")


@pytest.mark.skipif(not REF_CORPUS.exists(), reason="reference corpus not present (GPU box)")
def test_loader_bundled_corpus(L):
    """The reference's bundled corpus (pkg/corpus) through the native loader
    equals bundled_corpus.npz, which the reference's own loader produced."""
    g = np.load(Path(__file__).resolve().parent / "golden" / "bundled_corpus.npz")
    mats = L.load_corpus_matrices(REF_CORPUS)
    assert [m.kernel_id for m in mats] == [str(x) for x in g["ids"]]
    o = 0
    for m, n in zip(mats, g["sizes"]):
        n = int(n)
        assert np.array_equal(m.entries, g["flat"][o:o + n * n].reshape(n, n))
        o += n * n
