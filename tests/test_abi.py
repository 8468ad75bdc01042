"""CPU checks of the boundary: the C-ABI library loads and exports every
symbol include/cfgsim.h declares, and host-side logic (packing, errors)
behaves like the reference.  No compute calls (no GPU here)."""

from __future__ import annotations

import re
import subprocess

import numpy as np
import pytest

from conftest import REPO


def declared_symbols():
    text = (REPO / "include" / "cfgsim.h").read_text()
    return sorted(set(re.findall(r"\b(cfgsim_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    from paper_1707_02423_b200 import _native
    lib = _native.LIB_PATH
    out = subprocess.run(["nm", "-D", "--defined-only", str(lib)], capture_output=True, text=True, check=True).stdout
    exported = set(re.findall(r"\bT (cfgsim_\w+)", out))
    decl = declared_symbols()
    assert decl, "no declarations parsed"
    missing = [s for s in decl if s not in exported]
    assert not missing, missing
    for s in decl:
        assert hasattr(_native.lib, s)
    assert set(_native.EXPORTED) == set(decl)


def test_library_is_sm100a_only():
    from paper_1707_02423_b200 import _native
    out = subprocess.run(["cuobjdump", "--list-elf", str(_native.LIB_PATH)], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    assert "sm_90" not in out and "sm_80" not in out


def test_version_and_device_count_without_gpu():
    from paper_1707_02423_b200 import _native
    assert _native.lib.cfgsim_version() == 100
    assert _native.device_count() >= 0


def test_no_cpu_fallback_without_gpu():
    from paper_1707_02423_b200 import _native
    if _native.device_count() > 0:
        pytest.skip("a GPU is present")
    import paper_1707_02423_b200 as P
    m = P.TransitionMatrix("a.s.t.x", np.eye(3), (0, 1, 2), P.RAW_COUNTS)
    with pytest.raises(P.DeviceError):
        P.measure_distance(m, m, P.MeasureId.ISO)
    with pytest.raises(P.DeviceError):
        P.DeviceCorpus([np.eye(3)])


def test_pack_layout():
    from paper_1707_02423_b200.packing import pack
    a = np.array([[0.0, 0.5], [1.0, 0.0]])
    b = np.array([[0.25, 0.0, 0.75], [0.0, 0.0, 0.0], [0.0, 1.0, 0.0]])
    p = pack([a, b])
    assert p["n_nodes"].tolist() == [2, 3]
    assert p["rp_off"].tolist() == [0, 3]
    assert p["nz_off"].tolist() == [0, 2]
    assert p["rowptr"].tolist() == [0, 1, 2, 0, 2, 2, 3]
    assert p["col"].tolist() == [1, 0, 0, 2, 1]
    assert p["val"].tolist() == [0.5, 1.0, 0.25, 0.75, 1.0]


def test_host_side_reference_semantics():
    import paper_1707_02423_b200 as P
    with pytest.raises(ValueError):
        P.pairwise([P.TransitionMatrix("a", np.eye(1), (0,), P.RAW_COUNTS)], P.MeasureId.ISO)
    with pytest.raises(P.DuplicateKernel):
        P.pairwise([P.TransitionMatrix("a", np.eye(1), (0,), P.RAW_COUNTS)] * 2, P.MeasureId.ISO)
    with pytest.raises(P.DimMismatch):
        P.isorank_align(P.TransitionMatrix("a", np.eye(1), (0,), P.RAW_COUNTS),
                        P.TransitionMatrix("b", np.eye(2), (0, 1), P.RAW_COUNTS))
    with pytest.raises(ValueError):
        P.TransitionMatrix("a", -np.eye(2), (0, 1), P.RAW_COUNTS)
    m = P.TransitionMatrix("a", np.eye(2), (0, 1), P.RAW_COUNTS)
    assert P.interpolate_to(m, 2) is m
    with pytest.raises(P.BadTarget):
        P.interpolate_to(m, 1)


def test_minmax_and_csv_match_reference_semantics():
    import paper_1707_02423_b200 as P
    ids = ("k0.s.t.h", "k1.s.t.h")
    pm = P.PairwiseMatrix(P.MeasureId.ISO, ids, np.array([[1.0, 1.5], [1.5, 2.0]]))
    np.testing.assert_allclose(P.minmax_scale(pm).scores, [[0.0, 0.5], [0.5, 1.0]])  # test_similarity.py:344-346
    pm = P.PairwiseMatrix(P.MeasureId.EUC, ids, np.array([[0.0, 1.0 / 3.0], [np.nan, 0.0]]))
    assert P.export_heatmap_csv(pm).splitlines() == [",k0.s.t.h,k1.s.t.h", "k0.s.t.h,0.000000,0.333333",
                                                     "k1.s.t.h,nan,0.000000"]
    with pytest.raises(P.DegenerateInput):
        P.minmax_scale(P.PairwiseMatrix(P.MeasureId.EUC, ids, np.array([[0.0, np.nan], [np.nan, 0.0]])))


def test_native_csv_writer_byte_identical():
    """cfgsim_heatmap_csv (host code, runs without a GPU) against the
    reference's formatting (similarity.py:287-293) and its golden bytes."""
    import paper_1707_02423_b200 as P
    from conftest import GOLDEN, load_golden
    rng = np.random.default_rng(12)
    for k in (1, 2, 65, 300):
        sc = rng.random((k, k)) * 2.0
        sc[rng.random((k, k)) < 0.02] = np.nan
        if k > 1:
            sc[0, 1], sc[1, 0] = np.inf, -0.0
        sc[0, 0] = 0.0000005  # half-way cases round on the exact binary value
        ids = tuple(f"k{i:04d}.k.x.y" for i in range(k))
        pm = P.PairwiseMatrix(P.MeasureId.ISO, ids, sc)
        assert P.export_heatmap_csv(pm, native=True) == P.export_heatmap_csv(pm, native=False)
    g = load_golden("bundled_corpus.npz")
    pm = P.PairwiseMatrix(P.MeasureId.ISO, tuple(str(x) for x in g["ids"]), g["scores"])
    assert P.export_heatmap_csv(pm, native=True) == (GOLDEN / "iso.csv").read_text()


def test_corpus_data_pointers():
    """DeviceCorpus reads ndarray data addresses from the array objects
    (corpus._data_pointers); they must equal numpy's own, views included."""
    import numpy as np
    from paper_1707_02423_b200.corpus import _data_pointers
    base = np.arange(64.0).reshape(8, 8)
    arrs = [np.zeros((3, 3)), base[2:5, 2:5].copy(), np.ascontiguousarray(base[1:]), base[4:], np.ones((1, 1))]
    assert _data_pointers(arrs) == [a.__array_interface__["data"][0] for a in arrs]
    assert _data_pointers([]) == []
