"""The benchmark corpora's matrices are the reference pipeline's matrices.

``synth.transition_matrix`` (the seeded generator behind every bench config)
must equal, bit for bit, what the reference produces for the same CFG
structure: listing -> ``build_cfg`` -> ``attribute_profile`` ->
``transition_matrix`` (golden vectors from ``tests/golden/make_synth.py``,
240 shapes over the three edge-weighting modes and 1..96 blocks).  When the
reference tree is present the pipeline is also run live on fresh shapes.
"""

from __future__ import annotations

import os

import numpy as np
import pytest

from conftest import GOLDEN, load_golden, unravel


def test_synth_matches_reference_golden():
    import importlib.util
    spec = importlib.util.spec_from_file_location("make_synth", GOLDEN / "make_synth.py")
    ms = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(ms)
    from paper_1707_02423_b200 import synth
    g = load_golden("synth_ref.npz")
    ref = unravel(g["sizes"], g["flat"])
    shapes = ms.shapes()
    assert len(shapes) == len(ref)
    modes = set()
    for s, r in zip(shapes, ref):
        got = synth.transition_matrix(s)
        assert got.shape == r.shape
        np.testing.assert_array_equal(got, r)
        modes.add("observed" if s.edge_counts is not None else ("sampled" if s.block_counts else "static"))
    assert modes == {"observed", "sampled", "static"}


@pytest.mark.skipif(not os.path.isdir("/root/reference/pkg/src/sasscfg"), reason="reference tree not present")
def test_synth_matches_reference_live():
    import sys
    sys.path.insert(0, "/root/reference/pkg/src")
    import importlib.util
    spec = importlib.util.spec_from_file_location("make_synth", GOLDEN / "make_synth.py")
    ms = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(ms)
    from paper_1707_02423_b200 import synth
    rng = np.random.default_rng(99)
    for i in range(60):
        wt = ("sampled", "observed", "static")[i % 3]
        s = synth.random_shape(rng, int(rng.integers(1, 70)), wt)
        np.testing.assert_array_equal(synth.transition_matrix(s), ms.reference_matrix(s))
