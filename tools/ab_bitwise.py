#!/usr/bin/env python
"""Dump the all-pairs ISO scores + iterations of a fixed corpus with the
library selected by CFGSIM_LIBRARY, to check two builds for bitwise-equal
results (A/B of a kernel change that must not change arithmetic).

  CFGSIM_LIBRARY=... python tools/ab_bitwise.py c4|c5|c2 out.npz [--graphs K]
  python tools/ab_bitwise.py cmp a.npz b.npz
"""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

if sys.argv[1] == "cmp":
    a, b = np.load(sys.argv[2]), np.load(sys.argv[3])
    same_s = np.array_equal(a["scores"], b["scores"])
    same_i = np.array_equal(a["iters"], b["iters"])
    print(f"scores bitwise equal: {same_s}; iterations equal: {same_i}; "
          f"max |diff| {np.nanmax(np.abs(a['scores'] - b['scores'])):.3e}")
    sys.exit(0 if same_s and same_i else 1)

import paper_1707_02423_b200 as P
from paper_1707_02423_b200 import synth

cfg, out = sys.argv[1], sys.argv[2]
k = int(sys.argv[4]) if len(sys.argv) > 4 else {"c2": 300, "c4": 60, "c5": 200}[cfg]
c = synth.CONFIGS[cfg]
mats = synth.random_corpus(k, c["lo"], c["hi"], seed=7, weighting=c["weighting"])
tms = [P.TransitionMatrix(f"k{i:05d}.s.ab", m, tuple(range(len(m))), P.ROW_STOCHASTIC) for i, m in enumerate(mats)]
pm, it = P.pairwise(tms, P.MeasureId.ISO, return_iterations=True)
np.savez(out, scores=np.array(pm.scores), iters=it)
print(f"{cfg}: {k} graphs -> {out}")
