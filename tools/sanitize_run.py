#!/usr/bin/env python
"""One reduced run of a benchmark path, for compute-sanitizer (tools/sanitize.sh).

  python tools/sanitize_run.py c2|c3|c4|c3small [--graphs K] [--queries Q]

c2: all-pairs over K graphs of 16-64 blocks (two-stage path: stage-1
four-combo + one-combo kernels, stage-2 kernel, scatter); c3: Q queries x K
corpus best match (the query-vs-corpus rectangles, including the stage-2
kernel running right before each stage 1); c3small: the same with every graph
below 32 blocks (the case that exposed the stale list-offset read); c4: K
graphs of 256-1024 blocks with observed edge counts (large-N kernel).
Results are checked against the per-pair list path (bitwise) so a sanitizer
run is also a parity run.
"""

from __future__ import annotations

import argparse
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main() -> int:
    ap = argparse.ArgumentParser()
    ap.add_argument("config", choices=["c2", "c3", "c3small", "c4"])
    ap.add_argument("--graphs", type=int, default=None)
    ap.add_argument("--queries", type=int, default=None)
    a = ap.parse_args()
    import paper_1707_02423_b200 as P
    from paper_1707_02423_b200 import synth

    if a.config == "c2" or a.config == "c4":
        lo, hi, wt, k = (16, 64, "sampled", 160) if a.config == "c2" else (256, 1024, "observed", 6)
        k = a.graphs or k
        mats = synth.random_corpus(k, lo, hi, seed=2, weighting=wt)
        tms = [P.TransitionMatrix(f"k{i:05d}.s.{a.config}", m, tuple(range(len(m))), P.ROW_STOCHASTIC)
               for i, m in enumerate(mats)]
        pm = P.pairwise(tms, P.MeasureId.ISO)
        iu, ju = np.triu_indices(k)
        with P.DeviceCorpus(mats) as C:
            d, *_ = P.isorank_pairs(C, C, iu, ju)
        ok = np.array_equal(pm.scores[iu, ju], d)
        print(f"{a.config}: {len(iu)} alignments, triangle == list path bitwise: {ok}")
        return 0 if ok else 1
    lo, hi = (16, 64) if a.config == "c3" else (4, 31)
    nq, nc = a.queries or 100, a.graphs or 8000
    # a stage-2 launch first: it leaves its sentinels in shared memory
    warm = synth.random_corpus(24, 16, 64, seed=9)
    P.pairwise([P.TransitionMatrix(f"w{i:03d}.s.w", m, tuple(range(len(m))), P.ROW_STOCHASTIC)
                for i, m in enumerate(warm)], P.MeasureId.ISO)
    q = synth.random_corpus(nq, lo, hi, seed=3)
    c = synth.random_corpus(nc, lo, hi, seed=2)
    bd, bi = P.nearest(q, c)
    sub = np.random.default_rng(0).choice(nq, min(nq, 8), replace=False)
    with P.DeviceCorpus([q[i] for i in sub]) as CQ, P.DeviceCorpus(c) as CC:
        ia = np.repeat(np.arange(len(sub)), nc)
        ib = np.tile(np.arange(nc), len(sub))
        dl, *_ = P.isorank_pairs(CQ, CC, ia, ib)
    dl = dl.reshape(len(sub), nc)
    ok = np.array_equal(bd[sub], dl.min(axis=1)) and np.array_equal(bi[sub], dl.argmin(axis=1))
    print(f"{a.config}: {nq} x {nc} nearest; {len(sub)} queries checked against the list path bitwise: {ok}")
    return 0 if ok else 1


if __name__ == "__main__":
    sys.exit(main())
