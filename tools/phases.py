#!/usr/bin/env python
"""Per-phase cycle shares of the stage-2 / large-N kernels (CFGSIM_PHASES=1 debug
accounting), eager all-pairs over a bench corpus.

  CFGSIM_PHASES=1 python tools/phases.py c2|c4|c5 [--graphs K] 2> phases.log
"""
from __future__ import annotations

import argparse
import os
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("config", choices=["c2", "c4", "c5"])
    ap.add_argument("--graphs", type=int, default=None)
    a = ap.parse_args()
    os.environ.setdefault("CFGSIM_PHASES", "1")
    import paper_1707_02423_b200 as P
    from paper_1707_02423_b200 import synth
    lo, hi, wt, k = {"c2": (16, 64, "sampled", 2000), "c4": (256, 1024, "observed", 100),
                     "c5": (16, 512, "sampled", 1000)}[a.config]
    mats = synth.random_corpus(a.graphs or k, lo, hi, seed=2, weighting=wt)
    tms = [P.TransitionMatrix(f"k{i:05d}.s.p", m, tuple(range(len(m))), P.ROW_STOCHASTIC) for i, m in enumerate(mats)]
    t = time.time()
    P.pairwise(tms, P.MeasureId.ISO)
    print(f"{a.config}: {len(mats)} graphs, wall {time.time() - t:.2f} s", flush=True)


if __name__ == "__main__":
    main()
