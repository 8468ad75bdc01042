#!/usr/bin/env python
"""Measure the per-unit device cost of an all-pairs alignment as a function of
N = max(n_a, n_b), for the multi-GPU split's cost model (csrc/cost_model.h).

  python tools/calibrate_split.py [--graphs 20000] [--out gpurun_out/cost.json]

Corpus: the c5 distribution (16-512 blocks).  For N > 64 a random sample of
pairs with that N (rows of size N, partners of any smaller size — the mix a
row of the triangle sees) through ``isorank_pairs`` (the same kernels as the
all-pairs ranges); for N <= 64 contiguous unit slices of the row group through
``cfgsim_allpairs_range`` (the two-stage path), two slice lengths to separate
the group's fixed stage-1 cost.  Device time by CUDA events.
"""

from __future__ import annotations

import argparse
import json
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--graphs", type=int, default=20000)
    ap.add_argument("--pairs", type=int, default=3000)
    ap.add_argument("--out", default="gpurun_out/cost.json")
    a = ap.parse_args()
    import torch

    import paper_1707_02423_b200 as P
    from paper_1707_02423_b200 import _native as nat
    from paper_1707_02423_b200 import synth
    t0 = time.time()
    mats = synth.random_corpus(a.graphs, 16, 512, seed=2, weighting="sampled")
    n = np.array([len(m) for m in mats])
    print(f"corpus {a.graphs} graphs in {time.time() - t0:.1f} s", flush=True)
    rng = np.random.default_rng(0)
    prm = nat.params(0.85, 1e-9, 1000, "fp64")
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    res = {}
    with P.DeviceCorpus(mats) as C:
        st = torch.cuda.current_stream().cuda_stream
        # every sampled N: allpairs_range over whole rows of that N's row group
        # (a row's partners are all smaller graphs: the mix the triangle has)
        order = np.argsort(-n, kind="stable")
        ns = n[order]
        k = len(n)
        rs = np.concatenate([[0], np.cumsum(np.arange(k, 0, -1))])
        out = torch.empty(k * 60 + 1, dtype=torch.float64, device="cuda")  # >= units of one row group (~k * rows)
        for N in sorted(set(list(range(16, 513, 24)) + [32, 33, 48, 64, 65, 72, 96, 97, 120, 128, 129, 160, 192, 256, 257, 384, 512])):
            grp = np.flatnonzero(ns == N)
            if len(grp) == 0:
                continue
            # whole row groups: the large-N path's history mode (shared
            # sequences) applies per group, so a partial group would be
            # timed on the per-pair path instead
            budget = 1 << 62
            r1 = grp[0]
            while r1 + 1 <= grp[-1] and rs[r1 + 1] - rs[grp[0]] < budget:
                r1 += 1
            u0, u1 = int(rs[grp[0]]), int(rs[r1 + 1])
            ts = []
            for rep in range(2):
                torch.cuda.synchronize()
                ev0.record()
                nat.check(nat.lib.cfgsim_allpairs_range(C.handle, u0, u1, 0, nat.C.byref(prm), nat.ptr(out), None, st))
                ev1.record()
                torch.cuda.synchronize()
                ts.append(ev0.elapsed_time(ev1) * 1e3 / (u1 - u0))
            res[N] = {"us_per_unit": min(ts), "reps": [round(t, 4) for t in ts], "units": u1 - u0,
                      "rows": int(r1 - grp[0] + 1)}
            print(N, res[N], flush=True)
    Path(a.out).parent.mkdir(parents=True, exist_ok=True)
    Path(a.out).write_text(json.dumps({"graphs": a.graphs, "costs": {str(k): v for k, v in sorted(res.items())}},
                                      indent=1))
    print("wrote", a.out)


if __name__ == "__main__":
    main()
