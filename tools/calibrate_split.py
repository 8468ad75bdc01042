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
        # large / mid N: random pairs (row graph of size N, partner uniformly among n <= N)
        for N in list(range(72, 513, 24)) + [65, 96, 128, 129, 160, 256, 257, 384, 512]:
            rows = np.flatnonzero(n == N)
            parts = np.flatnonzero(n <= N)
            if len(rows) == 0:
                continue
            npairs = a.pairs if N > 128 else 4 * a.pairs
            ia = rng.choice(rows, npairs).astype(np.int32)
            ib = rng.choice(parts, npairs).astype(np.int32)
            best = None
            for rep in range(2):
                torch.cuda.synchronize()
                ev0.record()
                P.isorank_pairs(C, C, ia, ib)
                ev1.record()
                torch.cuda.synchronize()
                t = ev0.elapsed_time(ev1) * 1e3 / npairs
                best = t if best is None else min(best, t)
            res[N] = {"us_per_unit": best, "how": "isorank_pairs sample", "pairs": npairs}
            print(N, res[N], flush=True)
        # small N: two-stage ranges over the row group
        order = np.argsort(-n, kind="stable")
        ns = n[order]
        k = len(n)
        rs = np.concatenate([[0], np.cumsum(np.arange(k, 0, -1))])
        out = torch.empty(400000, dtype=torch.float64, device="cuda")
        for N in (16, 24, 32, 40, 48, 56, 64):
            grp = np.flatnonzero(ns == N)
            if len(grp) == 0:
                continue
            u0 = int(rs[grp[0]])
            uend = int(rs[grp[-1] + 1])
            ts = []
            for U in (100000, 200000):
                U = min(U, uend - u0)
                best = None
                for rep in range(2):
                    torch.cuda.synchronize()
                    ev0.record()
                    nat.check(nat.lib.cfgsim_allpairs_range(C.handle, u0, u0 + U, 0, nat.C.byref(prm), nat.ptr(out),
                                                            None, st))
                    ev1.record()
                    torch.cuda.synchronize()
                    t = ev0.elapsed_time(ev1) * 1e3
                    best = t if best is None else min(best, t)
                ts.append((U, best))
            (U1, t1), (U2, t2) = ts
            per = (t2 - t1) / (U2 - U1) if U2 > U1 else t2 / U2
            res[N] = {"us_per_unit": per, "fixed_us": t1 - per * U1, "how": "allpairs_range slices", "units": [U1, U2]}
            print(N, res[N], flush=True)
    Path(a.out).parent.mkdir(parents=True, exist_ok=True)
    Path(a.out).write_text(json.dumps({"graphs": a.graphs, "costs": {str(k): v for k, v in sorted(res.items())}},
                                      indent=1))
    print("wrote", a.out)


if __name__ == "__main__":
    main()
