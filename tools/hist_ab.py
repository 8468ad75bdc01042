#!/usr/bin/env python
"""All-pairs device time of a corpus with many graphs per size (large-N
history-mode A/B): CFGSIM_BIG_HIST=0|1 python tools/hist_ab.py K lo hi"""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

import paper_1707_02423_b200 as P  # noqa: E402
from paper_1707_02423_b200 import _native as nat, synth  # noqa: E402

k, lo, hi = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
mats = synth.random_corpus(k, lo, hi, seed=5)
prm = nat.params()
with P.DeviceCorpus(mats) as C:
    nu = C.n_units()
    d = torch.empty(nu, dtype=torch.float64, device="cuda")
    it = torch.empty(nu, dtype=torch.int32, device="cuda")
    st = torch.cuda.current_stream().cuda_stream
    ts = []
    for rep in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        nat.check(nat.lib.cfgsim_allpairs_range(C.handle, 0, nu, 0, nat.C.byref(prm), nat.ptr(d), nat.ptr(it), st))
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    print(f"K={k} n in [{lo},{hi}] units={nu} ms={[round(t, 1) for t in ts]} pairs/s={nu / min(ts) * 1e3:.0f} "
          f"checksum={float(d.sum()):.17g} iters={int(it.sum())}")
