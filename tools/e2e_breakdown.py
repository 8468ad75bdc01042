#!/usr/bin/env python
"""Where the e2e time of pairwise(..., ISO) goes on C2 (host-side wall
clock around each stage, device synchronised between stages)."""
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

import paper_1707_02423_b200 as P  # noqa: E402
from paper_1707_02423_b200 import _native as nat, synth  # noqa: E402
from paper_1707_02423_b200.corpus import DeviceCorpus  # noqa: E402

mats = synth.random_corpus(2000, 16, 64, seed=2)
tms = [P.TransitionMatrix(f"k{i:05d}.synth.c2", m, tuple(range(len(m))), P.ROW_STOCHASTIC) for i, m in enumerate(mats)]
P.pairwise(tms, P.MeasureId.ISO)
for rep in range(5):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    ordered = sorted(tms, key=lambda m: m.kernel_id)
    t1 = time.perf_counter()
    C = DeviceCorpus(ordered, 0)
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    k = len(ordered)
    scores = nat.pinned_array((k, k))
    prm = nat.params()
    nat.check(nat.lib.cfgsim_allpairs(C.handle, 0, nat.C.byref(prm), nat.ptr(scores), None, None))
    t3 = time.perf_counter()
    C.close()
    t4 = time.perf_counter()
    pm = P.pairwise(tms, P.MeasureId.ISO)
    t5 = time.perf_counter()
    print(f"sort {1e3*(t1-t0):.2f} corpus {1e3*(t2-t1):.2f} allpairs {1e3*(t3-t2):.2f} close {1e3*(t4-t3):.2f} "
          f"| pairwise() {1e3*(t5-t4):.2f} ms", flush=True)
