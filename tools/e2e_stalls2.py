#!/usr/bin/env python
"""Where a stalled C2 e2e call loses its time: per phase of pairwise (corpus
build, all-pairs call, result wrap) the wall time, the main thread's CPU time,
its voluntary / involuntary context switches and page faults (getrusage)."""
import gc
import resource
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1707_02423_b200 as P  # noqa: E402
from paper_1707_02423_b200 import _native as nat, synth  # noqa: E402
from paper_1707_02423_b200.corpus import DeviceCorpus  # noqa: E402

mats = synth.random_corpus(2000, 16, 64, seed=2)
tms = [P.TransitionMatrix(f"k{i:05d}.synth.c2", m, tuple(range(len(m))), P.ROW_STOCHASTIC) for i, m in enumerate(mats)]
P.pairwise(tms, P.MeasureId.ISO)


def snap():
    r = resource.getrusage(resource.RUSAGE_THREAD)
    return time.perf_counter(), r.ru_utime + r.ru_stime, r.ru_nvcsw, r.ru_nivcsw, r.ru_minflt, r.ru_majflt


def d(a, b):
    return f"{1e3*(b[0]-a[0]):7.1f}ms cpu {1e3*(b[1]-a[1]):6.1f} vcs {b[2]-a[2]:3d} ivcs {b[3]-a[3]:3d} flt {b[4]-a[4]:5d}/{b[5]-a[5]}"


keep = []
for rep in range(16):
    gc.collect()
    torch.cuda.synchronize()
    s0 = snap()
    ordered = sorted(tms, key=lambda m: m.kernel_id)
    k = len(ordered)
    scores = nat.pinned_array((k, k))
    C = DeviceCorpus(ordered, 0)
    s1 = snap()
    prm = nat.params()
    nat.check(nat.lib.cfgsim_allpairs(C.handle, 0, nat.C.byref(prm), nat.ptr(scores), None, None))
    s2 = snap()
    C.close()
    keep = [scores]
    s3 = snap()
    print(f"rep {rep:2d}: corpus {d(s0, s1)} | allpairs {d(s1, s2)} | close {d(s2, s3)}", flush=True)
