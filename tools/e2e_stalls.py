#!/usr/bin/env python
"""Host stalls in the C2 e2e path: times 10 pairwise(..., ISO) calls and reads
the cgroup CPU quota / throttling counters around them (cpu.max, cpu.stat)."""
import gc
import os
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

import paper_1707_02423_b200 as P  # noqa: E402
from paper_1707_02423_b200 import synth  # noqa: E402


def cg(name):
    for base in ("/sys/fs/cgroup", "/sys/fs/cgroup/cpu"):
        p = Path(base) / name
        if p.exists():
            return p.read_text().strip().replace("\n", "; ")
    return "n/a"


print("affinity", len(os.sched_getaffinity(0)), "cpu.max", cg("cpu.max"), "| torch threads", torch.get_num_threads(),
      "| loadavg", open("/proc/loadavg").read().strip(), flush=True)
mats = synth.random_corpus(2000, 16, 64, seed=2)
tms = [P.TransitionMatrix(f"k{i:05d}.synth.c2", m, tuple(range(len(m))), P.ROW_STOCHASTIC) for i, m in enumerate(mats)]
res = P.pairwise(tms, P.MeasureId.ISO)
res = P.pairwise(tms, P.MeasureId.ISO)
print("cpu.stat before", cg("cpu.stat"), flush=True)
ts = []
for s in range(10):
    gc.collect()
    torch.cuda.synchronize()
    c0 = time.process_time()
    t0 = time.perf_counter()
    res = P.pairwise(tms, P.MeasureId.ISO)
    ts.append((round(1e3 * (time.perf_counter() - t0), 1), round(1e3 * (time.process_time() - c0), 1)))
print("cpu.stat after ", cg("cpu.stat"), flush=True)
print("steps (wall ms, process cpu ms):", ts, flush=True)
