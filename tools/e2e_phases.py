"""Where the e2e time of C2 goes (GPU box): corpus build, all-pairs call,
result, with CUDA syncs between phases.  python tools/e2e_phases.py"""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch
import bench
import paper_1707_02423_b200 as P
from paper_1707_02423_b200 import _native as nat
sys.argv = ["bench.py"]
args = bench.parse()
cfg, mats, _ = bench.corpus(args)
tms = [P.TransitionMatrix(f"k{i:05d}", m, tuple(range(len(m))), P.ROW_STOCHASTIC) for i, m in enumerate(mats)]
for rep in range(4):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    ordered = sorted(tms, key=lambda m: m.kernel_id)
    t1 = time.perf_counter()
    corp = P.DeviceCorpus(ordered, 0)
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    k = len(ordered)
    scores = np.empty((k, k))
    prm = nat.params()
    nat.check(nat.lib.cfgsim_allpairs(corp.handle, 0, nat.C.byref(prm), nat.ptr(scores), None, None))
    t3 = time.perf_counter()
    corp.close() if hasattr(corp, "close") else corp.__exit__(None, None, None)
    torch.cuda.synchronize()
    t4 = time.perf_counter()
    pm = P.pairwise(tms, P.MeasureId.ISO, device=0)
    t5 = time.perf_counter()
    print(f"rep {rep}: sort {1e3*(t1-t0):.1f} ms, corpus {1e3*(t2-t1):.1f} ms, allpairs->host {1e3*(t3-t2):.1f} ms, "
          f"destroy {1e3*(t4-t3):.1f} ms | pairwise() {1e3*(t5-t4):.1f} ms", flush=True)
