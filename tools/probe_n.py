import sys, time, numpy as np, torch
sys.path.insert(0, '.')
import paper_1707_02423_b200 as P
from paper_1707_02423_b200 import synth
mats = synth.random_corpus(3000, 16, 300, seed=2)
n = np.array([len(m) for m in mats])
rng = np.random.default_rng(0)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
with P.DeviceCorpus(mats) as C:
    for N in [168, 129, 136, 144, 152, 160, 168, 176, 200, 129]:
        rows = np.flatnonzero(n == N); parts = np.flatnonzero(n <= N)
        for mode in ("any", "same"):
            ps = parts if mode == "any" else np.flatnonzero((n <= N) & (n >= N - 8))
            ia = rng.choice(rows, 2000).astype(np.int32); ib = rng.choice(ps, 2000).astype(np.int32)
            ts = []
            for rep in range(3):
                torch.cuda.synchronize(); e0.record()
                d, w, it, cv = P.isorank_pairs(C, C, ia, ib)
                e1.record(); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1) * 1e3 / 2000)
            print(N, mode, [round(t, 2) for t in ts], "mean iters", it.mean(), flush=True)
