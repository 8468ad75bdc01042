"""Does the host run ahead of the GPU in the bench loop?  Enqueue time of
10 C2 steps (no syncs) vs their device time."""
import sys, time
sys.path.insert(0, "/root/repo")
import numpy as np, torch
import bench
import paper_1707_02423_b200 as P
from paper_1707_02423_b200 import _native as nat
sys.argv = ["bench.py"]
args = bench.parse()
cfg, mats, _ = bench.corpus(args)
corpus_d = P.DeviceCorpus(mats, device=0)
k = len(mats)
bounds = corpus_d.split(1)
u0, u1 = int(bounds[0]), int(bounds[1])
d_lin = torch.empty(u1 - u0, dtype=torch.float64, device="cuda")
it_lin = torch.zeros(u1 - u0, dtype=torch.int32, device="cuda")
scores = torch.empty((k, k), dtype=torch.float64, device="cuda")
prm = nat.params()
st = torch.cuda.current_stream().cuda_stream
def step():
    nat.check(nat.lib.cfgsim_allpairs_range(corpus_d.handle, u0, u1, 0, nat.C.byref(prm), nat.ptr(d_lin), nat.ptr(it_lin), st))
    nat.check(nat.lib.cfgsim_allpairs_scatter(corpus_d.handle, 0, nat.ptr(d_lin), None, nat.ptr(scores), None, st))
for _ in range(3): step()
torch.cuda.synchronize()
for rep in range(3):
    t0 = time.perf_counter(); ts = []
    for s in range(10):
        step(); ts.append(1e3 * (time.perf_counter() - t0))
    t1 = time.perf_counter(); torch.cuda.synchronize(); t2 = time.perf_counter()
    print(f"enqueue 10 steps {1e3*(t1-t0):.1f} ms, then wait {1e3*(t2-t1):.1f} ms; cumulative enqueue ms {[round(x) for x in ts]}", flush=True)
