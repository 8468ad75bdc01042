"""Split of the C2 e2e overhead (GPU box): corpus build, all-pairs into a
device buffer vs into host memory, with and without a fresh corpus."""
import sys, time, statistics
sys.path.insert(0, "/root/repo")
import numpy as np, torch
import bench
import paper_1707_02423_b200 as P
from paper_1707_02423_b200 import _native as nat
sys.argv = ["bench.py"]
args = bench.parse()
cfg, mats, _ = bench.corpus(args)
tms = [P.TransitionMatrix(f"k{i:05d}", m, tuple(range(len(m))), P.ROW_STOCHASTIC) for i, m in enumerate(mats)]
k = len(tms)
prm = nat.params()
dev_scores = torch.empty((k, k), dtype=torch.float64, device="cuda")
host_scores = np.empty((k, k))
pin_scores = torch.empty((k, k), dtype=torch.float64, pin_memory=True)
def t(f, n=8):
    ts = []
    for _ in range(n):
        torch.cuda.synchronize(); t0 = time.perf_counter(); f(); torch.cuda.synchronize(); ts.append(1e3 * (time.perf_counter() - t0))
    return "median %.1f min %.1f" % (statistics.median(ts), min(ts))
corp = P.DeviceCorpus(tms, 0)
print("corpus build      ", t(lambda: P.DeviceCorpus(tms, 0).close()))
print("allpairs -> device", t(lambda: nat.check(nat.lib.cfgsim_allpairs(corp.handle, 0, nat.C.byref(prm), nat.ptr(dev_scores), None, None))))
print("allpairs -> host  ", t(lambda: nat.check(nat.lib.cfgsim_allpairs(corp.handle, 0, nat.C.byref(prm), nat.ptr(host_scores), None, None))))
print("allpairs -> pinned", t(lambda: nat.check(nat.lib.cfgsim_allpairs(corp.handle, 0, nat.C.byref(prm), nat.ptr(pin_scores), None, None))))
def fresh():
    with P.DeviceCorpus(tms, 0) as c:
        nat.check(nat.lib.cfgsim_allpairs(c.handle, 0, nat.C.byref(prm), nat.ptr(dev_scores), None, None))
print("fresh corpus+dev  ", t(fresh))
print("D2H 32MB pageable ", t(lambda: host_scores.__setitem__(slice(None), dev_scores.cpu().numpy())))
print("pairwise()        ", t(lambda: P.pairwise(tms, P.MeasureId.ISO, device=0)))
