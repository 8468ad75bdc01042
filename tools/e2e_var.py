import sys, time, gc, os, statistics
sys.path.insert(0, "/root/repo")
import numpy as np, torch
import bench
import paper_1707_02423_b200 as P
sys.argv = ["bench.py"]
args = bench.parse()
cfg, mats, _ = bench.corpus(args)
tms = [P.TransitionMatrix(f"k{i:05d}", m, tuple(range(len(m))), P.ROW_STOCHASTIC) for i, m in enumerate(mats)]
P.pairwise(tms, P.MeasureId.ISO, device=0)
mode = sys.argv[1] if len(sys.argv) > 1 else os.environ.get("VAR", "default")
if os.environ.get("NOGC"): gc.disable()
ts = []
for r in range(20):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    pm = P.pairwise(tms, P.MeasureId.ISO, device=0)
    ts.append(1e3 * (time.perf_counter() - t0))
print(os.environ.get("TAG"), "median %.1f max %.1f" % (statistics.median(ts), max(ts)), [round(t) for t in ts])
