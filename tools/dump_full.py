import sys, numpy as np
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
import paper_1707_02423_b200 as P
from test_gpu_large import dense
G = dict(np.load('tests/golden/large_pairs.npz'))
out = {}
for k, q in enumerate(np.nonzero(G['full'])[0]):
    a = P.TransitionMatrix('a', dense(G, int(G['ia'][q])), None, P.RAW_COUNTS)
    b = P.TransitionMatrix('b', dense(G, int(G['ib'][q])), None, P.RAW_COUNTS)
    a, b = P.normalize_pair(a, b)
    al = P.isorank_align(a, b, alpha=float(G['alpha'][q]), tol=float(G['tol'][q]), max_iter=int(G['max_iter'][q]))
    out[f'X{k}'] = al.matrix; out[f'm{k}'] = np.array(al.matching); out[f'A{k}'] = a.entries; out[f'B{k}'] = b.entries
    out[f'it{k}'] = al.iterations
np.savez('gpurun_out/dump_full.npz', **out)
print('ok')
