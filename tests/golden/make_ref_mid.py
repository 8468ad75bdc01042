"""Reference outputs for a mid-size pair (N = 160) — the largest N at which
the reference's dense Kronecker path (8 N^4 bytes = 5.2 GB) runs on the
build host.  Run in the build container:

    python tests/golden/make_ref_mid.py

Writes tests/golden/ref_mid.npz: the two raw matrices (160 x 160 sampled-
weight CFG, 150 x 150 observed-count CFG, from tests/golden/large_pairs.npz
case `full` 0), and the reference's normalize_pair -> isorank_align outputs
(X, matching, matched weight, iterations, converged) and
measure_distance(ISO).
"""

from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, "/root/reference/pkg/src")

from sasscfg import similarity as S  # noqa: E402
from sasscfg.matrix import RAW_COUNTS, TransitionMatrix, normalize_pair  # noqa: E402


def dense(G, g):
    p = {k[2:]: v for k, v in G.items() if k.startswith("g_")}
    n = int(p["n_nodes"][g])
    m = np.zeros((n, n))
    rp = p["rowptr"][p["rp_off"][g]:p["rp_off"][g] + n + 1]
    o = p["nz_off"][g]
    for r in range(n):
        for e in range(rp[r], rp[r + 1]):
            m[r, p["col"][o + e]] = p["val"][o + e]
    return m


def main():
    G = dict(np.load(HERE / "large_pairs.npz"))
    q = int(np.nonzero(G["full"])[0][0])
    A, B = dense(G, int(G["ia"][q])), dense(G, int(G["ib"][q]))
    a = TransitionMatrix("a.mid.ref.x", A, tuple(range(len(A))), RAW_COUNTS)
    b = TransitionMatrix("b.mid.ref.x", B, tuple(range(len(B))), RAW_COUNTS)
    na, nb = normalize_pair(a, b)
    al = S.isorank_align(na, nb)
    d = S.measure_distance(a, b, S.MeasureId.ISO)
    np.savez_compressed(HERE / "ref_mid.npz", A=A, B=B, X=al.matrix, matching=np.array(al.matching, np.int32),
                        W=al.matched_weight, iterations=al.iterations, converged=al.converged, d=d)
    print(al.iterations, al.converged, d)


if __name__ == "__main__":
    main()
