"""Golden vectors for the large-N path (N > 128; configs C4 / C5) from the
pinned C oracle.

The reference itself cannot run here at these sizes (its Kronecker matrix is
8 N^4 bytes: 34 GB at N = 256), so parity at large N is anchored
on the oracle (oracle/isorank_ref.c), which tests/test_oracle.py pins to the
reference's own outputs at small N.  Run in the build container:

    python tests/golden/make_large.py

Writes tests/golden/large_pairs.npz: packed CSR graphs (synthetic CFGs with
the reference's structure, paper_1707_02423_b200.synth, plus hand-built edge
cases), pair lists with parameters, and the oracle's d / W / iterations /
converged; for the cases flagged `full`, X and the matching as well.
"""

from __future__ import annotations

import os
import sys
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
REPO = HERE.parent.parent
sys.path.insert(0, str(REPO))

from oracle import ffi  # noqa: E402
from paper_1707_02423_b200 import synth  # noqa: E402
from paper_1707_02423_b200.packing import pack  # noqa: E402


def cfg(rng, n, weighting):
    return synth.transition_matrix(synth.random_shape(rng, n, weighting))


def main():
    rng = np.random.default_rng(20261017)
    graphs = []
    cases = []  # (ia, ib, alpha, tol, max_iter, full)

    def add(m):
        graphs.append(np.asarray(m, float))
        return len(graphs) - 1

    # C4: observed edge counts, 256..1024 blocks (fp64)
    for na, nb in [(1024, 1024), (1000, 256), (700, 690), (512, 300), (257, 900), (333, 333)]:
        cases.append((add(cfg(rng, na, "observed")), add(cfg(rng, nb, "observed")), 0.85, 1e-9, 1000, False))
    # C5: mixed 16..512, sampled / uniform-static weights, N > 128
    for na, nb in [(16, 512), (512, 17), (129, 129), (130, 64), (200, 450), (511, 512), (48, 300), (400, 129)]:
        cases.append((add(cfg(rng, na, "sampled")), add(cfg(rng, nb, "sampled")), 0.85, 1e-9, 1000, False))
    # full outputs (X, matching) at moderate N
    a, b = add(cfg(rng, 160, "sampled")), add(cfg(rng, 150, "observed"))
    cases.append((a, b, 0.85, 1e-9, 1000, True))
    # single-node side (matrix.py:87-89) against a large graph, zero and non-zero
    one0, one1 = add(np.zeros((1, 1))), add(np.full((1, 1), 0.5))
    big = add(cfg(rng, 200, "sampled"))
    cases.append((one0, big, 0.85, 1e-9, 1000, False))
    cases.append((big, one1, 0.85, 1e-9, 1000, False))
    # all-zero operator (every row uniform) and a random dense-ish weighted one
    zero = add(np.zeros((150, 150)))
    dense = rng.random((180, 180)) * (rng.random((180, 180)) < 0.05)
    dense[rng.random(180) < 0.2] = 0.0
    dz = add(dense)
    cases.append((zero, dz, 0.85, 1e-9, 1000, True))
    cases.append((dz, add(cfg(rng, 140, "observed")), 0.85, 1e-9, 1000, False))
    # max_iter cut-off and other parameters
    c1, c2 = add(cfg(rng, 220, "sampled")), add(cfg(rng, 210, "sampled"))
    cases.append((c1, c2, 0.85, 1e-9, 7, True))
    cases.append((c1, c2, 0.5, 1e-12, 1000, False))
    cases.append((c2, c1, 0.95, 1e-9, 1000, False))

    def run(case):
        ia, ib, alpha, tol, mi, full = case
        r = ffi.iso_pair(graphs[ia], graphs[ib], alpha=alpha, tol=tol, max_iter=mi)
        return r

    with ThreadPoolExecutor(max_workers=os.cpu_count() or 4) as ex:
        res = list(ex.map(run, cases))
    packed = pack(graphs)
    out = {f"g_{k}": v for k, v in packed.items()}
    out["ia"] = np.array([c[0] for c in cases], np.int32)
    out["ib"] = np.array([c[1] for c in cases], np.int32)
    out["alpha"] = np.array([c[2] for c in cases])
    out["tol"] = np.array([c[3] for c in cases])
    out["max_iter"] = np.array([c[4] for c in cases], np.int32)
    out["full"] = np.array([c[5] for c in cases], bool)
    out["d"] = np.array([r["d"] for r in res])
    out["W"] = np.array([r["W"] for r in res])
    out["iters"] = np.array([r["iterations"] for r in res], np.int32)
    out["converged"] = np.array([r["converged"] for r in res], bool)
    fx, fm, fn = [], [], []
    for c, r in zip(cases, res):
        if c[5]:
            fx.append(r["X"].ravel())
            fm.append(np.array(r["matching"], np.int32))
            fn.append(r["X"].shape[0])
    out["full_n"] = np.array(fn, np.int32)
    out["full_X"] = np.concatenate(fx)
    out["full_match"] = np.concatenate(fm)
    np.savez_compressed(HERE / "large_pairs.npz", **out)
    for c, r in zip(cases, res):
        print(graphs[c[0]].shape[0], graphs[c[1]].shape[0], c[2:5], r["iterations"], r["converged"], r["d"])


if __name__ == "__main__":
    main()
