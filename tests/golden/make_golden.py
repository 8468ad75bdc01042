"""Generate golden vectors for the IsoRank path by running the REFERENCE itself.

Run in the build container (the reference is importable only here):

    python tests/golden/make_golden.py

It imports ``sasscfg`` from /root/reference/pkg/src (read-only, unmodified)
and writes small .npz/.csv fixtures next to this script.  Tests on the GPU
box read only these fixtures; nothing at test time touches /root/reference.

Fixtures
  bundled_corpus.npz  config 1: the 6 bundled kernels' row-stochastic
                      matrices (kernel_id order) + reference pairwise(ISO)
                      scores, per-ordered-pair iterations / matched weight /
                      converged, and the iso.csv / iso_scaled.csv bytes
  small_pairs.npz     random raw matrices n=1..6 (incl. zero rows, different
                      sizes): reference measure_distance(ISO) and, for equal
                      sizes, isorank_align's matrix / matching / weight / iters
  synth_pairs.npz     synthetic CFG pairs (paper_1707_02423_b200.synth,
                      16..64 blocks): reference measure_distance(ISO) with
                      iterations and matched weight
  interp.npz          interpolate_to vectors (matrix.py:74-106)
  special.npz         the reference's pinned cases (test_similarity.py:149-244)
"""

from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
REPO = HERE.parent.parent
REF_SRC = Path("/root/reference/pkg/src")
REF_CORPUS = Path("/root/reference/pkg/corpus/manifest.txt")
sys.path.insert(0, str(REF_SRC))
sys.path.insert(0, str(REPO))

from sasscfg import similarity as S  # noqa: E402
from sasscfg.cli import _load_corpus, _matrices  # noqa: E402
from sasscfg.corpus import RunConfig, load_manifest  # noqa: E402
from sasscfg.matrix import RAW_COUNTS, TransitionMatrix, interpolate_to, normalize_pair  # noqa: E402

from paper_1707_02423_b200 import synth  # noqa: E402  (pure numpy module)


def ragged(mats):
    sizes = np.array([m.shape[0] for m in mats], np.int32)
    flat = np.concatenate([np.asarray(m, float).ravel() for m in mats]) if mats else np.zeros(0)
    return sizes, flat


def align_full(a, b):
    """Reference per-pair call with everything measure_distance hides."""
    na, nb = normalize_pair(a, b)
    al = S.isorank_align(na, nb)
    return S.isorank_distance(al), al


def bundled():
    kernels = _load_corpus(load_manifest(REF_CORPUS))
    mats = _matrices(kernels, RunConfig())
    pm = S.pairwise(mats, S.MeasureId.ISO)
    order = sorted(mats, key=lambda m: m.kernel_id)
    k = len(order)
    iters = np.zeros((k, k), np.int32)
    weight = np.zeros((k, k))
    conv = np.zeros((k, k), bool)
    for i in range(k):
        for j in range(k):
            d, al = align_full(order[i], order[j])
            assert d == pm.scores[i, j]
            iters[i, j] = al.iterations
            weight[i, j] = al.matched_weight
            conv[i, j] = al.converged
    sizes, flat = ragged([m.entries for m in order])
    np.savez_compressed(HERE / "bundled_corpus.npz", ids=np.array(pm.kernel_ids), sizes=sizes, flat=flat,
                        scores=pm.scores, iters=iters, weight=weight, converged=conv)
    (HERE / "iso.csv").write_text(S.export_heatmap_csv(pm))
    (HERE / "iso_scaled.csv").write_text(S.export_heatmap_csv(S.minmax_scale(pm)))


def mat(e, kid="r.synth.t.rand"):
    return TransitionMatrix(kid, np.asarray(e, float), tuple(range(len(e))), RAW_COUNTS)


def small_pairs():
    rng = np.random.default_rng(2024)
    A, B, d, w, it, cv, X, match, same = [], [], [], [], [], [], [], [], []
    for t in range(120):
        na = int(rng.integers(1, 7))
        nb = na if t % 2 == 0 else int(rng.integers(1, 7))
        a = rng.random((na, na)) * (rng.random((na, na)) < 0.6)
        b = rng.random((nb, nb)) * (rng.random((nb, nb)) < 0.6)
        if t % 5 == 0:
            a[rng.integers(0, na)] = 0.0  # a zero row -> uniform row
        dd, al = align_full(mat(a), mat(b))
        A.append(a); B.append(b); d.append(dd); w.append(al.matched_weight)
        it.append(al.iterations); cv.append(al.converged)
        X.append(al.matrix); match.append(np.array(al.matching, np.int32)); same.append(na == nb)
    sa, fa = ragged(A)
    sb, fb = ragged(B)
    sx, fx = ragged(X)
    np.savez_compressed(HERE / "small_pairs.npz", sa=sa, fa=fa, sb=sb, fb=fb, d=np.array(d), W=np.array(w),
                        iters=np.array(it, np.int32), converged=np.array(cv), sx=sx, fx=fx,
                        match=np.concatenate(match), same=np.array(same))


def synth_pairs(n_pairs=48):
    mats = synth.random_corpus(2 * n_pairs, 16, 64, seed=77)
    A, B, d, w, it = [], [], [], [], []
    for t in range(n_pairs):
        a, b = mats[2 * t], mats[2 * t + 1]
        dd, al = align_full(mat(a, "a.s.t.x"), mat(b, "b.s.t.x"))
        A.append(a); B.append(b); d.append(dd); w.append(al.matched_weight); it.append(al.iterations)
        print(f"synth pair {t}: n=({a.shape[0]},{b.shape[0]}) iters={al.iterations} d={dd:.12f}", flush=True)
    sa, fa = ragged(A)
    sb, fb = ragged(B)
    np.savez_compressed(HERE / "synth_pairs.npz", sa=sa, fa=fa, sb=sb, fb=fb, d=np.array(d), W=np.array(w),
                        iters=np.array(it, np.int32))


def interp():
    rng = np.random.default_rng(11)
    srcs, targets, outs = [], [], []
    for t in range(60):
        n = int(rng.integers(1, 20))
        target = n + int(rng.integers(0, 40))
        src = rng.random((n, n)) * (rng.random((n, n)) < 0.5)
        out = interpolate_to(mat(src), target).entries
        srcs.append(src); targets.append(target); outs.append(out)
    ss, fs = ragged(srcs)
    so, fo = ragged(outs)
    np.savez_compressed(HERE / "interp.npz", ss=ss, fs=fs, targets=np.array(targets, np.int32), so=so, fo=fo)


def special():
    out = {}
    al = S.isorank_align(mat([[0.0]]), mat([[0.0]]))
    out["singleton_X"] = al.matrix
    out["singleton_iters"] = al.iterations
    z = S.isorank_align(mat(np.zeros((3, 3))), mat(np.zeros((3, 3))))
    out["zeros_match"] = np.array(z.matching)
    rng = np.random.default_rng(92)
    a, b = rng.random((3, 3)), rng.random((3, 3))
    s = S.isorank_align(mat(a), mat(b), alpha=1e-9)
    out["small_alpha_a"], out["small_alpha_b"] = a, b
    out["small_alpha_X"], out["small_alpha_W"] = s.matrix, s.matched_weight
    rng = np.random.default_rng(93)
    a, b = rng.random((3, 3)), rng.random((3, 3))
    start = rng.random(9) + 0.01
    s = S.isorank_align(mat(a), mat(b), start=start)
    out["start_a"], out["start_b"], out["start_vec"] = a, b, start
    out["start_X"], out["start_iters"] = s.matrix, s.iterations
    rng = np.random.default_rng(91)
    a, b = rng.random((3, 3)), rng.random((3, 3))
    out["cut_a"], out["cut_b"] = a, b
    out["cut_X"] = np.stack([S.isorank_align(mat(a), mat(b), max_iter=c).matrix for c in range(1, 8)])
    np.savez_compressed(HERE / "special.npz", **out)


if __name__ == "__main__":
    bundled()
    small_pairs()
    interp()
    special()
    synth_pairs()
    print("golden fixtures written to", HERE)
