"""Parity of the sm_100a IsoRank path against the reference (golden vectors)
and the pinned CPU oracle.  Runs on the B200 box (``-m gpu``).

Bar (BASELINE.json north_star): fp64 — identical iteration counts, distance
within 1e-9 relative (observed ~1e-15); fp32 — distance within 1e-5.
"""

from __future__ import annotations

import numpy as np
import pytest

from conftest import GOLDEN, load_golden, unravel

pytestmark = pytest.mark.gpu

RTOL64 = 1e-9
RTOL32 = 1e-5


@pytest.fixture(scope="module")
def P(gpu):
    import paper_1707_02423_b200 as P
    return P


def mat(P, e, kid="r.synth.t.rand"):
    e = np.asarray(e, float)
    return P.TransitionMatrix(kid, e, tuple(range(len(e))), P.RAW_COUNTS)


# ------------------------------------------------------------ interpolation
def test_interpolate_bit_exact(P):
    g = load_golden("interp.npz")
    srcs, outs = unravel(g["ss"], g["fs"]), unravel(g["so"], g["fo"])
    for src, t, out in zip(srcs, g["targets"], outs):
        m = mat(P, src)
        got = P.interpolate_to(m, int(t))
        if int(t) == src.shape[0]:
            assert got is m  # matrix.py:85-86
        np.testing.assert_array_equal(got.entries, out)


# ------------------------------------------------------------ single pairs
def greedy_is_untied(X, rel=1e-9):
    """True when every round of _greedy_matching (similarity.py:96-108) on X
    has a unique best entry by a margin (then any correct implementation must
    return the reference's own matching)."""
    w = np.array(X, float)
    for _ in range(w.shape[0]):
        flat = w.ravel()
        top = np.partition(flat, -2)[-2:] if flat.size > 1 else np.array([-1.0, flat[0]])
        best, second = float(top.max()), float(top.min())
        if flat.size > 1 and best - second <= rel * max(abs(best), 1e-300):
            return False
        r, c = divmod(int(np.argmax(flat)), w.shape[1])
        w[r, :] = -1.0
        w[:, c] = -1.0
    return True


def test_small_pairs_against_reference(P):
    g = load_golden("small_pairs.npz")
    A, B, X = unravel(g["sa"], g["fa"]), unravel(g["sb"], g["fb"]), unravel(g["sx"], g["fx"])
    offs = np.concatenate([[0], np.cumsum(g["sx"])])
    untied = 0
    for i, (a, b) in enumerate(zip(A, B)):
        d = P.measure_distance(mat(P, a), mat(P, b), P.MeasureId.ISO)
        assert d == pytest.approx(g["d"][i], rel=1e-12, abs=1e-12), i
        if g["same"][i]:
            al = P.isorank_align(mat(P, a), mat(P, b))
            assert al.iterations == g["iters"][i]
            assert al.converged == g["converged"][i]
            np.testing.assert_allclose(al.matrix, X[i], rtol=1e-10, atol=1e-15)
            assert al.matched_weight == pytest.approx(g["W"][i], rel=1e-12)
            assert sorted(al.matching) == list(range(a.shape[0]))
            if greedy_is_untied(X[i]):  # the reference's own permutation
                assert al.matching == tuple(int(v) for v in g["match"][offs[i]:offs[i + 1]]), i
                untied += 1
    assert untied >= 20


def test_reference_pinned_cases(P):
    s = load_golden("special.npz")
    al = P.isorank_align(mat(P, [[0.0]]), mat(P, [[0.0]]))  # test_similarity.py:150-155
    np.testing.assert_array_equal(al.matrix, [[1.0]])
    assert al.matching == (0,) and al.matched_weight == 1.0
    assert al.converged and al.iterations == 1
    al = P.isorank_align(mat(P, np.zeros((3, 3))), mat(P, np.zeros((3, 3))))  # :191-195
    assert al.matching == (0, 1, 2)
    al = P.isorank_align(mat(P, s["small_alpha_a"]), mat(P, s["small_alpha_b"]), alpha=1e-9)  # :176-181
    np.testing.assert_allclose(al.matrix, np.full((3, 3), 1.0 / 9.0), atol=1e-8)
    assert al.matched_weight == pytest.approx(1.0 / 3.0, abs=1e-8)
    al = P.isorank_align(mat(P, s["start_a"]), mat(P, s["start_b"]), start=s["start_vec"])  # :183-189
    np.testing.assert_allclose(al.matrix, s["start_X"], rtol=1e-10)
    assert al.iterations == s["start_iters"]
    for c in range(1, 8):  # :167-174
        al = P.isorank_align(mat(P, s["cut_a"]), mat(P, s["cut_b"]), max_iter=c)
        assert al.iterations == c
        assert (al.matrix >= 0).all()
        assert al.matrix.sum() == pytest.approx(1.0, abs=1e-9)
        np.testing.assert_allclose(al.matrix, s["cut_X"][c - 1], rtol=1e-12)
    rng = np.random.default_rng(95)  # :204-208
    al = P.isorank_align(mat(P, rng.random((2, 2))), mat(P, rng.random((2, 2))), max_iter=1)
    assert not al.converged and al.iterations == 1


def test_uniform_alignment_scores_two(P):  # test_similarity.py:242-244
    al = P.isorank_align(mat(P, np.zeros((4, 4))), mat(P, np.zeros((4, 4))), alpha=1e-9)
    assert P.isorank_distance(al) == pytest.approx(2.0, abs=1e-6)


@pytest.mark.parametrize("alpha", [0.0, 1.0, 1.2, -0.1])
def test_alpha_range_enforced(P, alpha):
    with pytest.raises(ValueError):
        P.isorank_align(mat(P, np.eye(2)), mat(P, np.eye(2)[::-1]), alpha=alpha)


def test_dim_mismatch(P):
    with pytest.raises(P.DimMismatch):
        P.isorank_align(mat(P, [[1.0]]), mat(P, np.eye(2)))


def test_measure_distance_normalises_sizes(P):  # test_similarity.py:260-263
    rng = np.random.default_rng(8)
    d = P.measure_distance(mat(P, rng.random((2, 2))), mat(P, rng.random((3, 3))), P.MeasureId.ISO)
    assert 1.0 <= d <= 2.0


# ------------------------------------------------------------ synthetic CFG pairs (batched path)
def test_synthetic_cfg_pairs_against_reference(P):
    g = load_golden("synth_pairs.npz")
    A, B = unravel(g["sa"], g["fa"]), unravel(g["sb"], g["fb"])
    n = len(A)
    with P.DeviceCorpus(A) as CA, P.DeviceCorpus(B) as CB:
        d, w, it, cv = P.isorank_pairs(CA, CB, np.arange(n), np.arange(n))
    np.testing.assert_array_equal(it, g["iters"])
    np.testing.assert_allclose(d, g["d"], rtol=1e-12)
    np.testing.assert_allclose(w, g["W"], rtol=1e-10)
    assert cv.all()


# ------------------------------------------------------------ config 1: bundled corpus
def _bundled(P):
    g = load_golden("bundled_corpus.npz")
    mats = unravel(g["sizes"], g["flat"])
    # shuffled input order: pairwise must sort by kernel_id (similarity.py:229)
    tms = [P.TransitionMatrix(str(k), m, tuple(range(len(m))), P.ROW_STOCHASTIC) for k, m in zip(g["ids"], mats)]
    return g, tms[::-1]


@pytest.mark.parametrize("symmetric", [True, False])
def test_bundled_corpus_pairwise(P, symmetric):
    g, tms = _bundled(P)
    pm, iters = P.pairwise(tms, P.MeasureId.ISO, symmetric=symmetric, return_iterations=True)
    assert pm.kernel_ids == tuple(str(x) for x in g["ids"])
    np.testing.assert_allclose(pm.scores, g["scores"], rtol=1e-12)
    # the default (symmetric) mirrors d(a, b) into d(b, a); the reference runs
    # both directions (similarity.py:240-246), which agree with each other to
    # 4.4e-16 with identical iteration counts — so the mirrored
    # matrix equals the reference's ordered one at rtol 1e-12, iterations
    # included, in both modes
    np.testing.assert_array_equal(iters, g["iters"])


def test_bundled_corpus_csv_byte_identical(P):
    g, tms = _bundled(P)
    pm = P.pairwise(tms, P.MeasureId.ISO, symmetric=False)
    assert P.export_heatmap_csv(pm) == (GOLDEN / "iso.csv").read_text()
    assert P.export_heatmap_csv(P.minmax_scale(pm)) == (GOLDEN / "iso_scaled.csv").read_text()


def test_pairwise_errors(P):
    with pytest.raises(ValueError):
        P.pairwise([mat(P, [[1.0]])], P.MeasureId.ISO)
    with pytest.raises(P.DuplicateKernel):
        P.pairwise([mat(P, [[1.0]], "x.s.t.d"), mat(P, [[2.0]], "x.s.t.d")], P.MeasureId.ISO)


# ------------------------------------------------------------ config-2-like sample vs the C oracle
@pytest.fixture(scope="module")
def c2_sample(P):
    from paper_1707_02423_b200 import synth
    mats = synth.random_corpus(96, 16, 64, seed=5)
    return mats


def test_allpairs_sample_matches_oracle(P, c2_sample):
    from oracle import ffi
    mats = c2_sample
    k = len(mats)
    tms = [P.TransitionMatrix(f"g{i:04d}", m, tuple(range(len(m))), P.ROW_STOCHASTIC) for i, m in enumerate(mats)]
    pm, iters = P.pairwise(tms, P.MeasureId.ISO, return_iterations=True)
    iu, ju = np.triu_indices(k)
    d, w, it, cv = ffi.iso_batch(P.pack(mats), iu.astype(np.int32), ju.astype(np.int32))
    np.testing.assert_allclose(pm.scores[iu, ju], d, rtol=RTOL64)
    mism = int((iters[iu, ju] != it).sum())
    assert mism == 0, f"{mism} iteration-count mismatches of {len(iu)}"
    np.testing.assert_array_equal(pm.scores, pm.scores.T)


def test_fp32_mode_within_tolerance(P, c2_sample):
    from oracle import ffi
    mats = c2_sample[:40]
    k = len(mats)
    tms = [P.TransitionMatrix(f"g{i:04d}", m, tuple(range(len(m))), P.ROW_STOCHASTIC) for i, m in enumerate(mats)]
    pm = P.pairwise(tms, P.MeasureId.ISO, precision="fp32")
    iu, ju = np.triu_indices(k)
    d, *_ = ffi.iso_batch(P.pack(mats), iu.astype(np.int32), ju.astype(np.int32))
    np.testing.assert_allclose(pm.scores[iu, ju], d, rtol=RTOL32)


def test_deterministic_and_path_independent(P, c2_sample):
    mats = c2_sample[:48]
    tms = [P.TransitionMatrix(f"g{i:04d}", m, tuple(range(len(m))), P.ROW_STOCHASTIC) for i, m in enumerate(mats)]
    a = P.pairwise(tms, P.MeasureId.ISO).scores
    b = P.pairwise(tms, P.MeasureId.ISO).scores
    np.testing.assert_array_equal(a, b)
    iu, ju = np.triu_indices(len(mats))
    with P.DeviceCorpus(mats) as C:
        d, *_ = P.isorank_pairs(C, C, iu, ju)
    # the same pair through the list path and the triangle path: bitwise equal
    np.testing.assert_array_equal(d, a[iu, ju])


def test_nearest_matches_oracle(P, c2_sample):
    from oracle import ffi
    q = c2_sample[:6]
    corpus = c2_sample[6:60]
    bd, bi = P.nearest(q, corpus)
    allm = q + corpus
    packed = P.pack(allm)
    for i in range(len(q)):
        ia = np.full(len(corpus), i, np.int32)
        ib = np.arange(len(q), len(allm), dtype=np.int32)
        d, *_ = ffi.iso_batch(packed, ia, ib)
        assert bi[i] == int(np.argmin(d))
        assert bd[i] == pytest.approx(d.min(), rel=RTOL64)


# ------------------------------------------------------------ tiers and edge cases
def test_large_tier_pairs(P):
    from oracle import ffi
    from paper_1707_02423_b200 import synth
    mats = synth.random_corpus(8, 70, 104, seed=9)
    with P.DeviceCorpus(mats) as C:
        ia = np.arange(0, 8, 2)
        ib = ia + 1
        d, w, it, cv = P.isorank_pairs(C, C, ia, ib)
    for k in range(len(ia)):
        r = ffi.iso_pair(mats[ia[k]], mats[ib[k]])
        assert it[k] == r["iterations"]
        assert d[k] == pytest.approx(r["d"], rel=RTOL64)


def test_dense_operators_overflow_path(P):
    """Dense random operators exceed the typical list capacity and are re-run
    with dense-bound lists; results must not change."""
    from oracle import ffi
    rng = np.random.default_rng(3)
    mats = [rng.random((n, n)) for n in (40, 55, 63, 20, 31, 47)]
    with P.DeviceCorpus(mats) as C:
        ia = np.array([0, 1, 2, 3, 4, 5, 0], np.int32)
        ib = np.array([1, 2, 3, 4, 5, 0, 0], np.int32)
        d, w, it, cv = P.isorank_pairs(C, C, ia, ib)
    for k in range(len(ia)):
        r = ffi.iso_pair(mats[ia[k]], mats[ib[k]])
        assert it[k] == r["iterations"]
        assert d[k] == pytest.approx(r["d"], rel=RTOL64)


def test_degenerate_graphs(P):
    from oracle import ffi
    rng = np.random.default_rng(4)
    cases = [(np.zeros((1, 1)), rng.random((5, 5))), (np.ones((1, 1)) * 3, rng.random((7, 7))),
             (np.zeros((6, 6)), np.zeros((9, 9))), (np.eye(33), np.eye(33)[::-1].copy()),
             (np.zeros((64, 64)), rng.random((2, 2)))]
    for a, b in cases:
        d = P.measure_distance(mat(P, a), mat(P, b), P.MeasureId.ISO)
        r = ffi.iso_pair(a, b)
        assert d == pytest.approx(r["d"], rel=RTOL64)


def test_lazy_delta_correction_is_exact(P, c2_sample):
    """The normalisation correction term of delta is only accumulated near
    convergence; forcing it every sweep must not change any result."""
    import os
    import subprocess
    import sys
    code = ("import numpy as np, sys; sys.path.insert(0, '.');"
            "import paper_1707_02423_b200 as P; from paper_1707_02423_b200 import synth;"
            "m = synth.random_corpus(40, 16, 64, seed=5);"
            "t = [P.TransitionMatrix(f'g{i:03d}', x, tuple(range(len(x))), P.ROW_STOCHASTIC) for i, x in enumerate(m)];"
            "pm, it = P.pairwise(t, P.MeasureId.ISO, return_iterations=True);"
            "np.save(sys.argv[1], np.concatenate([pm.scores.ravel(), it.ravel().astype(float)]))")
    outs = []
    for force in ("0", "1"):
        path = f"/tmp/cfgsim_force_m_{force}.npy"
        env = dict(os.environ, CFGSIM_FORCE_M=force)
        subprocess.run([sys.executable, "-c", code, path], check=True, env=env, cwd=str(GOLDEN.parent.parent))
        outs.append(np.load(path))
    np.testing.assert_array_equal(outs[0], outs[1])


def test_lowrank_and_two_product_kernels_agree(P):
    """The default (closed-form, rank-structured) kernel and the general
    two-product kernel (CFGSIM_ALGO=dense) compute the same iterates."""
    import os
    import subprocess
    import sys
    code = ("import numpy as np, sys; sys.path.insert(0, '.');"
            "import paper_1707_02423_b200 as P; from paper_1707_02423_b200 import synth;"
            "m = synth.random_corpus(60, 16, 100, seed=21);"
            "t = [P.TransitionMatrix(f'g{i:03d}', x, tuple(range(len(x))), P.ROW_STOCHASTIC) for i, x in enumerate(m)];"
            "pm, it = P.pairwise(t, P.MeasureId.ISO, return_iterations=True, symmetric=False);"
            "np.save(sys.argv[1], np.concatenate([pm.scores.ravel(), it.ravel().astype(float)]))")
    outs = []
    for algo in ("lowrank", "dense"):
        path = f"/tmp/cfgsim_algo_{algo}.npy"
        env = dict(os.environ, CFGSIM_ALGO=algo)
        subprocess.run([sys.executable, "-c", code, path], check=True, env=env, cwd=str(GOLDEN.parent.parent))
        outs.append(np.load(path))
    n = len(outs[0]) // 2
    np.testing.assert_array_equal(outs[0][n:], outs[1][n:])  # iteration counts
    np.testing.assert_allclose(outs[0][:n], outs[1][:n], rtol=1e-12)


def test_two_stage_matches_per_pair_kernel(P):
    """Two-stage all-pairs (per-(graph, N) sequences, then per-pair rank-K
    products; isorank_seq.cuh) against the per-pair low-rank kernel
    (CFGSIM_TWOSTAGE=0): identical iteration counts, bitwise-equal d in fp64."""
    import os
    import subprocess
    import sys
    code = ("import numpy as np, sys; sys.path.insert(0, '.');"
            "import paper_1707_02423_b200 as P; from paper_1707_02423_b200 import synth;"
            "m = synth.random_corpus(120, 1, 64, seed=23) + [np.zeros((1, 1)), np.ones((1, 1)), np.zeros((7, 7))];"
            "m += [np.random.default_rng(2).random((n, n)) for n in (5, 30, 64)];"
            "t = [P.TransitionMatrix(f'g{i:03d}', x, tuple(range(len(x))), P.ROW_STOCHASTIC) for i, x in enumerate(m)];"
            "pm, it = P.pairwise(t, P.MeasureId.ISO, return_iterations=True, precision=sys.argv[2]);"
            "np.save(sys.argv[1], np.concatenate([pm.scores.ravel(), it.ravel().astype(float)]))")
    for prec in ("fp64", "fp32"):
        outs = []
        for two in ("1", "0"):
            path = f"/tmp/cfgsim_two_{two}_{prec}.npy"
            env = dict(os.environ, CFGSIM_TWOSTAGE=two)
            subprocess.run([sys.executable, "-c", code, path, prec], check=True, env=env,
                           cwd=str(GOLDEN.parent.parent))
            outs.append(np.load(path))
        n = len(outs[0]) // 2
        np.testing.assert_array_equal(outs[0][n:], outs[1][n:])
        if prec == "fp64":  # same fma chain (fp64 mma == sequential fma): bitwise
            np.testing.assert_array_equal(outs[0][:n], outs[1][:n])
        else:  # fp32 mode forms the rank-K product in fp64 on the tensor cores
            np.testing.assert_allclose(outs[0][:n], outs[1][:n], rtol=1e-6)


def test_nearest_mixed_sizes_matches_oracle(P):
    """Query-vs-corpus over sizes spanning the two-stage (N <= 64), per-pair
    low-rank (65..128) and large-N (> 128) kernels, fp64 and fp32."""
    from oracle import ffi
    from paper_1707_02423_b200 import synth
    rng = np.random.default_rng(41)
    q = [synth.transition_matrix(synth.random_shape(rng, int(n), "sampled")) for n in (8, 30, 64, 90, 150)]
    c = [synth.transition_matrix(synth.random_shape(rng, int(n), "sampled"))
         for n in rng.integers(4, 180, 40)] + [q[1].copy(), q[3].copy()]
    allm = q + c
    packed = P.pack(allm)
    ia = np.repeat(np.arange(len(q)), len(c)).astype(np.int32)
    ib = np.tile(np.arange(len(q), len(allm)), len(q)).astype(np.int32)
    d, *_ = ffi.iso_batch(packed, ia, ib)
    d = d.reshape(len(q), len(c))
    for prec, rtol in (("fp64", RTOL64), ("fp32", RTOL32)):
        bd, bi = P.nearest(q, c, precision=prec)
        np.testing.assert_allclose(bd, d.min(axis=1), rtol=rtol)
        if prec == "fp64":
            np.testing.assert_array_equal(bi, d.argmin(axis=1))
    # the rectangle path and the per-pair list path agree bitwise
    with P.DeviceCorpus(q) as CQ, P.DeviceCorpus(c) as CC:
        dl, *_ = P.isorank_pairs(CQ, CC, np.repeat(np.arange(len(q)), len(c)), np.tile(np.arange(len(c)), len(q)))
    bd, bi = P.nearest(q, c)
    np.testing.assert_array_equal(bd, dl.reshape(len(q), len(c)).min(axis=1))


def test_sharded_api_single_rank_matches(P):
    """distributed.pairwise_sharded / nearest_gpu_sharded (world 1) equal the
    unsharded API bitwise."""
    from paper_1707_02423_b200 import distributed as D
    from paper_1707_02423_b200 import synth
    mats = synth.random_corpus(40, 8, 150, seed=77)
    tms = [P.TransitionMatrix(f"g{i:03d}.s.h.d", m, tuple(range(len(m))), P.ROW_STOCHASTIC) for i, m in enumerate(mats)]
    a = P.pairwise(tms, P.MeasureId.ISO).scores
    b = D.pairwise_sharded(tms[::-1]).scores
    np.testing.assert_array_equal(a, b)
    bd, bi = P.nearest(mats[:5], mats[5:])
    sd, si = D.nearest_gpu_sharded(mats[:5], mats[5:])
    np.testing.assert_array_equal(bd, sd)
    np.testing.assert_array_equal(bi, si)


@pytest.mark.parametrize("alpha,tol,max_iter", [(0.85, 1e-9, 1), (0.85, 1e-9, 3), (0.85, 1e-9, 7), (0.5, 1e-12, 1000),
                                                (0.95, 1e-9, 1000), (0.99, 1e-9, 1000), (0.85, 1e-6, 50)])
def test_allpairs_parameters_match_oracle(P, alpha, tol, max_iter):
    """Parameter corners through the all-pairs path (two-stage for kcap <= 512,
    the per-pair low-rank kernel beyond, e.g. alpha = 0.99): iteration cut-offs,
    convergence flags, d against the oracle."""
    from oracle import ffi
    from paper_1707_02423_b200 import synth
    mats = synth.random_corpus(24, 4, 64, seed=int(alpha * 100) + max_iter)
    k = len(mats)
    tms = [P.TransitionMatrix(f"g{i:03d}.p.c.t", m, tuple(range(len(m))), P.ROW_STOCHASTIC) for i, m in enumerate(mats)]
    pm, iters = P.pairwise(tms, P.MeasureId.ISO, alpha=alpha, tol=tol, max_iter=max_iter, return_iterations=True)
    iu, ju = np.triu_indices(k)
    d, w, it, cv = ffi.iso_batch(P.pack(mats), iu.astype(np.int32), ju.astype(np.int32), alpha=alpha, tol=tol,
                                 max_iter=max_iter)
    np.testing.assert_array_equal(iters[iu, ju], it)
    np.testing.assert_allclose(pm.scores[iu, ju], d, rtol=RTOL64)


def test_nearest_small_queries_after_stage2(P):
    """Regression (r1 memcheck finding): query-vs-corpus over graphs below 32
    blocks right after a stage-2 launch, whose shared-memory sentinels used to
    leak into the four-combo stage-1 kernel's list offsets for lanes >= N.
    The rectangle path must equal the per-pair list path bitwise."""
    from paper_1707_02423_b200 import synth
    warm = synth.random_corpus(24, 16, 64, seed=9)
    P.pairwise([P.TransitionMatrix(f"w{i:03d}.s.w", m, tuple(range(len(m))), P.ROW_STOCHASTIC)
                for i, m in enumerate(warm)], P.MeasureId.ISO)
    q = synth.random_corpus(96, 4, 31, seed=3)
    c = synth.random_corpus(2500, 4, 31, seed=2)
    bd, bi = P.nearest(q, c)
    with P.DeviceCorpus(q) as CQ, P.DeviceCorpus(c) as CC:
        dl, *_ = P.isorank_pairs(CQ, CC, np.repeat(np.arange(len(q)), len(c)), np.tile(np.arange(len(c)), len(q)))
    dl = dl.reshape(len(q), len(c))
    np.testing.assert_array_equal(bd, dl.min(axis=1))
    np.testing.assert_array_equal(bi, dl.argmin(axis=1))
