"""Multi-GPU sharding logic on CPU: world-size-2 gloo, oracle as the per-rank
compute (the kernels need a GPU; the split / all-gather / scatter logic does
not)."""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest

from conftest import REPO


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_split_covers_triangle_and_balances():
    from paper_1707_02423_b200.distributed import row_starts, split_units
    rng = np.random.default_rng(0)
    n = rng.integers(16, 65, 300)
    for world in (1, 2, 3, 4, 8):
        b = split_units(n, world)
        assert b[0] == 0 and b[-1] == row_starts(len(n))[-1]
        assert (np.diff(b) >= 0).all()
    # balance of the measured cost model (csrc/cost_model.h) within 2% at 8 ranks
    from paper_1707_02423_b200.distributed import unit_cost_us
    from paper_1707_02423_b200.workload import triangle_units
    perm, a, _ = triangle_units(n)
    cost = unit_cost_us(n[perm[a]])
    b = split_units(n, 8)
    per = np.array([cost[b[r]:b[r + 1]].sum() for r in range(8)])
    assert per.max() / per.mean() < 1.02


def test_scatter_and_unit_pairs_direction():
    from paper_1707_02423_b200.distributed import scatter_units, unit_pairs
    n = np.array([5, 9, 9, 3])
    lo, hi = unit_pairs(n, 0, 10)
    assert (lo <= hi).all()
    assert len(set(zip(lo.tolist(), hi.tolist()))) == 10  # every unordered pair once (incl. diagonal)
    vals = np.arange(10, dtype=float)
    m = scatter_units(n, vals)
    np.testing.assert_array_equal(m, m.T)
    for u in range(10):
        assert m[lo[u], hi[u]] == vals[u]


def _worker(rank, world, port, out_path):
    import torch.distributed as dist
    import sys
    sys.path.insert(0, str(REPO))
    from oracle import ffi
    from paper_1707_02423_b200 import synth
    from paper_1707_02423_b200.packing import pack
    from paper_1707_02423_b200.distributed import allpairs_sharded, unit_pairs

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    mats = synth.random_corpus(14, 4, 12, seed=3)
    n = np.array([m.shape[0] for m in mats])
    packed = pack(mats)

    def compute(u0, u1):
        lo, hi = unit_pairs(n, u0, u1)
        d, *_ = ffi.iso_batch(packed, lo.astype(np.int32), hi.astype(np.int32), threads=1)
        return d

    m = allpairs_sharded(n, compute)
    if rank == 0:
        np.save(out_path, m)
    dist.destroy_process_group()


def test_gloo_world2_matches_single_rank(tmp_path):
    import torch.multiprocessing as mp
    import sys
    sys.path.insert(0, str(REPO))
    from oracle import ffi
    from paper_1707_02423_b200 import synth
    from paper_1707_02423_b200.packing import pack

    out = tmp_path / "m.npy"
    mp.start_processes(_worker, args=(2, _free_port(), str(out)), nprocs=2, start_method="spawn")
    m2 = np.load(out)
    mats = synth.random_corpus(14, 4, 12, seed=3)
    k = len(mats)
    iu, ju = np.triu_indices(k)
    d, *_ = ffi.iso_batch(pack(mats), iu.astype(np.int32), ju.astype(np.int32), threads=1)
    ref = np.empty((k, k))
    ref[iu, ju] = d
    ref[ju, iu] = d
    np.testing.assert_array_equal(m2, ref)  # bitwise: schedule-independent


def test_merge_best_lexicographic_ties():
    from paper_1707_02423_b200.distributed import merge_best
    d = np.array([[1.5, 1.2, 2.0], [1.5, 1.3, 1.9], [1.4, 1.2, 2.0]])
    i = np.array([[3, 1, 0], [10, 12, 11], [25, 27, 20]], np.int64)
    bd, bi = merge_best(d, i)
    np.testing.assert_array_equal(np.asarray(bd), [1.4, 1.2, 1.9])
    np.testing.assert_array_equal(np.asarray(bi), [25, 1, 11])  # tie on 1.2 -> lowest corpus index


def _nearest_worker(rank, world, port, out_path):
    import torch.distributed as dist
    import sys
    sys.path.insert(0, str(REPO))
    from oracle import ffi
    from paper_1707_02423_b200 import synth
    from paper_1707_02423_b200.packing import pack
    from paper_1707_02423_b200.distributed import nearest_sharded

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    q = synth.random_corpus(5, 4, 10, seed=7)
    c = synth.random_corpus(23, 3, 12, seed=8) + [q[2].copy()]  # an exact match (d = min)
    packed = pack(q + c)

    def shard(c0, c1):
        bd, bi = [], []
        for i in range(len(q)):
            ia = np.full(c1 - c0, i, np.int32)
            ib = np.arange(len(q) + c0, len(q) + c1, dtype=np.int32)
            d, *_ = ffi.iso_batch(packed, ia, ib, threads=1)
            j = int(np.argmin(d))
            bd.append(d[j])
            bi.append(c0 + j)
        return np.array(bd), np.array(bi, np.int64)

    bd, bi = nearest_sharded(len(c), shard)
    if rank == 0:
        np.save(out_path, np.concatenate([bd, bi.astype(float)]))
    dist.destroy_process_group()


def test_gloo_world2_nearest_matches_single_rank(tmp_path):
    import torch.multiprocessing as mp
    import sys
    sys.path.insert(0, str(REPO))
    from oracle import ffi
    from paper_1707_02423_b200 import synth
    from paper_1707_02423_b200.packing import pack

    out = tmp_path / "n.npy"
    mp.start_processes(_nearest_worker, args=(2, _free_port(), str(out)), nprocs=2, start_method="spawn")
    got = np.load(out)
    q = synth.random_corpus(5, 4, 10, seed=7)
    c = synth.random_corpus(23, 3, 12, seed=8) + [q[2].copy()]
    packed = pack(q + c)
    for i in range(len(q)):
        ia = np.full(len(c), i, np.int32)
        ib = np.arange(len(q), len(q) + len(c), dtype=np.int32)
        d, *_ = ffi.iso_batch(packed, ia, ib, threads=1)
        assert got[i] == d.min()
        assert int(got[len(q) + i]) == int(np.argmin(d))
