"""The production multi-GPU paths at world size 2 (missing).

Two ranks (torch.multiprocessing, gloo rendezvous on 127.0.0.1) share the
one GPU of the test box: each uploads the corpus, runs its share through the
sm_100a kernels (``cfgsim_allpairs_range`` / ``cfgsim_nearest``), the shares
are all-gathered and scattered exactly as on an 8-GPU NVLink node — only the
transport differs (gloo host copies instead of NCCL).  SPEC.md:456 requires
results independent of the degree of parallelism: both ranks' outputs must
equal the single-process ``pairwise`` / ``nearest`` bit for bit.  Also pins
the Python mirror of the unit split / scatter to the C ABI's.
"""

from __future__ import annotations

import os
import socket
import sys

import numpy as np
import pytest

from conftest import REPO

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _corpus():
    sys.path.insert(0, str(REPO))
    from paper_1707_02423_b200 import synth
    # all three all-pairs tiers: two-stage (N <= 64), low-rank (<= 128), large-N
    return (synth.random_corpus(40, 16, 64, seed=11) + synth.random_corpus(14, 65, 128, seed=12)
            + synth.random_corpus(6, 129, 300, seed=13, weighting="observed"))


def _worker(rank, world, port, out_dir):
    import torch.distributed as dist
    sys.path.insert(0, str(REPO))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_1707_02423_b200 as P
    from paper_1707_02423_b200 import distributed as D, synth
    mats = _corpus()
    tms = [P.TransitionMatrix(f"k{i:03d}.s.w2", m, tuple(range(len(m))), P.ROW_STOCHASTIC) for i, m in enumerate(mats)]
    pm = D.pairwise_sharded(tms, device=0)
    q = synth.random_corpus(9, 16, 64, seed=21)
    bd, bi = D.nearest_gpu_sharded(q, mats[:40], device=0)
    np.savez(os.path.join(out_dir, f"rank{rank}.npz"), scores=pm.scores, bd=bd, bi=bi)
    dist.barrier()
    dist.destroy_process_group()


def test_world2_sharded_equals_single_process(gpu, tmp_path):
    import torch.multiprocessing as mp
    import paper_1707_02423_b200 as P
    from paper_1707_02423_b200 import synth
    mp.spawn(_worker, args=(2, _free_port(), str(tmp_path)), nprocs=2, join=True)
    mats = _corpus()
    tms = [P.TransitionMatrix(f"k{i:03d}.s.w2", m, tuple(range(len(m))), P.ROW_STOCHASTIC) for i, m in enumerate(mats)]
    ref = P.pairwise(tms, P.MeasureId.ISO).scores
    q = synth.random_corpus(9, 16, 64, seed=21)
    rbd, rbi = P.nearest(q, mats[:40])
    for r in range(2):
        got = np.load(tmp_path / f"rank{r}.npz")
        np.testing.assert_array_equal(got["scores"], ref)
        np.testing.assert_array_equal(got["bd"], rbd)
        np.testing.assert_array_equal(got["bi"], rbi)


@pytest.mark.parametrize("world", [1, 2, 3, 8])
def test_python_split_and_scatter_mirror_the_abi(gpu, world):
    import torch

    import paper_1707_02423_b200 as P
    from paper_1707_02423_b200 import _native as nat
    from paper_1707_02423_b200 import distributed as D
    mats = _corpus()
    n = np.array([len(m) for m in mats])
    with P.DeviceCorpus(mats) as C:
        np.testing.assert_array_equal(C.split(world), D.split_units(n, world))
        units = C.n_units()
        vals = torch.arange(units, dtype=torch.float64, device="cuda:0") + 1.0
        out = torch.empty((len(mats), len(mats)), dtype=torch.float64, device="cuda:0")
        nat.check(nat.lib.cfgsim_allpairs_scatter(C.handle, 0, nat.ptr(vals), None, nat.ptr(out), None, None))
        torch.cuda.synchronize()
        np.testing.assert_array_equal(out.cpu().numpy(), D.scatter_units(n, vals.cpu().numpy()))
