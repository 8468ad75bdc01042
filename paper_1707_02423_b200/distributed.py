"""All-pairs ISO across GPUs: cost-balanced triangle ranges + one all-gather.

SURVEY §8(e): pairs are independent, so each rank aligns a contiguous range
of units of the size-sorted upper triangle (no collective while aligning);
the only exchange is one ``all_gather_into_tensor`` of the per-rank score
tiles (NCCL over NVLink on GPUs, gloo in the CPU tests), after which every
rank scatters the unit vector into the K x K matrix.  Per-pair arithmetic
does not depend on the schedule, so results are bitwise identical for any
world size.

The unit enumeration and the split mirror ``cfgsim_allpairs_split`` /
``cfgsim_allpairs_scatter`` in ``csrc/cfgsim.cu`` (checked against each other
in the GPU tests).
"""

from __future__ import annotations

from typing import Callable

import numpy as np

from .workload import triangle_units


def row_starts(k: int) -> np.ndarray:
    return np.concatenate([[0], np.cumsum(np.arange(k, 0, -1))]).astype(np.int64)


def _cost_table():
    """(N samples, us per unit) of csrc/cost_model.h — the one table the C
    split and this mirror share."""
    import re
    from pathlib import Path
    txt = (Path(__file__).resolve().parent / "csrc" / "cost_model.h").read_text()
    body = txt[txt.index("COST_TABLE_BEGIN"):txt.index("COST_TABLE_END")]
    ns = [int(x) for x in re.search(r"kCostN\[\] = \{([^}]*)\}", body).group(1).split(",")]
    us = [float(x) for x in re.search(r"kCostUs\[\] = \{([^}]*)\}", body).group(1).split(",")]
    return np.array(ns, np.float64), np.array(us, np.float64)


def unit_cost_us(n) -> np.ndarray:
    """Measured per-unit cost vs N (cost_model.h: piecewise linear, clamped),
    with the C routine's operation order (bitwise the same costs, hence the
    same split)."""
    xs, ys = _cost_table()
    n = np.asarray(n, np.float64)
    i = np.clip(np.searchsorted(xs, n, side="left"), 1, len(xs) - 1)
    t = (n - xs[i - 1]) / (xs[i] - xs[i - 1])
    out = ys[i - 1] + t * (ys[i] - ys[i - 1])
    out = np.where(n <= xs[0], ys[0], out)
    return np.where(n > xs[-1], ys[-1], out)


def split_units(n_nodes: np.ndarray, world: int) -> np.ndarray:
    """world+1 unit boundaries balancing the measured cost per rank
    (unit_cost_us of the row's N; rows sorted by n descending, stable) —
    mirrors cfgsim_allpairs_split."""
    n_nodes = np.asarray(n_nodes)
    k = len(n_nodes)
    ns = n_nodes[np.argsort(-n_nodes, kind="stable")].astype(np.float64)
    rs = row_starts(k)
    cost = unit_cost_us(ns)
    per_row = (k - np.arange(k)) * cost
    cum = np.concatenate([[0.0], np.cumsum(per_row)])
    total = cum[-1]
    bounds = np.zeros(world + 1, np.int64)
    for r in range(1, world):
        target = total * r / world
        a = int(np.searchsorted(cum, target, side="right")) - 1
        a_c = min(a, k - 1)
        per = cost[a_c]
        u = rs[a] + int(np.ceil((target - cum[a]) / per))
        u = min(u, rs[min(a + 1, k)])
        bounds[r] = max(u, bounds[r - 1])
    bounds[world] = rs[k]
    return bounds


def scatter_units(n_nodes: np.ndarray, d_units: np.ndarray) -> np.ndarray:
    """Unit-linear (unordered, symmetric) scores -> K x K matrix, caller's order."""
    perm, a, b = triangle_units(n_nodes)
    k = len(n_nodes)
    out = np.empty((k, k))
    out[perm[a], perm[b]] = d_units
    out[perm[b], perm[a]] = d_units
    return out


def unit_pairs(n_nodes: np.ndarray, u0: int, u1: int) -> tuple[np.ndarray, np.ndarray]:
    """Graph indices (low id, high id) of units [u0, u1) — the direction the
    kernels align in."""
    perm, a, b = triangle_units(n_nodes)
    ga, gb = perm[a[u0:u1]], perm[b[u0:u1]]
    return np.minimum(ga, gb), np.maximum(ga, gb)


def allpairs_sharded(n_nodes: np.ndarray, compute_range: Callable[[int, int], np.ndarray], *, group=None,
                     device=None):
    """Run ``compute_range(u0, u1) -> d[u1-u0]`` on this rank's share and
    all-gather; returns the K x K matrix on every rank.

    ``compute_range`` is the GPU kernel call in production
    (``DeviceCorpus`` + ``cfgsim_allpairs_range``) and the CPU oracle in the
    gloo tests."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    bounds = split_units(n_nodes, world)
    u0, u1 = int(bounds[rank]), int(bounds[rank + 1])
    chunk = int(max(bounds[1:] - bounds[:-1]))
    local = np.zeros(chunk)
    local[: u1 - u0] = compute_range(u0, u1)
    dev = device if device is not None else torch.device("cpu")
    t_local = torch.as_tensor(local, dtype=torch.float64, device=dev)
    if world > 1:
        gathered = torch.empty(world * chunk, dtype=torch.float64, device=dev)
        dist.all_gather_into_tensor(gathered, t_local, group=group)
        g = gathered.cpu().numpy()
        full = np.concatenate([g[r * chunk: r * chunk + int(bounds[r + 1] - bounds[r])] for r in range(world)])
    else:
        full = local[: u1 - u0]
    return scatter_units(n_nodes, full)


def gpu_compute_range(corpus, params, stream=None):
    """compute_range backed by the sm_100a kernels (device-resident corpus)."""
    import torch

    from . import _native as nat

    def run(u0: int, u1: int) -> np.ndarray:
        out = torch.empty(max(u1 - u0, 1), dtype=torch.float64, device=torch.device("cuda", corpus.device))
        if u1 > u0:
            nat.check(nat.lib.cfgsim_allpairs_range(corpus.handle, u0, u1, 0, nat.C.byref(params), nat.ptr(out),
                                                    None, stream))
        torch.cuda.synchronize(corpus.device)
        return out[: u1 - u0].cpu().numpy()

    return run


def merge_best(d, idx):
    """Lexicographic (d, index) minimum over shards: d, idx are [world, nq]
    tensors (or arrays) of per-shard best matches; returns (best_d, best_idx)
    — np.argmin's lowest-index tie rule over the concatenated corpus."""
    import torch

    d = torch.as_tensor(d)
    idx = torch.as_tensor(idx)
    best = d.min(dim=0).values
    cand = torch.where(d == best.unsqueeze(0), idx, torch.full_like(idx, torch.iinfo(idx.dtype).max))
    return best, cand.min(dim=0).values


def nearest_sharded(n_corpus: int, compute_shard: Callable[[int, int], tuple], *, group=None, device=None):
    """Query-vs-corpus best match with the corpus split into world shards
    (SURVEY §8(e)): ``compute_shard(c0, c1) -> (best_d[nq], best_idx[nq])``
    on this rank's shard, then one all-gather of the candidates and the
    lexicographic (d, index) minimum on every rank."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    bounds = np.linspace(0, n_corpus, world + 1).astype(np.int64)
    bd, bi = compute_shard(int(bounds[rank]), int(bounds[rank + 1]))
    dev = device if device is not None else torch.device("cpu")
    td = torch.as_tensor(np.asarray(bd, np.float64), device=dev)
    ti = torch.as_tensor(np.asarray(bi, np.int64), device=dev)
    if world == 1:
        return td.cpu().numpy(), ti.cpu().numpy()
    gd = torch.empty(world * len(td), dtype=torch.float64, device=dev)
    gi = torch.empty(world * len(ti), dtype=torch.int64, device=dev)
    dist.all_gather_into_tensor(gd, td, group=group)
    dist.all_gather_into_tensor(gi, ti, group=group)
    best, idx = merge_best(gd.view(world, -1), gi.view(world, -1))
    return best.cpu().numpy(), idx.cpu().numpy()


def _all_gather(dst, src, group=None):
    """``all_gather_into_tensor`` on the group's backend: NCCL gathers device
    tensors over NVLink in place; gloo (the CPU multi-process tests, and
    several ranks sharing one GPU) gathers host copies."""
    import torch.distributed as dist

    if src.is_cuda and dist.get_backend(group) == "gloo":
        import torch
        g = torch.empty(dst.shape, dtype=dst.dtype)
        dist.all_gather_into_tensor(g, src.cpu(), group=group)
        dst.copy_(g)
    else:
        dist.all_gather_into_tensor(dst, src, group=group)


def _world(group):
    import torch.distributed as dist
    if dist.is_available() and dist.is_initialized():
        return dist.get_world_size(group), dist.get_rank(group)
    return 1, 0


def pairwise_sharded(matrices, *, alpha: float = 0.85, tol: float = 1e-9, max_iter: int = 1000,
                     precision: str = "fp64", device: int | None = None, group=None):
    """``pairwise(matrices, MeasureId.ISO)`` across the ranks of a
    torch.distributed group (one GPU per rank): each rank uploads the corpus,
    aligns its cost-balanced share of the size-sorted upper triangle, one
    all-gather (NCCL over NVLink) assembles the unit vector, the K x K matrix
    is scattered on the device and returned on every rank.  Same result as
    ``pairwise`` bitwise, for any world size."""
    import torch
    import torch.distributed as dist

    from . import _native as nat
    from .corpus import DeviceCorpus
    from .errors import DuplicateKernel
    from .similarity import MeasureId, PairwiseMatrix, _check_alpha

    if len(matrices) < 2:
        raise ValueError("pairwise comparison needs at least 2 kernels")
    ordered = sorted(matrices, key=lambda m: m.kernel_id)
    ids = tuple(m.kernel_id for m in ordered)
    if len(set(ids)) != len(ids):
        raise DuplicateKernel("duplicate kernel_id in pairwise input")
    _check_alpha(alpha)
    world, rank = _world(group)
    dev_idx = nat.default_device() if device is None else int(device)
    dev = torch.device("cuda", dev_idx)
    prm = nat.params(alpha, tol, max_iter, precision)
    k = len(ordered)
    with DeviceCorpus(ordered, dev_idx) as C:
        bounds = C.split(world)
        u0, u1 = int(bounds[rank]), int(bounds[rank + 1])
        chunk = max(int(max(bounds[1:] - bounds[:-1])), 1)
        st = torch.cuda.current_stream(dev).cuda_stream
        d_lin = torch.zeros(chunk, dtype=torch.float64, device=dev)
        if u1 > u0:
            nat.check(nat.lib.cfgsim_allpairs_range(C.handle, u0, u1, 0, nat.C.byref(prm), nat.ptr(d_lin), None, st))
        if world > 1:
            gathered = torch.empty(world * chunk, dtype=torch.float64, device=dev)
            _all_gather(gathered, d_lin, group)
            full = torch.cat([gathered[r * chunk:r * chunk + int(bounds[r + 1] - bounds[r])] for r in range(world)])
        else:
            full = d_lin[: u1 - u0]
        scores_d = torch.empty((k, k), dtype=torch.float64, device=dev)
        nat.check(nat.lib.cfgsim_allpairs_scatter(C.handle, 0, nat.ptr(full), None, nat.ptr(scores_d), None, st))
        scores = scores_d.cpu().numpy()
    return PairwiseMatrix(measure=MeasureId.ISO, kernel_ids=ids, scores=scores, scaled=False)


def nearest_gpu_sharded(queries, corpus, *, alpha: float = 0.85, tol: float = 1e-9, max_iter: int = 1000,
                        precision: str = "fp64", device: int | None = None, group=None):
    """``nearest(queries, corpus)`` across the ranks of a torch.distributed
    group: rank r searches corpus shard r (``cfgsim_nearest`` on [c0, c1)),
    one all-gather of the (d, index) candidates, lexicographic minimum."""
    import torch
    import torch.distributed as dist

    from . import _native as nat
    from .corpus import DeviceCorpus
    from .similarity import _check_alpha

    _check_alpha(alpha)
    world, rank = _world(group)
    dev_idx = nat.default_device() if device is None else int(device)
    dev = torch.device("cuda", dev_idx)
    prm = nat.params(alpha, tol, max_iter, precision)
    nq, nc = len(queries), len(corpus)
    bounds = np.linspace(0, nc, world + 1).astype(np.int64)
    c0, c1 = int(bounds[rank]), int(bounds[rank + 1])
    bd = torch.full((nq,), float("inf"), dtype=torch.float64, device=dev)
    bi = torch.full((nq,), np.iinfo(np.int64).max, dtype=torch.int64, device=dev)
    with DeviceCorpus(queries, dev_idx) as Q, DeviceCorpus(corpus, dev_idx) as Cc:
        st = torch.cuda.current_stream(dev).cuda_stream
        if c1 > c0:
            nat.check(nat.lib.cfgsim_nearest(Q.handle, Cc.handle, c0, c1, nat.C.byref(prm), nat.ptr(bd), nat.ptr(bi),
                                             st))
        if world > 1:
            gd = torch.empty(world * nq, dtype=torch.float64, device=dev)
            gi = torch.empty(world * nq, dtype=torch.int64, device=dev)
            _all_gather(gd, bd, group)
            _all_gather(gi, bi, group)
            bd, bi = merge_best(gd.view(world, nq), gi.view(world, nq))
        return bd.cpu().numpy(), bi.cpu().numpy()
