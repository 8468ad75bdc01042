"""Seeded synthetic CFG corpora (row-stochastic block-transition matrices).

Mirrors the reference's own synthetic inputs so the benchmark graphs have
the reference's structure, not just its sizes:

* block terminators drawn uniformly from {bra, cond_bra, pred_exit, fall,
  exit}, last block exits, one random branch target per block
  (``pkg/tests/helpers.py:54-82``);
* edges as ``build_cfg`` emits them (``pkg/src/sasscfg/cfg.py:139-183``),
  STOP edges dropped from the matrix (``matrix.py:57-59``);
* rows/columns in reverse post-order from START, unreachable blocks appended
  in listing order (``cfg.py:86-117``);
* edge weights by flow balance over sampled block counts U[0,200) for 80% of
  graphs, uniform static otherwise (``helpers.py:89-99``,
  ``profile.py:211-231``), or observed edge counts U[1,1000) on every edge
  (config 4, ``profile.py:197-210``);
* ``row_stochastic`` normalisation (``matrix.py:61-64``).

``tests/test_synth.py`` checks, in the build container, that these matrices
are bit-identical to what the reference pipeline (listing -> ``build_cfg`` ->
``attribute_profile`` -> ``transition_matrix``) produces for the same
structure.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

KINDS = ("bra", "cond_bra", "pred_exit", "fall", "exit")


@dataclass(frozen=True)
class CfgShape:
    """Block-level structure of one synthetic kernel (STOP == n_blocks)."""

    n_blocks: int
    kinds: tuple[str, ...]
    targets: tuple[int, ...]
    block_counts: tuple[int, ...] | None  # sampled PC counts, None = no profile
    edge_counts: dict | None = None  # observed (src, dst) -> count


def successors(shape: CfgShape) -> list[list[int]]:
    """Per block, sorted successor ids incl. STOP (cfg.py:139-183, profile.py:159-167)."""
    n = shape.n_blocks
    out = []
    for b in range(n):
        kind = shape.kinds[b]
        fall = b + 1 if b + 1 < n else n
        if kind == "fall":
            s = {fall}
        elif kind == "bra":
            s = {shape.targets[b]}
        elif kind == "cond_bra":
            s = {shape.targets[b], fall}
        elif kind == "pred_exit":
            s = {n, fall}
        else:  # exit
            s = {n}
        out.append(sorted(s))
    return out


def canonical_order(shape: CfgShape, succ: list[list[int]]) -> list[int]:
    """Reverse post-order from START (cfg.py:86-117)."""
    n = shape.n_blocks
    real = [[t for t in s if t != n] for s in succ]
    post: list[int] = []
    seen = {0}
    stack = [(0, iter(real[0]))]
    while stack:
        node, it = stack[-1]
        child = next(it, None)
        if child is None:
            stack.pop()
            post.append(node)
        elif child not in seen:
            seen.add(child)
            stack.append((child, iter(real[child])))
    order = list(reversed(post))
    rest = sorted(set(range(n)) - set(order))
    return order + rest


def _pairwise_sum(a: np.ndarray) -> float:
    return float(np.sum(a))


def transition_matrix(shape: CfgShape) -> np.ndarray:
    """Row-stochastic block-transition matrix in canonical order."""
    n = shape.n_blocks
    succ = successors(shape)
    edge: dict[tuple[int, int], float] = {}
    if shape.edge_counts is not None:  # observed (profile.py:197-210)
        for b in range(n):
            for t in succ[b]:
                edge[(b, t)] = float(shape.edge_counts.get((b, t), 0.0))
    elif shape.block_counts is not None and any(c > 0 for c in shape.block_counts):
        bc = shape.block_counts  # flow balance (profile.py:211-225)
        for b in range(n):
            targets = succ[b]
            weights = [bc[t] if t < n else 0 for t in targets]
            wsum = sum(weights)
            for t, w in zip(targets, weights):
                share = w / wsum if wsum > 0 else 1.0 / len(targets)
                edge[(b, t)] = bc[b] * share
    else:  # uniform static (profile.py:226-231)
        for b in range(n):
            for t in succ[b]:
                edge[(b, t)] = 1.0 / len(succ[b])
    order = canonical_order(shape, succ)
    index = {blk: i for i, blk in enumerate(order)}
    counts = np.zeros((n, n))
    for (src, dst), c in edge.items():
        if dst < n:
            counts[index[src], index[dst]] += c
    row_sums = counts.sum(axis=1, keepdims=True)  # matrix.py:62-64
    with np.errstate(invalid="ignore", divide="ignore"):
        return np.where(row_sums > 0, counts / np.where(row_sums > 0, row_sums, 1.0), 0.0)


def random_shape(rng: np.random.Generator, n_blocks: int, weighting: str = "sampled") -> CfgShape:
    kinds = [KINDS[int(k)] for k in rng.integers(0, len(KINDS), n_blocks)]
    kinds[-1] = "exit"
    targets = tuple(int(t) for t in rng.integers(0, n_blocks, n_blocks))
    if weighting == "observed":
        shape = CfgShape(n_blocks, tuple(kinds), targets, None)
        succ = successors(shape)
        ec = {}
        for b in range(n_blocks):
            for t in succ[b]:
                ec[(b, t)] = int(rng.integers(1, 1000))
        return CfgShape(n_blocks, tuple(kinds), targets, None, ec)
    bc = None
    if weighting == "sampled" and rng.random() < 0.8:
        bc = tuple(int(c) for c in rng.integers(0, 200, n_blocks))
    return CfgShape(n_blocks, tuple(kinds), targets, bc)


def random_corpus(n_graphs: int, lo: int, hi: int, seed: int = 0, weighting: str = "sampled") -> list[np.ndarray]:
    """``n_graphs`` matrices with block counts uniform in [lo, hi]."""
    rng = np.random.default_rng(seed)
    sizes = rng.integers(lo, hi + 1, n_graphs)
    return [transition_matrix(random_shape(rng, int(n), weighting)) for n in sizes]


# Named benchmark configurations (BASELINE.json "configs").
CONFIGS = {
    "c2": dict(n_graphs=2000, lo=16, hi=64, weighting="sampled"),
    "c3_queries": dict(n_graphs=1000, lo=16, hi=64, weighting="sampled"),
    "c3_corpus": dict(n_graphs=100_000, lo=16, hi=64, weighting="sampled"),
    "c4": dict(n_graphs=1000, lo=256, hi=1024, weighting="observed"),
    "c5": dict(n_graphs=20_000, lo=16, hi=512, weighting="sampled"),
}
