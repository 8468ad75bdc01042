#!/usr/bin/env python
"""Golden vectors for the synthetic corpus generator (paper_1707_02423_b200/synth.py).

For seeded CfgShapes (all three weightings, 1..96 blocks) this writes each
shape as a SASS listing in the reference grammar (one label per block, the
terminators of ``pkg/tests/helpers.py:54-82``), runs the reference pipeline
on it — ``parse_listing`` -> ``build_cfg`` -> ``attribute_profile`` (sampled
block counts as PC samples at block starts, or observed edge records) ->
``transition_matrix(mode=row_stochastic)`` — and stores the reference's
matrix.  ``tests/test_synth.py`` checks synth.transition_matrix against these
bitwise.  Run in the build container (needs /root/reference):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_synth.py
"""

from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

REPO = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(REPO))
sys.path.insert(0, "/root/reference/pkg/src")

from paper_1707_02423_b200 import synth  # noqa: E402

CASES = 240


def shapes():
    """The seeded shapes: (seed, n_blocks, weighting) -> CfgShape."""
    rng = np.random.default_rng(1234)
    out = []
    for i in range(CASES):
        n = int(rng.integers(1, 97))
        wt = ("sampled", "observed", "static")[i % 3]
        out.append(synth.random_shape(np.random.default_rng(10_000 + i), n, wt))
    return out


def listing(shape: synth.CfgShape) -> tuple[str, list[int]]:
    """Listing text and each block's start offset."""
    lines, starts, off = [], [], 0x10
    for b in range(shape.n_blocks):
        lines.append(f".L_{b}:")
        starts.append(off)
        lines.append(f"        /*{off:04x}*/ MOV R5, R6 ;")
        off += 0x10
        kind, t = shape.kinds[b], shape.targets[b]
        term = {"bra": f"BRA `(.L_{t})", "cond_bra": f"@P1 BRA `(.L_{t})", "pred_exit": "@!P2 EXIT",
                "exit": "EXIT"}.get(kind)
        if term:
            lines.append(f"        /*{off:04x}*/ {term} ;")
            off += 0x10
    return "\n".join(lines) + "\n", starts


def reference_matrix(shape: synth.CfgShape) -> np.ndarray:
    from sasscfg.cfg import build_cfg
    from sasscfg.matrix import ROW_STOCHASTIC, transition_matrix
    from sasscfg.profile import KernelProfile, attribute_profile
    from sasscfg.sass import parse_listing

    kid = "syn.synth.k.k"
    text, starts = listing(shape)
    cfg = build_cfg(parse_listing(text, kid), arch="synth")
    assert cfg.n_blocks == shape.n_blocks
    if shape.edge_counts is not None:
        n = shape.n_blocks
        recs = {(f"B{s}", "STOP" if t == n else f"B{t}"): c for (s, t), c in shape.edge_counts.items()}
        prof = KernelProfile(kernel_id=kid, edge_counts=recs)
    elif shape.block_counts is not None:
        prof = KernelProfile(kernel_id=kid, samples={starts[b]: c for b, c in enumerate(shape.block_counts) if c})
    else:
        prof = KernelProfile(kernel_id=kid)
    return np.asarray(transition_matrix(attribute_profile(cfg, prof), ROW_STOCHASTIC).entries, dtype=np.float64)


def main():
    mats = [reference_matrix(s) for s in shapes()]
    sizes = np.array([m.shape[0] for m in mats], np.int32)
    flat = np.concatenate([m.ravel() for m in mats])
    np.savez_compressed(REPO / "tests" / "golden" / "synth_ref.npz", sizes=sizes, flat=flat)
    print(f"wrote {len(mats)} reference matrices ({int((sizes ** 2).sum())} entries)")


if __name__ == "__main__":
    main()
