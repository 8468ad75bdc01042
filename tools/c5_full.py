#!/usr/bin/env python
"""C5 (the north-star config: 20k synthetic CFGs of 16-512 blocks, all-pairs)
at full size on ONE GPU, run as the 8 ranks of an 8-GPU job would run it:
cfgsim_allpairs_split(8) -> each rank's unit range timed with CUDA events,
one after the other on this GPU, then the scatter.  Reports each rank's
device time, max/mean imbalance (the 8-GPU step time is the max), the total
and parity of a random unit sample against the oracle (the checker).

  python tools/c5_full.py [--graphs 20000] [--world 8] [--out gpurun_out/c5_full.json]
"""

from __future__ import annotations

import argparse
import json
import sys
import time
from pathlib import Path

import numpy as np

REPO = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(REPO))


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--graphs", type=int, default=20000)
    ap.add_argument("--world", type=int, default=8)
    ap.add_argument("--parity", type=int, default=1500)
    ap.add_argument("--out", default="gpurun_out/c5_full.json")
    ap.add_argument("--ranks", default=None, help="comma-separated subset of ranks to run (default: all)")
    a = ap.parse_args()
    import torch

    import paper_1707_02423_b200 as P
    from paper_1707_02423_b200 import _native as nat
    from paper_1707_02423_b200 import synth, workload
    t0 = time.time()
    cfg = synth.CONFIGS["c5"]
    mats = synth.random_corpus(a.graphs, cfg["lo"], cfg["hi"], seed=2, weighting=cfg["weighting"])
    print(f"corpus {a.graphs} graphs ({time.time() - t0:.1f} s)", flush=True)
    prm = nat.params(0.85, 1e-9, 1000, "fp64")
    res = {"workload": f"c5: all-pairs IsoRank over {a.graphs} synthetic CFGs, {cfg['lo']}-{cfg['hi']} blocks",
           "world": a.world}
    with P.DeviceCorpus(mats) as C:
        nu = C.n_units()
        b = C.split(a.world)
        st = torch.cuda.current_stream().cuda_stream
        d_lin = torch.empty(nu, dtype=torch.float64, device="cuda")
        it_lin = torch.empty(nu, dtype=torch.int32, device="cuda")
        # warm-up: a small range per kernel family
        nat.check(nat.lib.cfgsim_allpairs_range(C.handle, 0, min(nu, 20000), 0, nat.C.byref(prm), nat.ptr(d_lin),
                                                nat.ptr(it_lin), st))
        nat.check(nat.lib.cfgsim_allpairs_range(C.handle, nu - 20000, nu, 0, nat.C.byref(prm),
                                                nat.ptr(d_lin[nu - 20000:]), nat.ptr(it_lin[nu - 20000:]), st))
        torch.cuda.synchronize()
        ms = []
        ranks = range(a.world) if a.ranks is None else [int(x) for x in a.ranks.split(",")]
        for r in ranks:
            u0, u1 = int(b[r]), int(b[r + 1])
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            nat.check(nat.lib.cfgsim_allpairs_range(C.handle, u0, u1, 0, nat.C.byref(prm), nat.ptr(d_lin[u0:]),
                                                    nat.ptr(it_lin[u0:]), st))
            e1.record()
            torch.cuda.synchronize()
            ms.append(e0.elapsed_time(e1))
            print(f"rank {r}: units [{u0}, {u1}) {u1 - u0} alignments, {ms[-1]:.1f} ms "
                  f"({(u1 - u0) / ms[-1] * 1e3:.0f} pairs/s)", flush=True)
        tot = sum(ms)
        res.update({"units": nu, "bounds": [int(x) for x in b], "ranks_run": list(ranks), "rank_ms": ms})
        if len(ms) == a.world:
            res.update({"total_ms_1gpu": tot, "pairs_per_s_1gpu": nu / tot * 1e3,
                        "imbalance_max_over_mean": max(ms) / (tot / a.world), "projected_step_ms_at_world": max(ms),
                        "projected_pairs_per_s_at_world": nu / max(ms) * 1e3})
        # parity of a random unit sample (the checker, after the timed ranges)
        if a.parity:
            from oracle import ffi
            rng = np.random.default_rng(0)
            lo_u = int(b[min(ranks)])
            hi_u = int(b[max(ranks) + 1])
            us = np.unique(rng.integers(lo_u, hi_u, 2 * a.parity))[: a.parity]
            perm, ai, bi = workload.triangle_units(C.n_nodes)
            ga, gb = perm[ai[us]], perm[bi[us]]
            lo, hi = np.minimum(ga, gb), np.maximum(ga, gb)
            t1 = time.time()
            d_ref, _, it_ref, _ = ffi.iso_batch(P.pack(mats), lo.astype(np.int32), hi.astype(np.int32))
            got_d = d_lin.cpu().numpy()[us]
            got_it = it_lin.cpu().numpy()[us]
            res["parity"] = {"pairs": int(len(us)), "iter_mismatches": int((got_it != it_ref).sum()),
                             "max_rel_err": float(np.max(np.abs(got_d - d_ref) / d_ref)),
                             "oracle_seconds": round(time.time() - t1, 1)}
            print("parity", res["parity"], flush=True)
    Path(a.out).parent.mkdir(parents=True, exist_ok=True)
    Path(a.out).write_text(json.dumps(res, indent=1))
    print(json.dumps({k: v for k, v in res.items() if k != "bounds"}), flush=True)


if __name__ == "__main__":
    main()
