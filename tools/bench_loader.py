"""Loader throughput: kernels/s from listing + profile
text to transition matrices, native (csrc/loader.cpp through
matrices_from_listings) vs the reference's Python path (cli.py:55-74 +
matrix.py:45-71, imported from /root/reference when present).

    python tools/bench_loader.py [--kernels 4000] [--blocks 64] [--threads 0]
"""

from __future__ import annotations

import argparse
import json
import os
import random
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

OPS = ["FADD R0, R1, R2", "DFMA R6, R6, R7, R8", "IMAD.WIDE R2, R2, R3, R4", "LDG.E.64 R4, [R2.64+0x10]",
       "MOV R5, R6", "ISETP.GE.AND P0, PT, R1, R2, PT", "SHF.R.U32 R4, R4, 0x1, RZ", "STG.E [R2], R4"]


def synth(rng: random.Random, kid: str, nb: int) -> tuple[str, str, str]:
    lines, offs, off = [], [], 0x10
    for b in range(nb):
        lines.append(f".L_{b}:")
        for _ in range(rng.randint(2, 12)):
            lines.append(f"        /*{off:04x}*/ {rng.choice(OPS)} ;")
            offs.append(off)
            off += 16
        if b == nb - 1:
            lines.append(f"        /*{off:04x}*/ EXIT ;")
        else:
            t = rng.randrange(nb)
            lines.append(f"        /*{off:04x}*/ {rng.choice(['@P0 ', '@!P1 ', ''])}BRA `(.L_{t}) ;")
        off += 16
    prof = [f"kernel {kid}"] + [f"sample {o:x} {rng.randrange(1, 500)}" for o in rng.sample(offs, len(offs) // 3)]
    return kid, "\n".join(lines) + "\n", "\n".join(prof) + "\n"


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--kernels", type=int, default=4000)
    ap.add_argument("--blocks", type=int, default=64)
    ap.add_argument("--threads", type=int, default=0)
    ap.add_argument("--ref-sample", type=int, default=400)
    args = ap.parse_args()
    rng = random.Random(5)
    ks = [synth(rng, f"k{i}.s.f.m", rng.randint(args.blocks // 2, args.blocks)) for i in range(args.kernels)]
    from paper_1707_02423_b200.loader import matrices_from_listings
    matrices_from_listings(ks[:50])
    t0 = time.perf_counter()
    mats = matrices_from_listings(ks, threads=args.threads)
    t_nat = time.perf_counter() - t0
    line = {"kernels": args.kernels, "blocks": f"{args.blocks // 2}-{args.blocks}",
            "native_kernels_per_s": args.kernels / t_nat, "threads": args.threads or os.cpu_count()}
    if Path("/root/reference/pkg/src").exists():
        sys.path.insert(0, "/root/reference/pkg/src")
        from sasscfg.cfg import build_cfg
        from sasscfg.matrix import transition_matrix
        from sasscfg.profile import attribute_profile, parse_profiles
        from sasscfg.sass import parse_listing
        import numpy as np
        sample = ks[: args.ref_sample]
        t0 = time.perf_counter()
        ref = [transition_matrix(attribute_profile(build_cfg(parse_listing(l, k)), parse_profiles(p)[k]))
               for k, l, p in sample]
        t_ref = time.perf_counter() - t0
        line["reference_kernels_per_s"] = len(sample) / t_ref
        line["reference_sample"] = len(sample)
        line["speedup"] = line["native_kernels_per_s"] / line["reference_kernels_per_s"]
        line["identical"] = all(np.array_equal(a.entries, b.entries) and a.ordering == b.ordering
                                for a, b in zip(mats, ref))
    print(json.dumps(line))


if __name__ == "__main__":
    main()
