#!/usr/bin/env python
"""Summarise an A/B run directory (tools/gpu_ab.sh): bench values + stage-2 phase shares."""
import json
import re
import sys
from pathlib import Path

d = Path(sys.argv[1])
for f in sorted(d.glob("bench_*.jsonl")):
    try:
        j = json.loads(f.read_text().strip().splitlines()[-1])
        e = j.get("e2e") or {}
        print(f"{f.stem:22s} {j['value']:>14.0f} {j['unit']}  {j['ms_per_step']:9.2f} ms/step  e2e {e.get('value', 0):>12.0f}")
    except Exception as ex:  # noqa: BLE001
        print(f.stem, "unreadable", ex)
for f in sorted(d.glob("pytest*.txt")):
    print(f.name, " ".join(f.read_text().strip().splitlines()[-2:]))
ph = d / "phases_c2.txt"
if ph.exists():
    tp, tc, P, C = [0.0] * 5, [0.0] * 2, 0.0, 0.0
    for line in ph.read_text().splitlines():
        m = re.search(r"N=(\d+).*wait/claim ([\d.]+)% bracket\+delta ([\d.]+)% stage\+mma\+keys ([\d.]+)% row-orders "
                      r"([\d.]+)% tail ([\d.]+)% \(([\d.e+]+) cyc\) \| consumer: wait ([\d.]+)% rounds ([\d.]+)% \(([\d.e+]+)", line)
        if not m:
            continue
        v = list(map(float, m.groups()))
        for k in range(5):
            tp[k] += v[1 + k] * v[6] / 100
        tc[0] += v[7] * v[9] / 100
        tc[1] += v[8] * v[9] / 100
        P += v[6]
        C += v[9]
        if int(v[0]) in (16, 24, 32, 48, 64):
            print("  N=%d producer wait %.1f bracket %.1f mma %.1f orders %.1f | consumer wait %.1f  (%.2e cyc)" % (
                v[0], v[1], v[2], v[3], v[4], v[7], v[6]))
    print("stage-2 total: producer", [round(100 * x / P, 1) for x in tp], f"{P:.3e} cyc; consumer wait/rounds",
          [round(100 * x / C, 1) for x in tc])
