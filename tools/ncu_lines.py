#!/usr/bin/env python
"""Attribute ncu warp-stall samples of one kernel to CUDA source lines.

ncu's `--page source --print-source sass` CSV has per-SASS-instruction sample
counts but no line mapping for inlined code; nvdisasm -g on the cubin has the
line table.  Usage:

  ncu -i prof.ncu-rep --page source --csv --print-source sass > sass.csv
  cuobjdump -xelf all libcfgsim.so   (in a scratch dir)
  python tools/ncu_lines.py sass.csv tiers_lr_f64.sm_100a.cubin <mangled-substr> [top]
"""
import csv
import re
import subprocess
import sys
from collections import defaultdict


def line_table(cubin, fn_sub):
    out = subprocess.run(["nvdisasm", "-g", "-c", cubin], capture_output=True, text=True).stdout
    table, cur, inside = {}, None, False
    for ln in out.splitlines():
        if ln.startswith("//---------------------"):
            inside = fn_sub in ln
            continue
        if not inside:
            continue
        m = re.match(r'\s*//## File "([^"]+)", line (\d+)', ln)
        if m:
            cur = (m.group(1).split("/")[-1], int(m.group(2)))
            continue
        m = re.match(r"\s*/\*([0-9a-f]+)\*/\s+(.*)", ln)
        if m:
            table[int(m.group(1), 16)] = (cur, m.group(2).strip())
    return table


def main():
    path, cubin, fn_sub = sys.argv[1:4]
    top = int(sys.argv[4]) if len(sys.argv) > 4 else 40
    table = line_table(cubin, fn_sub)
    rows = list(csv.reader(open(path)))
    hdr = next(r for r in rows if r and r[0] == "Address")
    si = hdr.index("Warp Stall Sampling (All Samples)")
    start = rows.index(hdr) + 1
    base = None
    agg = defaultdict(int)
    tot = 0
    for r in rows[start:]:
        if not r or r[0] == "Kernel Name":
            break
        a = int(r[0], 16)
        base = a if base is None else base
        s = int(float(r[si] or 0))
        ent = table.get(a - base)
        key = ent[0] if ent else ("?", 0)
        agg[key] += s
        tot += s
    print(f"total samples {tot}")
    for k, v in sorted(agg.items(), key=lambda x: -x[1])[:top]:
        print(f"{100.0 * v / max(tot, 1):6.2f}%  {v:9d}  {k[0]}:{k[1]}")


if __name__ == "__main__":
    main()
