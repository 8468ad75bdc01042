#!/usr/bin/env python
"""Static evidence of the built library for profiles/: per-kernel ptxas
resources (registers, spills, stack, barriers) from the build logs and SASS
instruction-class counts (DMMA, LDGSTS, UBLKCP/SYNCS, ATOMS.CAS.128, BAR,
REDUX, SHFL ...) from cuobjdump of libcfgsim.so.

  python tools/sass_evidence.py ptxas > paper_1707_02423_b200/csrc/ptxas_summary.txt
  python tools/sass_evidence.py sass  > profiles/<round>_sass_summary.txt
  python tools/sass_evidence.py dump <mangled-substring> > profiles/<round>_sass_<name>.txt
"""
from __future__ import annotations

import collections
import re
import subprocess
import sys
import tempfile
from pathlib import Path

REPO = Path(__file__).resolve().parents[1]
CSRC = REPO / "paper_1707_02423_b200" / "csrc"
LIB = REPO / "paper_1707_02423_b200" / "libcfgsim.so"
CLASSES = ["DMMA", "HMMA", "UTCMMA", "UTCHMMA", "LDGSTS", "UBLKCP", "UTMALDG", "SYNCS", "ATOMS.CAS.128", "ATOMS",
           "BAR.SYNC", "BAR.ARV", "BAR.RED", "REDUX", "CREDUX", "SHFL", "LDS", "STS", "LDG", "STG", "DFMA", "DADD",
           "DMUL", "FFMA"]


def demangle(names):
    out = subprocess.run(["c++filt"], input="\n".join(names), capture_output=True, text=True).stdout.splitlines()
    return out if len(out) == len(names) else names


def ptxas():
    for log in sorted((CSRC / "build").glob("*.log")):
        txt = log.read_text().splitlines()
        fn = None
        for ln in txt:
            m = re.search(r"Compiling entry function '([^']+)'", ln)
            if m:
                fn = m.group(1)
                continue
            m = re.search(r"(\d+) bytes stack frame, (\d+) bytes spill stores, (\d+) bytes spill loads", ln)
            if m and fn:
                stack, sst, sld = m.groups()
                continue
            m = re.search(r"Used (\d+) registers(?:, used (\d+) barriers)?", ln)
            if m and fn:
                name = demangle([fn])[0]
                print(f"{log.stem:14s} regs {m.group(1):>3s} barriers {m.group(2) or '0':>2s} stack {stack:>4s} "
                      f"spill st/ld {sst}/{sld}  {name[:150]}")
                fn = None


def sass_all():
    with tempfile.TemporaryDirectory() as d:
        subprocess.run(["cuobjdump", "-xelf", "all", str(LIB)], cwd=d, capture_output=True)
        for cub in sorted(Path(d).glob("*.cubin")):
            txt = subprocess.run(["cuobjdump", "-sass", str(cub)], capture_output=True, text=True).stdout
            for fn, body in re.findall(r"Function : (\S+)\n(.*?)(?=\n\s+Function : |\Z)", txt, re.S):
                cnt = collections.Counter()
                for ins in re.findall(r"/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_.]+)", body):
                    for c in CLASSES:
                        if ins == c or ins.startswith(c + "."):
                            cnt[c] += 1
                            break
                tot = len(re.findall(r"/\*[0-9a-f]{4,}\*/\s+\S", body))
                if not any(k in fn for k in ("pair2", "big_kernel", "seq4", "seq_kernel", "lowrank", "start_", "flat",
                                             "ward", "scatter")):
                    continue
                name = demangle([fn])[0]
                print(f"{name[:140]}\n    {tot} instructions; " + ", ".join(f"{c} {cnt[c]}" for c in CLASSES if cnt[c]))


def dump(sub):
    with tempfile.TemporaryDirectory() as d:
        subprocess.run(["cuobjdump", "-xelf", "all", str(LIB)], cwd=d, capture_output=True)
        for cub in sorted(Path(d).glob("*.cubin")):
            txt = subprocess.run(["cuobjdump", "-sass", str(cub)], capture_output=True, text=True).stdout
            for fn, body in re.findall(r"Function : (\S+)\n(.*?)(?=\n\s+Function : |\Z)", txt, re.S):
                if sub in fn:
                    print("Function:", demangle([fn])[0])
                    for ln in body.splitlines():
                        m = re.match(r"\s+/\*([0-9a-f]{4,})\*/\s+(.*?);", ln)
                        if m:
                            print(m.group(1), m.group(2).strip())
                    return


if __name__ == "__main__":
    {"ptxas": ptxas, "sass": sass_all}.get(sys.argv[1], lambda: dump(sys.argv[2]))()
