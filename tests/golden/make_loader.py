"""Golden vectors for the native corpus loader from the
reference itself.  Run in the build container:

    python tests/golden/make_loader.py

Writes tests/golden/loader.json.gz: seeded synthetic listings (labels,
unlabelled blocks after control instructions, predicated BRA/EXIT, BRX, JMP,
CAL, unreachable code, comments, odd spacing) with profiles of every kind
(none, samples incl. orphans, observed edge records by label / B<i> / index /
START / STOP / unknown endpoints, time/calls/dynmix records), each run
through the reference's parse_listing → build_cfg → parse_profiles →
attribute_profile → transition_matrix in all three modes; plus malformed
listings and profiles with the reference's exception class, line number and
message.  Matrices are stored sparsely with float.hex values (exact).
"""

from __future__ import annotations

import gzip
import json
import random
import sys
from pathlib import Path

HERE = Path(__file__).resolve().parent
sys.path.insert(0, "/root/reference/pkg/src")

from sasscfg.cfg import build_cfg  # noqa: E402
from sasscfg.matrix import GLOBAL, RAW_COUNTS, ROW_STOCHASTIC, transition_matrix  # noqa: E402
from sasscfg.profile import attribute_profile, parse_profiles  # noqa: E402
from sasscfg.sass import parse_listing  # noqa: E402

MODES = (ROW_STOCHASTIC, GLOBAL, RAW_COUNTS)
OPS = ["FADD R0, R1, R2", "FFMA.FTZ R3, R3, R4, R5", "DFMA R6, R6, R7, R8", "IADD3 R0, R0, 0x1, RZ",
       "IMAD.WIDE R2, R2, R3, R4", "LDG.E.64 R4, [R2.64+0x10]", "STS [R3], R4", "MOV R5, R6",
       "S2R R0, SR_TID.X", "F2I.S32.F32 R2, R3", "VADD.U32 R1, R1, R2", "SHF.R.U32 R4, R4, 0x1, RZ",
       "ISETP.GE.AND P0, PT, R1, R2, PT", "DSETP.LE.AND P0, PT, |R6|, +INF, PT", "PSETP.AND P1, PT, P0, PT",
       "SEL R1, R2, R3, P0", "MUFU.RCP R4, R5", "NOP", "HMMA.16816.F32 R8, R4, R6, R8", "POPC R1, R2",
       "ATOMG.E.ADD.STRONG.GPU PT, R4, [R2], R5", "BAR.SYNC 0x0", "CAL `(.L_x)", "ssy `(.L_1)"]


def make_listing(rng: random.Random, nb: int) -> tuple[str, list[int]]:
    """Random listing with nb label slots; returns the text and the offsets of
    every instruction (for sample records)."""
    lines, offs = [], []
    off = rng.choice([0, 0x8, 0x10, 0x100])
    labelled = [rng.random() < 0.7 or b == 0 for b in range(nb)]
    labelled[0] = rng.random() < 0.8
    names = [f".L_{b}" for b in range(nb)]
    targets = [b for b in range(nb) if labelled[b]]
    for b in range(nb):
        if rng.random() < 0.1:
            lines.append(rng.choice(["", "   ", "// comment", "# note", "\t"]))
        if labelled[b]:
            lines.append(f"{names[b]}:" if rng.random() < 0.9 else f"  {names[b]}:  ")
        for _ in range(rng.randint(1, 4)):
            op = rng.choice(OPS)
            if "`(.L_x)" in op or "`(.L_1)" in op:
                op = op.split("`")[0] + (f"`({rng.choice(names[:1] + [names[t] for t in targets])})" if targets else "0x0")
            pred = f"@{rng.choice(['', '!'])}P{rng.randrange(7)} " if rng.random() < 0.15 else ""
            sp = rng.choice([" ", "  ", "\t"])
            lines.append(f"{sp}/*{off:04x}*/{rng.choice([' ', '  ', ''])}{pred}{op} ;")
            offs.append(off)
            off += rng.choice([8, 16])
        kind = rng.choice(["bra", "cbra", "pexit", "exit", "fall", "fall", "brx", "jmp", "ret", "cal"])
        if b == nb - 1 and rng.random() < 0.7:
            kind = "exit"
        tgt = names[rng.choice(targets)] if targets else None
        pred = f"@{rng.choice(['', '!'])}P{rng.randrange(7)} "
        if kind in ("bra", "cbra", "jmp") and tgt is None:
            kind = "fall"
        text = {"bra": f"BRA `({tgt})", "cbra": f"{pred}BRA `({tgt})", "pexit": f"{pred}EXIT",
                "exit": "EXIT", "brx": f"{pred if rng.random() < 0.5 else ''}BRX R4 -0x20",
                "jmp": f"{pred if rng.random() < 0.5 else ''}JMP `({tgt})", "ret": "RET.REL.NODEC R20 0x0",
                "cal": f"CALL.REL.NOINC `({tgt})" if tgt else "CALL.ABS.NOINC 0x0", "fall": None}[kind]
        if kind == "bra" and rng.random() < 0.1:
            text = "BRA 0x120"  # branch without a label target
        if text is not None:
            lines.append(f"        /*{off:04x}*/ {text} ;")
            offs.append(off)
            off += 8
    return "\n".join(lines) + rng.choice(["\n", "", "\n\n"]), offs


def make_profile(rng: random.Random, kid: str, nb: int, offs: list[int]) -> str | None:
    kind = rng.choice(["none", "samples", "samples", "edges", "edges", "empty", "other"])
    if kind == "none":
        return None
    out = ["# profile", f"kernel {kid}"]
    if kind == "empty":
        pass
    elif kind == "samples":
        for o in rng.sample(offs, k=min(len(offs), rng.randint(1, len(offs)))):
            out.append(f"sample {o + rng.choice([0, 0, 0, 4]):x} {rng.randrange(0, 300)}")
        if rng.random() < 0.3:
            out.append(f"sample {max(offs) + 0x100:x} 7")  # orphan
        if rng.random() < 0.2:
            out.append(f"sample 0x{offs[0]:X} 3")
    elif kind == "edges":
        toks = ["START", "STOP"] + [f".L_{b}" for b in range(nb)] + [f"B{b}" for b in range(nb + 2)] + \
               [str(b) for b in range(nb + 1)] + [".L_missing", "B", "x1"]
        for _ in range(rng.randint(1, 3 * nb)):
            out.append(f"edge {rng.choice(toks)} {rng.choice(toks)} {rng.randrange(0, 1000)}")
    if rng.random() < 0.3:
        out.append(f"time_ns {rng.randrange(1, 10**6)}")
    if rng.random() < 0.3:
        out.append(f"calls {rng.randrange(1, 50)}")
    if rng.random() < 0.2:
        out.append("dynmix FP32=10 INT=4 MEM=2")
    if kind == "other" or rng.random() < 0.2:  # another kernel's section
        out += [f"kernel other.{rng.randrange(99)}", "sample 8 1"]
    rng.shuffle(out[2:]) if rng.random() < 0.3 else None
    return "\n".join(out) + "\n"


def run(kid: str, listing: str, profile: str | None, mode: str) -> dict:
    try:
        cfg = build_cfg(parse_listing(listing, kid))
        prof = None
        if profile is not None:
            profs = parse_profiles(profile)
            prof = profs.get(kid)
            if prof is None:
                return {"error": "CorpusError", "line": 0, "msg": f"profile has no profile for kernel {kid!r}"}
        tm = transition_matrix(attribute_profile(cfg, prof), mode=mode)
    except Exception as exc:  # noqa: BLE001 — the class and message are the fixture
        return {"error": type(exc).__name__, "line": getattr(exc, "line_no", 0),
                "msg": getattr(exc, "reason", None) or str(exc)}
    e = tm.entries
    nz = [[int(i), int(j), float(e[i, j]).hex()] for i, j in zip(*e.nonzero())]
    return {"n": int(e.shape[0]), "ordering": list(tm.ordering), "nz": nz}


BAD_LISTINGS = [
    "/*0008*/ FADD R0, R1, R2\n",                       # unterminated
    "/*00g8*/ FADD R0, R1, R2 ;\n",                     # malformed offset
    "/**/ NOP ;\n",                                     # malformed offset
    "FADD R0, R1, R2 ;\n",                              # unrecognized
    ".L_1-x:\n/*0008*/ NOP ;\n",                        # unrecognized (bad label)
    "/*0008*/ ;\n",                                     # missing opcode
    "/*0008*/ @P0 ;\n",                                 # missing opcode (predicate only)
    "/*0008*/ @P0;\n",                                  # malformed opcode token
    "/*0008*/ 9FADD R0 ;\n",                            # malformed opcode token
    "/*0008*/ FADD..F32 R0 ;\n",                        # malformed opcode token
    "/*0008*/ FADD\tR0, R1 ;\n",                        # tab is not the operand separator
    "/*0010*/ NOP ;\n/*0008*/ NOP ;\n",                 # non-increasing offsets
    "/*0010*/ NOP ;\n/*0010*/ NOP ;\n",
    ".L_1:\n/*0008*/ NOP ;\n.L_1:\n/*0010*/ NOP ;\n",  # duplicate label
    ".L_1:\n.L_2:\n/*0008*/ NOP ;\n",                  # label after label
    "/*0008*/ NOP ;\n.L_9:\n",                          # dangling label
    "/*0008*/ BRA `(.L_7) ;\n/*0010*/ EXIT ;\n",        # unresolved
    "/*0008*/ @!P3 BRA `(.L_7) ;\n.L_8:\n/*0010*/ BRA `(.L_6) ;\n",
    "",                                                 # empty graph
    "// only a comment\n\n# and another\n",
    "/*0008*/ FADD 'q' ;\n",                            # repr quoting in messages
    "FADD \"x\" 'y';\n",
    "/*0008*/ EXIT ;\r\n/*0010*/ NOP ;\r\n\r\n/*0004*/ NOP ;\r\n",
]

GOOD_LISTING = ".L_0:\n/*0008*/ @P0 BRA `(.L_2) ;\n/*0010*/ NOP ;\n.L_2:\n/*0018*/ EXIT ;\n"
BAD_PROFILES = [
    "sample 8 1\n",                                     # before any kernel header
    "kernel\n",
    "kernel a b\n",
    "kernel k\nsample 8\n",
    "kernel k\nsample zz 1\n",
    "kernel k\nsample 8 x\n",
    "kernel k\nsample 0x8 1_0\nedge .L_0 .L_2 4\nedge .L_0 .L_2 x\n",
    "kernel k\nedge a b\n",
    "kernel k\ntime_ns\n",
    "kernel k\ntime_ns 0\n",
    "kernel k\ncalls 0\n",
    "kernel k\ncalls x\n",
    "kernel k\ndynmix FP32=1\ndynmix INT=2\n",
    "kernel k\ndynmix FOO=1\n",
    "kernel k\ndynmix FOO=x\n",
    "kernel k\ndynmix FP32=-1\n",
    "kernel k\ndynmix FP32\n",
    "kernel k\nbogus 1 2\n",
    "kernel k\nsample 8 -5\n",
    "kernel k\nsample 8 -5\nsample 8 9\n",              # accumulates to 4: fine
    "kernel k\nedge .L_0 .L_2 -1\n",
    "kernel k\nkernel k\n",
    "kernel j\nsample 8 1\nkernel j\n",
    "kernel j\nsample 8 1\n",                           # no section for k
    "kernel k\nsample -0x8 1\nsample +10 2\nsample 0X_1_0 3\n",
    "kernel k\nedge B0 B2 5\nedge 0 2 6\nedge .L_0 STOP 3\nedge START B0 1\n",
]


def main():
    rng = random.Random(20261017)
    cases = []
    for t in range(260):
        nb = rng.choice([1, 1, 2, 3, 4, 6, 8, 12, 20, 40]) if t < 240 else rng.choice([150, 400, 900])
        kid = f"k{t}.synth.f.m"
        listing, offs = make_listing(rng, nb)
        profile = make_profile(rng, kid, nb, offs)
        mode = MODES[t % 3]
        cases.append({"kernel_id": kid, "listing": listing, "profile": profile, "mode": mode,
                      "expect": run(kid, listing, profile, mode)})
    for i, bad in enumerate(BAD_LISTINGS):
        cases.append({"kernel_id": "bad.k", "listing": bad, "profile": None, "mode": ROW_STOCHASTIC,
                      "expect": run("bad.k", bad, None, ROW_STOCHASTIC)})
    for i, bad in enumerate(BAD_PROFILES):
        for mode in MODES:
            cases.append({"kernel_id": "k", "listing": GOOD_LISTING, "profile": bad, "mode": mode,
                          "expect": run("k", GOOD_LISTING, bad, mode)})
    ok = sum("n" in c["expect"] for c in cases)
    with gzip.open(HERE / "loader.json.gz", "wt") as f:
        json.dump(cases, f)
    kinds = {}
    for c in cases:
        k = c["expect"].get("error", "ok")
        kinds[k] = kinds.get(k, 0) + 1
    print(f"{len(cases)} cases ({ok} matrices): {kinds}")


if __name__ == "__main__":
    main()
