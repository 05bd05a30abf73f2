"""SASS opcode census of the in-tree library, per kernel (no GPU needed):
cuobjdump -sass paper_1908_09376_b200/libmidbf_b200.so, count the opcodes
that evidence each kernel's design (DMMA = FP64 tensor core, DFMA/DMUL/DADD =
FP64 pipe, UBLKCP = TMA bulk copy, SYNCS = mbarrier ops, LDG/STG/LDS/STS,
strong polls LDG.E.*STRONG.GPU, ST*.STRONG.GPU stores).  Writes a markdown
table to stdout.  Usage: python tools/sass_census.py > profiles/r2_sass_census.md"""
import collections
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SO = os.path.join(ROOT, "paper_1908_09376_b200", "libmidbf_b200.so")
KEYS = ["DMMA", "DFMA", "DMUL", "DADD", "MUFU", "UBLKCP", "SYNCS", "LDG", "LDG.STRONG.GPU", "STG", "STG.STRONG.GPU",
        "LDS", "STS", "BAR", "RED", "ATOM", "FENCE"]


def demangle(names):
    out = subprocess.run(["c++filt"], input="\n".join(names), capture_output=True, text=True).stdout.splitlines()
    return dict(zip(names, out))


def main():
    txt = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-sass", SO], capture_output=True, text=True).stdout
    funcs = collections.OrderedDict()
    cur = None
    for line in txt.splitlines():
        m = re.match(r"\s*Function : (\S+)", line)
        if m:
            cur = m.group(1)
            funcs[cur] = collections.Counter()
            continue
        if cur is None:
            continue
        m = re.match(r"\s*/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_.]*)", line)
        if not m:
            continue
        op = m.group(1)
        base = op.split(".")[0]
        c = funcs[cur]
        c["_total"] += 1
        if base in KEYS:
            c[base] += 1
        if base == "LDG" and "STRONG.GPU" in op:
            c["LDG.STRONG.GPU"] += 1
        if base in ("STG", "ST") and "STRONG.GPU" in op:
            c["STG.STRONG.GPU"] += 1
        if base in ("MEMBAR", "FENCE", "CCTL"):
            c["FENCE"] += 1
    dm = demangle(list(funcs))
    print("# SASS opcode census — `paper_1908_09376_b200/libmidbf_b200.so` (sm_100a)\n")
    print("Produced by `python tools/sass_census.py` from `cuobjdump -sass` (static instruction counts per "
          "kernel instantiation, not executed counts).  UBLKCP = `cp.async.bulk` (TMA bulk engine); SYNCS = "
          "mbarrier ops; DMMA = `mma.sync.m8n8k4.f64` (FP64 tensor core); `*.STRONG.GPU` = the relaxed.gpu "
          "polls / stores of the data-as-signal protocol; FENCE counts MEMBAR / FENCE / CCTL.\n")
    print("| kernel | instrs | " + " | ".join(KEYS) + " |")
    print("|---|---|" + "---|" * len(KEYS))
    for f, c in funcs.items():
        name = dm.get(f, f)
        name = re.sub(r"midbf::dev::|\(anonymous namespace\)::|midbf::|dev::", "", name)
        name = re.sub(r"\(.*", "", name) if len(name) > 90 else name
        print(f"| `{name[:90]}` | {c['_total']} | " + " | ".join(str(c[k]) for k in KEYS) + " |")


if __name__ == "__main__":
    main()
