#!/usr/bin/env python
"""Instruction histogram of the built library's hot kernels from
`cuobjdump -sass` (evidence that the tensor-core path is tcgen05/TMEM: UTCHMMA
= tcgen05.mma, LDTM/STTM = tcgen05.ld/st, UBLKCP = cp.async.bulk, REDG =
global reductions).  Writes profiles/<tag>_sass_histogram.md.

usage: python tools/sass_histogram.py <tag> [lib.so]
"""
import collections
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KEYS = ["UTCHMMA", "UTCQMMA", "UTCBAR", "LDTM", "STTM", "UBLKCP", "UTMALDG", "HMMA", "REDG", "RED", "ATOMG",
        "LDG", "STG", "LDS", "STS", "DFMA", "DMUL", "DADD", "FFMA", "MUFU", "SHFL", "BAR", "SYNCS"]
KERNELS = ["mlp_bwd_kernel", "mlp_fwd_kernel", "hash_fwd_kernel", "composite_kernel", "raygen_kernel",
           "write_kernel", "adam_kernel", "accept_solve_kernel", "accept_memo_kernel", "occupancy_kernel",
           "import_plan_kernel", "import_scatter_kernel"]


def main():
    tag = sys.argv[1] if len(sys.argv) > 1 else "rXX"
    lib = sys.argv[2] if len(sys.argv) > 2 else os.path.join(ROOT, "paper_2507_01631_b200", "libtilefield_gpu.so")
    sass = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True, check=True).stdout
    funcs = {}
    cur = None
    for line in sass.splitlines():
        m = re.match(r"\s*Function : (\S+)", line)
        if m:
            cur = m.group(1)
            funcs[cur] = collections.Counter()
            continue
        m = re.match(r"\s*/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*)", line)
        if cur and m:
            funcs[cur][m.group(1)] += 1
    rows = []
    for k in KERNELS:
        for f, c in funcs.items():
            if k in f:
                # template arguments from the mangled name: ...kernelILb0ELi2EE... -> <0, 2>
                m = re.search(re.escape(k) + r"I((?:L[a-z]+-?\d+E)+)E", f)
                args = re.findall(r"L[a-z]+(-?\d+)E", m.group(1)) if m else []
                rows.append((k + (f"<{', '.join(args)}>" if args else ""), c))
    lines = [f"# SASS instruction histogram ({tag})", "",
             f"`cuobjdump -sass {os.path.relpath(lib, ROOT)}` (sm_100a), static instruction counts per kernel "
             "(prefix match: `RED` counts every RED* form, `LDG` every LDG*).", "",
             "| kernel | " + " | ".join(KEYS) + " |", "|---|" + "---|" * len(KEYS)]
    for name, c in rows:
        vals = [sum(n for op, n in c.items() if op == k or (op.startswith(k) and k in ("RED", "LDG", "STG", "LDS",
                                                                                      "STS", "BAR")))
                for k in KEYS]
        lines.append(f"| {name} | " + " | ".join(str(v) for v in vals) + " |")
    out = os.path.join(ROOT, "profiles", f"{tag}_sass_histogram.md")
    open(out, "w").write("\n".join(lines) + "\n")
    print(out)


if __name__ == "__main__":
    main()
