"""Aggregate an ncu source page (stall samples / instructions) per engine.cu function.

    python scripts/ncu_funcs.py REP.ncu-rep
"""
import csv
import io
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv", "--print-source",
                      "cuda,sass"], capture_output=True, text=True, check=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[2]
i_s = hdr.index("Warp Stall Sampling (All Samples)")
i_i = hdr.index("Instructions Executed")
src = open(sys.argv[2] if len(sys.argv) > 2 else os.path.join(ROOT, "paper_2602_11530_b200/csrc/engine.cu")).read().split("\n")
funcs = []
for n, line in enumerate(src, 1):
    m = re.match(r"(?:DEVI|__global__|template <[^>]*>|int)\s+[\w:<>\*& ]*?(\w+)\(", line)
    if m and not line.startswith(" "):
        funcs.append((n, m.group(1)))


def fn(ln):
    name = "?"
    for n, f in funcs:
        if n <= ln:
            name = f
    return name


agg = {}
for r in rows[3:]:
    try:
        ln, s, ins = int(r[0]), int(r[i_s]), int(r[i_i])
    except (ValueError, IndexError):
        continue
    a = agg.setdefault(fn(ln), [0, 0])
    a[0] += s
    a[1] += ins
ts = sum(v[0] for v in agg.values()) or 1
ti = sum(v[1] for v in agg.values()) or 1
print(f"{'function':28s} {'samples':>8s} {'instr':>8s}")
for k, v in sorted(agg.items(), key=lambda x: -x[1][0]):
    print(f"{k:28s} {100 * v[0] / ts:7.1f}% {100 * v[1] / ti:7.1f}%")
