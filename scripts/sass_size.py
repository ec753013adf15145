"""SASS instruction count of one kernel attributed to engine.cu functions:
innermost engine.cu frame and outermost frame below the kernel body.
    python scripts/sass_size.py CUBIN KERNEL_MANGLED_NAME"""
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
full = subprocess.run(["nvdisasm", "--print-line-info-inline", sys.argv[1]], capture_output=True,
                      text=True).stdout
i0 = full.index(".text." + sys.argv[2] + ":")
i1 = full.find("\n\t.section", i0)
out = full[i0:i1 if i1 > 0 else len(full)]
src = open(os.path.join(ROOT, "paper_2602_11530_b200/csrc/engine.cu")).read().split("\n")
funcs = []
for n, line in enumerate(src, 1):
    m = re.match(r"(?:DEVI|__global__|template <[^>]*>|int|__device__ __noinline__)\s+"
                 r"[\w:<>\*& ]*?(\w+)\(", line)
    if m and not line.startswith(" "):
        funcs.append((n, m.group(1)))


def fn(ln):
    name = "?"
    for n, f in funcs:
        if n <= ln:
            name = f
    return name


inner, outer = {}, {}
chain_in, chain_out = "?", "?"
pending = []
for line in out.split("\n"):
    if "//## File" in line:
        pending += re.findall(r'"([^"]+)", line (\d+)', line)
        continue
    if re.match(r"\s+/\*[0-9a-f]{4,}\*/", line):
        if pending:
            eng = []
            for f, ln in pending:
                if f.endswith("engine.cu"):
                    name = fn(int(ln))
                    if name not in eng:
                        eng.append(name)
            if eng:
                chain_in = eng[0]
                top = [e for e in eng if e not in ("run_replica", "sched_kernel",
                                                    "__launch_bounds__")]
                chain_out = top[-1] if top else eng[-1]
            pending = []
        inner[chain_in] = inner.get(chain_in, 0) + 1
        outer[chain_out] = outer.get(chain_out, 0) + 1
tot = sum(inner.values())
print(f"total {tot} instructions = {tot * 16 / 1024:.1f} KB")
print("-- by outermost frame (handler / phase)")
for k, v in sorted(outer.items(), key=lambda x: -x[1])[:25]:
    print(f"{v:6d} {100 * v / tot:5.1f}% {k}")
print("-- by innermost engine.cu frame")
for k, v in sorted(inner.items(), key=lambda x: -x[1])[:25]:
    print(f"{v:6d} {100 * v / tot:5.1f}% {k}")
