"""Test helpers: materialise tests/cases.py recipes through libpascal.so, and run
the C oracle restatement (oracle/_build/oracle_dump) on the same inputs.
The oracle is the checker only (see oracle/pascal_oracle.h)."""
from __future__ import annotations

import hashlib
import json
import os
import subprocess

import paper_2602_11530_b200 as pb
from cases import cfg_text

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLD = os.path.join(ROOT, "tests", "golden")
ORACLE_DUMP = os.path.join(ROOT, "oracle", "_build", "oracle_dump")
REF_DUMP = os.path.join(ROOT, "oracle", "_ref", "ref_dump")


def build_trace(recipe) -> pb.Trace:
    if "rows" in recipe:
        r = recipe["rows"]
        return pb.Trace.from_arrays([x[0] for x in r], [float(x[1]) for x in r],
                                    [x[2] for x in r], [x[3] for x in r], [x[4] for x in r],
                                    [int(x[5]) for x in r])
    if "gen" in recipe:
        n, rate, pd, rd, ad, seed, pre = recipe["gen"]
        return pb.Trace.generate(n, rate, pd, rd, ad, seed, pre)
    base, repl, frac, seed = recipe["mix"]
    return pb.Trace.mix(build_trace(base), build_trace(repl), frac, seed)


def make_cfg(c):
    return pb.run_config(**c["cfg"])


def make_profile(c):
    return pb.Profile.default(**c["profile"])


def sha_file(path):
    h = hashlib.sha256()
    n = 0
    with open(path, "rb") as f:
        while True:
            b = f.read(1 << 20)
            if not b:
                break
            h.update(b)
            n += b.count(b"\n")
    return [h.hexdigest(), n]


def golden():
    with open(os.path.join(GOLD, "index.json")) as f:
        return json.load(f)


def oracle_run(c, trace: pb.Trace, tmp):
    """Records + event log of the C restatement for case `c` on `trace`."""
    name = c["name"]
    hexp = os.path.join(tmp, name + ".oracle.hex")
    trace.save_hex(hexp)
    cfgp = os.path.join(tmp, name + ".oracle.cfg")
    with open(cfgp, "w") as f:
        f.write(cfg_text(c))
    rec = os.path.join(tmp, name + ".oracle.rec")
    ev = os.path.join(tmp, name + ".oracle.ev")
    subprocess.run([ORACLE_DUMP, "run", hexp, cfgp, rec, ev], check=True, timeout=600)
    return rec, ev


def first_diff(a, b, limit=3):
    """First differing lines of two text files (for failure messages)."""
    out = []
    with open(a, "rb") as fa, open(b, "rb") as fb:
        for i, (x, y) in enumerate(zip(fa, fb)):
            if x != y:
                out.append(f"line {i + 1}:\n  got  {x[:300]!r}\n  want {y[:300]!r}")
                if len(out) >= limit:
                    break
    return "\n".join(out) or "(one file is a prefix of the other)"
