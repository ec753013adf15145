"""Offline goldens for the randomised parity draws — TEST INFRASTRUCTURE, runs
only in the build container (it needs oracle/_ref, the reference compiled
unmodified from /root/reference).

tests/test_fuzz_gpu.py draws 256 (trace, RunConfig, LatencyProfile) cases.
Some land in evict / swap-in thrash regimes where the reference runs for
minutes or hours; the GPU test cannot afford to run the reference live for
those. This script runs the REAL reference (oracle/_ref/ref_dump) on every
draw with no time budget, in parallel, and records the sha256 + line counts
of its hex-float records and pascal-events-v1 log (or its failure) in
tests/golden/fuzz_index.json. The GPU test compares against these.

Thrash draws write decision logs at ~30 MB/s for as long as they run (GBs),
so the procedure is two passes: every draw with its log under a short
timeout, then the draws that timed out again with no log and no time budget
("events": null — the GPU test then compares records only).

    python oracle/make_fuzz_golden.py --timeout 20          # pass 1
    python oracle/make_fuzz_golden.py --missing --no-events # pass 2
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import tempfile
import time
from concurrent.futures import ProcessPoolExecutor, as_completed

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "oracle"))
sys.path.insert(0, os.path.join(ROOT, "tests"))

from cases import cfg_text  # noqa: E402
from make_golden import REF_DUMP, build_trace_hex, sha_file  # noqa: E402

INDEX = os.path.join(ROOT, "tests", "golden", "fuzz_index.json")


def fuzz_cases():
    import test_fuzz_gpu as tf  # the draw list itself (seeded; no GPU needed)
    return tf.FUZZ


def one(c, timeout, events):
    with tempfile.TemporaryDirectory(dir="/tmp") as tmp:
        hexp = os.path.join(tmp, "t.hex")
        build_trace_hex(c["trace"], hexp, tmp)
        cfgp = os.path.join(tmp, "c.cfg")
        with open(cfgp, "w") as f:
            f.write(cfg_text(c))
        rec, ev = os.path.join(tmp, "r.rec"), os.path.join(tmp, "r.ev")
        t0 = time.time()
        try:
            r = subprocess.run([REF_DUMP, "run", hexp, cfgp, rec, ev if events else "-"],
                               capture_output=True,
                               text=True, timeout=timeout)
        except subprocess.TimeoutExpired:
            return c["name"], {"timeout_s": timeout}
        dt = time.time() - t0
        g = {"ref_s": round(dt, 3), "rc": r.returncode, "trace": sha_file(hexp)}
        if r.returncode == 0:
            g["records"] = sha_file(rec)
            g["events"] = sha_file(ev) if events else None
        else:
            g["stderr"] = r.stderr.strip()[-300:]
        return c["name"], g


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--jobs", type=int, default=6)
    ap.add_argument("--only", nargs="*", type=int)
    ap.add_argument("--timeout", type=float, default=None)
    ap.add_argument("--missing", action="store_true", help="only draws without a result")
    ap.add_argument("--no-events", action="store_true", help="records only (thrash draws)")
    args = ap.parse_args()
    cases = fuzz_cases()
    index = json.load(open(INDEX)) if os.path.exists(INDEX) else {}
    todo = [c for k, c in enumerate(cases) if not args.only or k in args.only]
    if args.missing:
        todo = [c for c in todo if "rc" not in index.get(c["name"], {})]
    with ProcessPoolExecutor(args.jobs) as ex:
        futs = [ex.submit(one, c, args.timeout, not args.no_events) for c in todo]
        for f in as_completed(futs):
            name, g = f.result()
            index[name] = g
            print(name, json.dumps(g)[:160], flush=True)
            with open(INDEX + ".tmp", "w") as fo:
                json.dump(index, fo, indent=1, sort_keys=True)
            os.replace(INDEX + ".tmp", INDEX)


if __name__ == "__main__":
    main()
