"""Golden-vector producer — TEST INFRASTRUCTURE, runs only in the build container
(it needs oracle/_ref, i.e. the reference compiled from /root/reference).

For every case in tests/cases.py it runs the REAL reference:
  * oracle/_ref/ref_dump gen/mix   -> the trace (lossless hex), sha256 pinned
  * oracle/_ref/ref_dump run       -> hex-float RequestRecords + pascal-events-v1
  * libpascal_ref.so pascal_run    -> the three pascal-report-v1 files
and stores sha256/line counts (plus full text for tiny cases) under
tests/golden/. The GPU tests recompute the same artefacts through
libpascal.so and compare.

    python oracle/make_golden.py [--only NAME ...] [--skip-large] [--jobs J]
                                 [--sizes xlarge huge ...] [--missing]

Sizes "xlarge" / "huge" / "thrash" (tests/cases.py) go through
`ref_dump all`: one capacity derivation + one simulation with that capacity
made explicit (identical results, see oracle/ref_dump.cpp) + the report files
with pascal_run's config echo, instead of the three simulations of the
run + capacity + C-ABI path. "huge" (C4 at 1M requests) pipes its records
straight into sha256sum (~26 GB of text is never stored).
"""
from __future__ import annotations

import argparse
import ctypes as C
import hashlib
import json
import os
import subprocess
import sys
import tempfile
import time
from concurrent.futures import ProcessPoolExecutor, as_completed

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

from cases import CASES, cfg_text  # noqa: E402
from paper_2602_11530_b200 import _lib  # noqa: E402

REF_DUMP = os.path.join(ROOT, "oracle", "_ref", "ref_dump")
REF_SO = os.path.join(ROOT, "oracle", "_ref", "libpascal_ref.so")
GOLD = os.path.join(ROOT, "tests", "golden")


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
    return h.hexdigest(), n


def build_trace_hex(recipe, out, tmp):
    """Materialise a recipe with the reference generator."""
    if "rows" in recipe:
        raw = out + ".py"
        with open(raw, "w") as f:
            f.write("pascal-trace-hex-v1\n")
            for (i, t, p, r, a, pre) in recipe["rows"]:
                f.write(f"{i} {float(t).hex()} {p} {r} {a} {int(pre)}\n")
        # mix with fraction 0 returns the base unchanged; re-emits it with C's %a
        subprocess.run([REF_DUMP, "mix", raw, raw, "0", "0", out], check=True)
        return
    if "gen" in recipe:
        n, rate, pd, rd, ad, seed, pre = recipe["gen"]
        subprocess.run([REF_DUMP, "gen", str(n), repr(float(rate)), pd, rd, ad, str(seed),
                        str(int(pre)), out], check=True)
        return
    base, repl, frac, seed = recipe["mix"]
    a = os.path.join(tmp, os.path.basename(out) + ".a")
    b = os.path.join(tmp, os.path.basename(out) + ".b")
    build_trace_hex(base, a, tmp)
    build_trace_hex(repl, b, tmp)
    subprocess.run([REF_DUMP, "mix", a, b, repr(float(frac)), str(seed), out], check=True)


def ref_trace_handle(lib, recipe, tmp):
    """Same recipe through the reference C ABI (for pascal_run report goldens)."""
    out = C.c_void_p()
    if "rows" in recipe:
        path = os.path.join(tmp, "rows.trace")
        with open(path, "w") as f:
            f.write("pascal-trace-v1\n")
            for (i, t, p, r, a, pre) in recipe["rows"]:
                f.write(f"{i},{t:.9f},{p},{r},{a},{int(pre)}\n")
        assert lib.pascal_trace_load(path.encode(), C.byref(out)) == 0
        return out
    if "gen" in recipe:
        n, rate, pd, rd, ad, seed, pre = recipe["gen"]
        st = lib.pascal_trace_generate(n, rate, pd.encode(), rd.encode(), ad.encode(), seed,
                                       int(pre), C.byref(out))
        assert st == 0, lib.pascal_last_error()
        return out
    base, repl, frac, seed = recipe["mix"]
    a = ref_trace_handle(lib, base, tmp)
    b = ref_trace_handle(lib, repl, tmp)
    assert lib.pascal_trace_mix(a, b, frac, seed, C.byref(out)) == 0
    lib.pascal_trace_free(a)
    lib.pascal_trace_free(b)
    return out


def ref_config(lib, c):
    cfg = _lib.RunConfig()
    lib.pascal_run_config_init(C.byref(cfg))
    for k, v in c["cfg"].items():
        setattr(cfg, k, v.encode() if k == "policy" else v)
    prof = C.c_void_p()
    assert lib.pascal_profile_default(C.byref(prof)) == 0
    for k, v in c["profile"].items():
        assert lib.pascal_profile_set(prof, k.encode(), float(v)) == 0
    return cfg, prof


BIG = ("xlarge", "huge", "thrash")


def golden_big(c, timeout):
    """One `ref_dump all` run (records sha, reports; no decision log)."""
    name = c["name"]
    with tempfile.TemporaryDirectory(dir="/tmp") as tmp:
        trace = os.path.join(tmp, name + ".hex")
        build_trace_hex(c["trace"], trace, tmp)
        cfgp = os.path.join(tmp, name + ".cfg")
        with open(cfgp, "w") as f:
            f.write(cfg_text(c))
        prefix = os.path.join(tmp, name + ".rep")
        rec = os.path.join(tmp, name + ".rec")
        rec_spec = f"|sha256sum > {rec}.sha" if c["size"] == "huge" else rec
        t0 = time.time()
        try:
            r = subprocess.run([REF_DUMP, "all", trace, cfgp, rec_spec, "-", prefix],
                               check=True, capture_output=True, text=True, timeout=timeout)
        except subprocess.TimeoutExpired:
            return name, {"timeout_s": timeout}
        info = json.loads(r.stdout)
        if c["size"] == "huge":
            records = [open(rec + ".sha").read().split()[0], c_requests(trace)]
        else:
            records = list(sha_file(rec))
        g = {"trace": list(sha_file(trace)), "records": records, "events": None,
             "capacity": info["capacity"], "ref_derive_s": info["derive_s"],
             "ref_run_s": info["run_s"], "ref_wall_s": round(time.time() - t0, 1),
             "report": {ext: list(sha_file(prefix + "." + ext))
                        for ext in ("requests.csv", "summary.txt", "bins.csv")}}
        with open(prefix + ".summary.txt") as f:
            g["summary_text"] = f.read()
        return name, g


def c_requests(trace_hex):
    with open(trace_hex) as f:
        return sum(1 for _ in f) - 1


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--only", nargs="*")
    ap.add_argument("--skip-large", action="store_true")
    ap.add_argument("--sizes", nargs="*", help="only cases of these sizes")
    ap.add_argument("--missing", action="store_true", help="only cases not in the index")
    ap.add_argument("--jobs", type=int, default=1, help="parallel workers (xlarge/huge/thrash)")
    ap.add_argument("--timeout", type=float, default=300.0)
    args = ap.parse_args()
    os.makedirs(GOLD, exist_ok=True)
    lib = _lib.bind(C.CDLL(REF_SO), extensions=False)
    index_path = os.path.join(GOLD, "index.json")
    index = json.load(open(index_path)) if os.path.exists(index_path) else {}

    mine = {}

    def save():
        # several generator processes may run at once: merge under a lock
        import fcntl
        with open(index_path + ".lock", "w") as lk:
            fcntl.flock(lk, fcntl.LOCK_EX)
            cur = json.load(open(index_path)) if os.path.exists(index_path) else {}
            cur.update(mine)
            with open(index_path + ".tmp", "w") as f:
                json.dump(cur, f, indent=1, sort_keys=True)
            os.replace(index_path + ".tmp", index_path)

    def wanted(c):
        if args.only and c["name"] not in args.only:
            return False
        if args.skip_large and c["size"] == "large":
            return False
        if args.sizes and c["size"] not in args.sizes:
            return False
        if args.missing and c["name"] in index and "timeout_s" not in index[c["name"]]:
            return False
        return True

    big = [c for c in CASES if wanted(c) and c["size"] in BIG]
    if big:
        with ProcessPoolExecutor(max(1, args.jobs)) as ex:
            futs = [ex.submit(golden_big, c, None if c["size"] == "huge" else args.timeout)
                    for c in big]
            for fu in as_completed(futs):
                name, g = fu.result()
                index[name] = mine[name] = g
                print(f"{name:28s} {json.dumps({k: g.get(k) for k in ('capacity', 'ref_run_s', 'timeout_s')})}",
                      flush=True)
                save()
    with tempfile.TemporaryDirectory() as tmp:
        for c in CASES:
            name = c["name"]
            if not wanted(c) or c["size"] in BIG:
                continue
            trace = os.path.join(tmp, name + ".hex")
            build_trace_hex(c["trace"], trace, tmp)
            cfgp = os.path.join(tmp, name + ".cfg")
            with open(cfgp, "w") as f:
                f.write(cfg_text(c))
            rec = os.path.join(tmp, name + ".rec")
            xl = c["size"] == "xlarge"  # records + reports only, no decision log
            ev = "-" if xl else os.path.join(tmp, name + ".ev")
            subprocess.run([REF_DUMP, "run", trace, cfgp, rec, ev], check=True, timeout=args.timeout)
            cap = subprocess.run([REF_DUMP, "capacity", trace, cfgp], check=True,
                                 capture_output=True, text=True).stdout.strip()
            g = {"trace": sha_file(trace), "records": sha_file(rec),
                 "events": None if xl else sha_file(ev), "capacity": int(cap)}
            # report files through the reference's own C ABI
            th = ref_trace_handle(lib, c["trace"], tmp)
            cfg, prof = ref_config(lib, c)
            prefix = os.path.join(tmp, name + ".rep")
            evlog = os.path.join(tmp, name + ".capi.ev")
            st = lib.pascal_run(th, prof, C.byref(cfg), prefix.encode(),
                                None if xl else evlog.encode())
            assert st == 0, (name, lib.pascal_last_error())
            g["report"] = {ext: sha_file(prefix + "." + ext)
                           for ext in ("requests.csv", "summary.txt", "bins.csv")}
            if not xl:
                assert sha_file(evlog) == g["events"], name  # C-ABI log == engine log
            lib.pascal_trace_free(th)
            lib.pascal_profile_free(prof)
            if c["size"] == "tiny":
                for src, ext in ((rec, "records"), (ev, "events")):
                    with open(src) as f, open(os.path.join(GOLD, f"{name}.{ext}"), "w") as o:
                        o.write(f.read())
                with open(prefix + ".summary.txt") as f, \
                        open(os.path.join(GOLD, f"{name}.summary.txt"), "w") as o:
                    o.write(f.read())
            index[name] = mine[name] = g
            print(f"{name:28s} records={g['records'][1]:6d} "
                  f"events={g['events'][1] if g['events'] else '-':>9} "
                  f"cap={g['capacity']}", flush=True)
            save()


if __name__ == "__main__":
    main()
