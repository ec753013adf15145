"""Golden-vector producer — TEST INFRASTRUCTURE, runs only in the build container
(it needs oracle/_ref, i.e. the reference compiled from /root/reference).

For every case in tests/cases.py it runs the REAL reference:
  * oracle/_ref/ref_dump gen/mix   -> the trace (lossless hex), sha256 pinned
  * oracle/_ref/ref_dump run       -> hex-float RequestRecords + pascal-events-v1
  * libpascal_ref.so pascal_run    -> the three pascal-report-v1 files
and stores sha256/line counts (plus full text for tiny cases) under
tests/golden/. The GPU tests recompute the same artefacts through
libpascal.so and compare.

    python oracle/make_golden.py [--only NAME ...] [--skip-large]
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


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--only", nargs="*")
    ap.add_argument("--skip-large", action="store_true")
    ap.add_argument("--timeout", type=float, default=300.0)
    args = ap.parse_args()
    os.makedirs(GOLD, exist_ok=True)
    lib = _lib.bind(C.CDLL(REF_SO), extensions=False)
    index_path = os.path.join(GOLD, "index.json")
    index = json.load(open(index_path)) if os.path.exists(index_path) else {}
    with tempfile.TemporaryDirectory() as tmp:
        for c in CASES:
            name = c["name"]
            if args.only and name not in args.only:
                continue
            if args.skip_large and c["size"] == "large":
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
            index[name] = g
            print(f"{name:28s} records={g['records'][1]:6d} "
                  f"events={g['events'][1] if g['events'] else '-':>9} "
                  f"cap={g['capacity']}", flush=True)
            with open(index_path, "w") as f:
                json.dump(index, f, indent=1, sort_keys=True)


if __name__ == "__main__":
    main()
