"""Single-simulation latency of the drop-in path (pascal_run: capacity
derivation + policy run + report files) on the GPU vs the reference compiled
unmodified (oracle/_ref/ref_dump time: derive + run, one core) on the same
host, for the BASELINE configs C3 (rate sweep, stress point) and C4.

    python scripts/single_runs.py OUT.jsonl NAME[:cpu] ...

`:cpu` also times the reference here (skip it for the hour-long points; the
build container's golden timing is reported instead, tests/golden/index.json
ref_derive_s / ref_run_s)."""
import json
import os
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import paper_2602_11530_b200 as pb  # noqa: E402
from cases import BY_NAME, cfg_text  # noqa: E402
from harness import REF_DUMP, build_trace, golden, make_cfg, make_profile, sha_file  # noqa: E402

G = golden()
out = open(sys.argv[1], "a")
for arg in sys.argv[2:]:
    name, _, flag = arg.partition(":")
    c = BY_NAME[name]
    t = build_trace(c["trace"])
    g = G.get(name, {})
    rec = {"case": name, "requests": len(t), "instances": c["cfg"].get("instance_count"),
           "policy": c["cfg"].get("policy"), "request_iterations": t.request_iterations()}
    with tempfile.TemporaryDirectory() as tmp:
        prefix = os.path.join(tmp, "rep")
        t0 = time.perf_counter()
        pb.run(t, make_profile(c), make_cfg(c), prefix)
        rec["gpu_pascal_run_s"] = round(time.perf_counter() - t0, 3)
        tm = pb.last_timing()
        rec["gpu_derive_ms"] = round(tm.derive_ms, 1)
        rec["gpu_engine_ms"] = round(tm.engine_ms, 1)
        rec["instance_parallel"] = tm.instance_parallel
        if "report" in g:
            rec["report_matches_reference"] = all(
                sha_file(f"{prefix}.{ext}") == want for ext, want in g["report"].items())
        if flag == "cpu":
            hexp, cfgp = os.path.join(tmp, "t.hex"), os.path.join(tmp, "c.cfg")
            t.save_hex(hexp)
            with open(cfgp, "w") as f:
                f.write(cfg_text(c))
            r = subprocess.run([REF_DUMP, "time", hexp, cfgp, "1"], capture_output=True,
                               text=True, check=True)
            j = json.loads(r.stdout)
            rec["cpu_ref_s"] = round(j["derive_s"] + j["run_s"], 3)
            rec["cpu_ref_where"] = "this host, one core"
        elif "ref_run_s" in g and g.get("ref_run_s") is not None:
            rec["cpu_ref_s"] = round(g["ref_derive_s"] + g["ref_run_s"], 3)
            rec["cpu_ref_where"] = "build container (8-core Xeon), one core, oracle/make_golden.py"
    if "cpu_ref_s" in rec:
        rec["speedup"] = round(rec["cpu_ref_s"] / rec["gpu_pascal_run_s"], 2)
    print(json.dumps(rec), flush=True)
    out.write(json.dumps(rec) + "\n")
    out.flush()
