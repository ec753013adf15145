"""Instance-parallel engine: records of every multi-instance parity case vs
the golden sha, whether the engine kept or declined each, and single-replica
timings against the serial engine (PB_PDES=0 in a second process)."""
import json
import os
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import paper_2602_11530_b200 as pb  # noqa: E402
from cases import CASES  # noqa: E402
from harness import build_trace, golden, make_cfg, make_profile, sha_file  # noqa: E402

G = golden()
mode = sys.argv[1] if len(sys.argv) > 1 else "parity"
if mode == "parity":
    ok = bad = dec = 0
    with tempfile.TemporaryDirectory() as tmp:
        for c in CASES:
            if c["name"] not in G or c["size"] not in ("tiny", "small", "medium"):
                continue
            if c["cfg"].get("instance_count", 8) < 2:
                continue
            t = build_trace(c["trace"])
            rec = os.path.join(tmp, "r")
            pb.run_dump(t, make_profile(c), make_cfg(c), rec, None)
            used = pb.last_timing().instance_parallel
            same = sha_file(rec) == G[c["name"]]["records"]
            ok += same
            bad += not same
            dec += used == 0
            print(f"{c['name']:28s} {'OK ' if same else 'BAD'} instance_parallel={used}", flush=True)
    print(f"parity: {ok} ok, {bad} bad, {dec} declined")
else:
    for name in sys.argv[2:]:
        c = next(x for x in CASES if x["name"] == name)
        t = build_trace(c["trace"])
        b = pb.Batch([t], [make_profile(c)], [make_cfg(c)])
        t0 = time.perf_counter()
        b.execute()
        wall = time.perf_counter() - t0
        s = b.summaries()[0]
        tm = pb.last_timing()
        ok = None
        g = G.get(name)
        print(json.dumps({"case": name, "pdes": os.environ.get("PB_PDES", "1"), "status": s.status,
                          "instance_parallel": tm.instance_parallel, "derive_ms": tm.derive_ms,
                          "engine_ms": tm.engine_ms, "total_ms": tm.total_ms, "wall_s": wall,
                          "capacity": s.capacity,
                          "capacity_ok": (g or {}).get("capacity") in (None, s.capacity),
                          "ttft_p99": s.ttft_p99}), flush=True)
