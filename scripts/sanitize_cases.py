"""Small parity cases driven through every engine build for compute-sanitizer:
    compute-sanitizer --tool memcheck|racecheck|synccheck python scripts/sanitize_cases.py
(logging build via run_dump, lean single-policy builds + metrics via Batch,
shared-memory heap spills via PB_SMEM_HEAP, HBM-resident request state via
PB_SMEM=0 in a second pass)."""
import os
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import paper_2602_11530_b200 as pb  # noqa: E402
from cases import BY_NAME  # noqa: E402
from harness import build_trace, make_cfg, make_profile  # noqa: E402

NAMES = ["trio_rr", "trio_pascal", "r0a1_pascal", "c1_pascal", "c1_fcfs", "abl60_nonadaptive",
         "demote_pascal", "preload_rr", "tinyq_pascal", "infswap_pascal"]
with tempfile.TemporaryDirectory() as tmp:
    for name in NAMES:
        c = BY_NAME[name]
        t = build_trace(c["trace"])
        pb.run_dump(t, make_profile(c), make_cfg(c), os.path.join(tmp, "r"), os.path.join(tmp, "e"))
        b = pb.Batch([t, t], [make_profile(c)] * 2, [make_cfg(c)] * 2)
        b.set_groups([0, 1], 2)
        b.execute()
        s = b.summaries()
        b.histograms()
        assert all(x.status == 0 for x in s), name
        print(name, "ok", flush=True)
    # a mixed-policy batch (generic nolog build)
    cs = [BY_NAME[n] for n in ("c1_pascal", "c1_fcfs", "c1_rr", "c1_oracle")]
    ts = [build_trace(c["trace"]) for c in cs]
    s = pb.run_batch(ts, [make_profile(c) for c in cs], [make_cfg(c) for c in cs])
    assert all(x.status == 0 for x in s)
    print("mixed batch ok")
