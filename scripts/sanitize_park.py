"""The lean Pascal build's parked-tail path under compute-sanitizer: Pascal
cases that park (C5 acceptance replicas, C2) as lean-engine batches
(PB_PDES=0), request state in shared memory and in HBM.
    compute-sanitizer --tool memcheck|racecheck|synccheck python scripts/sanitize_park.py"""
import os
import sys

os.environ["PB_PDES"] = "0"
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import paper_2602_11530_b200 as pb  # noqa: E402
from cases import BY_NAME  # noqa: E402
from harness import build_trace, make_cfg, make_profile  # noqa: E402

for smem in ("1", "0"):
    os.environ["PB_SMEM"] = smem
    names = ["c5_s7_k6_pascal", "c5_s7_k6_nonadaptive", "tinyq_pascal"]
    if not os.environ.get("PARK_SAN_LIGHT"):  # C2 only under memcheck (racecheck: hours)
        names.append("c2_pascal")
    for name in names:
        c = BY_NAME[name]
        t = build_trace(c["trace"])
        b = pb.Batch([t, t], [make_profile(c)] * 2, [make_cfg(c)] * 2)
        b.execute()
        s = b.summaries()
        assert all(x.status == 0 for x in s), name
        assert s[0].ttft_p99 == s[1].ttft_p99, name
        print(name, "smem" if smem == "1" else "hbm", "ok", flush=True)
