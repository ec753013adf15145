"""Parked-tail counters of a stats build (-DPB_PARK_STATS: admission_rounds =
skipped parked visits, admission_slow_steps = 16-bit fields: re-plans because
a resident ranked after the tail was still there / the free KV reached a
member's need / the stack held a class-1 resident or nothing was admitted,
and plans that skipped their parked tail)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import paper_2602_11530_b200 as pb  # noqa: E402
from cases import BY_NAME  # noqa: E402
from harness import build_trace, make_cfg, make_profile  # noqa: E402

for name in sys.argv[1:] or ["c2_pascal"]:
    c = BY_NAME[name]
    t = build_trace(c["trace"])
    b = pb.Batch([t] * 8, [make_profile(c)] * 8, [make_cfg(c)] * 8)
    b.execute()
    s = b.summaries()[0]
    v = s.admission_slow_steps
    fa, fb, fc, sk = v & 0xffff, (v >> 16) & 0xffff, (v >> 32) & 0xffff, v >> 48
    print(f"{name}: plans {s.plans} visits {s.candidate_visits} skipped {s.admission_rounds} "
          f"({100.0 * s.admission_rounds / max(1, s.candidate_visits):.1f}%) re-plans "
          f"resident {fa} free {fb} other {fc} ({100.0 * (fa + fb + fc) / max(1, s.plans):.1f}% "
          f"of plans; fields mod 65536), skipping plans {sk} ({100.0 * sk / max(1, s.plans):.1f}%)")
