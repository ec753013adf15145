"""Time one tests/cases.py-style replica on the GPU: python scripts/time_case.py NAME [reps]"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import paper_2602_11530_b200 as pb  # noqa: E402
from paper_2602_11530_b200 import sweep  # noqa: E402
from cases import BY_NAME  # noqa: E402
from harness import build_trace, make_cfg, make_profile  # noqa: E402

name = sys.argv[1]
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 1
if name.startswith("sweep:"):
    c = {"trace": None}
    recipe, cfg, prof = sweep.replica_recipe(int(name.split(":")[1]))
    c = {"trace": recipe, "cfg": cfg, "profile": prof}
else:
    c = BY_NAME[name]
t = build_trace(c["trace"])
b = pb.Batch([t] * reps, [make_profile(c)] * reps, [make_cfg(c)] * reps)
t0 = time.perf_counter()
b.execute()
wall = time.perf_counter() - t0
s = b.summaries()[0]
tm = pb.last_timing()
print(f"{name} reps={reps} T={t.request_iterations()} status={s.status} events={s.events} "
      f"adm_rounds={s.admission_rounds} adm_slow={s.admission_slow_steps} "
      f"plans={s.plans} visits={s.candidate_visits} derive_ms={tm.derive_ms:.1f} "
      f"engine_ms={tm.engine_ms:.1f} wall_s={wall:.2f}")
