"""One single-replica run of a chat-preset trace (C3 shape scaled by N) for
ncu source-level profiling: python scripts/ncu_single.py N RATE INSTANCES CAP POLICY"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2602_11530_b200 as pb  # noqa: E402

n, rate, ni, cap, pol = int(sys.argv[1]), float(sys.argv[2]), int(sys.argv[3]), float(sys.argv[4]), sys.argv[5]
t = pb.Trace.preset("chat", n, rate, 1)
b = pb.Batch([t], [pb.Profile.default()], [pb.run_config(pol, instance_count=ni, capacity_fraction=cap)])
b.execute()
s = b.summaries()[0]
tm = pb.last_timing()
print(f"n={n} status={s.status} T={t.request_iterations()} events={s.events} plans={s.plans} "
      f"visits={s.candidate_visits} derive_ms={tm.derive_ms:.1f} engine_ms={tm.engine_ms:.1f}")
