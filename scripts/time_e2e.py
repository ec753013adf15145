"""Break down the end-to-end batch call (host staging + alloc + H2D / execute /
summaries / free) for the bench workload: python scripts/time_e2e.py [REPLICAS]"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import bench  # noqa: E402
import paper_2602_11530_b200 as pb  # noqa: E402
from harness import build_trace  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 2368
specs = bench.replica_specs("c2", 0, reps)
traces = [build_trace(r) for r, _, _ in specs]
cfgs = [pb.run_config(**c) for _, c, _ in specs]
profs = [pb.Profile.default(**p) for _, _, p in specs]
for it in range(3):
    t0 = time.perf_counter()
    b = pb.Batch(traces, profs, cfgs)
    t1 = time.perf_counter()
    b.execute()
    t2 = time.perf_counter()
    b.summaries()
    t3 = time.perf_counter()
    del b
    t4 = time.perf_counter()
    tm = pb.last_timing()
    print(f"create {1e3*(t1-t0):.0f} ms (h2d {tm.h2d_ms:.0f} ms, {tm.h2d_bytes/1e6:.0f} MB) "
          f"execute {1e3*(t2-t1):.0f} ms (device {tm.total_ms:.0f}) summaries {1e3*(t3-t2):.1f} ms "
          f"free {1e3*(t4-t3):.0f} ms")
