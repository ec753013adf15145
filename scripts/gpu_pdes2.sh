OUT=gpurun_out/pdes; mkdir -p $OUT
PB_PDES_DEBUG=1 timeout 600 python scripts/pdes_check.py time c2_pascal c3_l8_pascal c3_l8_fcfs c4s_pascal c4s_fcfs > $OUT/times2.txt 2>&1
cat $OUT/times2.txt
# racecheck on two small multi-instance cases through the instance-parallel engine
cat > /tmp/rc.py <<'PY'
import os, sys
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.path.join(os.getcwd(), "tests"))
import paper_2602_11530_b200 as pb
from cases import BY_NAME
from harness import build_trace, make_cfg, make_profile
for n in ("abl60_pascal", "det77_oracle", "fabric_pascal", "wide40_fcfs"):
    c = BY_NAME[n]; t = build_trace(c["trace"])
    b = pb.Batch([t], [make_profile(c)], [make_cfg(c)]); b.execute()
    print(n, b.summaries()[0].status, pb.last_timing().instance_parallel, flush=True)
PY
timeout 900 /usr/local/cuda/bin/compute-sanitizer --tool racecheck --racecheck-report hazard --print-limit 20 python /tmp/rc.py > $OUT/racecheck_pdes.log 2>&1
echo "racecheck exit $?"; grep -E "SUMMARY|^[a-z]" $OUT/racecheck_pdes.log | tail; grep -B1 -A3 "Error" $OUT/racecheck_pdes.log | head -30
