# Single-replica latency shapes: timings + one ncu source-level capture.
OUT=gpurun_out/single; mkdir -p $OUT
for c in c3_l8_pascal c4s_pascal c2_pascal c1_pascal; do
  timeout 300 python scripts/time_case.py $c 1 >> $OUT/times.txt 2>&1
done
cat $OUT/times.txt
timeout 900 ncu --set full --clock-control none --import-source on -k regex:sched_kernel \
  --launch-skip 1 --launch-count 1 -o $OUT/c3s4k -f python scripts/ncu_single.py 4000 8 8 0.9 pascal > $OUT/ncu.log 2>&1
echo "ncu exit $?"; tail -3 $OUT/ncu.log
