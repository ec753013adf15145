OUT=gpurun_out/pdes; mkdir -p $OUT
PB_PDES_DEBUG=1 timeout 600 python scripts/pdes_check.py parity > $OUT/parity.txt 2>&1; echo "parity exit $?"; tail -3 $OUT/parity.txt; grep BAD $OUT/parity.txt | head
for pd in 1; do
  PB_PDES_DEBUG=1 PB_PDES=$pd timeout 600 python scripts/pdes_check.py time c2_pascal c3_l8_pascal c3_l8_fcfs c4s_pascal c4s_fcfs >> $OUT/times.txt 2>&1
done
cat $OUT/times.txt
