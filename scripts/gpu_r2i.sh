OUT=gpurun_out/r2i; mkdir -p $OUT
L=paper_2602_11530_b200/libpascal.so
cp $L /tmp/libB.so; cp build/ab/libstats.so $L
timeout 300 python scripts/park_stats.py c2_pascal c3_l8_pascal c4s_pascal c5_s7_k6_pascal > $OUT/stats.txt 2>&1; cat $OUT/stats.txt | tail -6
cp /tmp/libB.so $L
