OUT=gpurun_out/r2j; mkdir -p $OUT
L=paper_2602_11530_b200/libpascal.so
cp $L /tmp/libB.so; cp build/ab/libstats.so $L
timeout 300 python scripts/park_stats.py c2_pascal c3_l8_pascal c4s_pascal c5_s7_k6_pascal > $OUT/stats.txt 2>&1; cat $OUT/stats.txt | tail -6
cp /tmp/libB.so $L
timeout 900 python -m pytest tests/test_park_gpu.py -x -q -m gpu > $OUT/pytest_park.log 2>&1; echo "park tests exit $?"; tail -3 $OUT/pytest_park.log
bash scripts/gpu_ab.sh r2j/ab build/ab/libA_base.so 2368
