OUT=gpurun_out/$1; mkdir -p $OUT
timeout 600 python -m pytest tests/test_sweep_dist.py -m gpu -q > $OUT/c5test.log 2>&1; echo "c5 test exit $?"; tail -2 $OUT/c5test.log
( time timeout 900 python -m paper_2602_11530_b200.sweep --seeds ${2:-64} --out $OUT/c5_sweep.csv ) > $OUT/c5run.log 2>&1
echo "c5 run exit $?"; tail -5 $OUT/c5run.log; head -5 $OUT/c5_sweep.csv
( time timeout 300 python -m paper_2602_11530_b200.sweep --seeds 1 --rates 2 --policies 0 --out $OUT/c5_k2.csv ) > $OUT/c5k2.log 2>&1
echo "k2 exit $?"; tail -4 $OUT/c5k2.log
