OUT=gpurun_out/$1; mkdir -p $OUT
( time timeout 300 python -m paper_2602_11530_b200.sweep --seeds 4 --rates 0 1 2 --out $OUT/c5_low.csv ) > $OUT/c5low.log 2>&1
echo "low exit $?"; tail -5 $OUT/c5low.log
( time timeout 2400 python -m paper_2602_11530_b200.sweep --seeds 4096 --rates $(seq 0 15) --chunk 9472 --out $OUT/c5_full.csv ) > $OUT/c5full.log 2>&1
echo "full exit $?"; tail -5 $OUT/c5full.log
