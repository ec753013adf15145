# compute-sanitizer memcheck / racecheck / synccheck over scripts/sanitize_cases.py
OUT=gpurun_out/sanitizer; mkdir -p $OUT
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck racecheck synccheck; do
  for mode in auto hbm; do
    if [ $mode = hbm ]; then export PB_SMEM=0 PB_SMEM_HEAP=4; else unset PB_SMEM PB_SMEM_HEAP; fi
    timeout 900 $CS --tool $tool --print-limit 50 --error-exitcode 9 \
      python scripts/sanitize_cases.py > $OUT/${tool}_${mode}.log 2>&1
    echo "$tool $mode exit $?" | tee -a $OUT/summary.txt
    tail -4 $OUT/${tool}_${mode}.log
  done
done
