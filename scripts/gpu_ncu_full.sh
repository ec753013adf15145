# ncu --set full of the policy-run sched_kernel at REPLICAS C2 replicas.
#   bash scripts/gpu_ncu_full.sh LABEL REPLICAS
OUT=gpurun_out/$1; mkdir -p $OUT
timeout 3000 ncu --set full --clock-control none --import-source on \
  -k regex:sched_kernel --launch-skip 1 --launch-count 1 -o $OUT/prof -f \
  python bench.py --replicas $2 --steps 1 --warmup 0 --no-cpu-baseline > $OUT/ncu_full.log 2>&1
echo "ncu full exit $?"; tail -3 $OUT/ncu_full.log
