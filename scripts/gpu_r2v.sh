# A/B of the last micro-optimisations + host staging, sanitizers on the parked-tail path
bash scripts/gpu_abn.sh r2v 2368 build/ab/libJ2_head.so build/ab/libM2_host_pref.so
OUT=gpurun_out/r2v/san; mkdir -p $OUT
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck racecheck synccheck; do
  if [ $tool = memcheck ]; then unset PARK_SAN_LIGHT; else export PARK_SAN_LIGHT=1; fi
  timeout 1200 $CS --tool $tool --print-limit 20 --error-exitcode 9 python scripts/sanitize_park.py > $OUT/$tool.log 2>&1
  echo "$tool exit $?"; tail -2 $OUT/$tool.log
done
