# parked tails (PB_PARK): parity of the lean Pascal build, then an A/B against the previous build
OUT=gpurun_out/r2h; mkdir -p $OUT
timeout 900 python -m pytest tests/test_park_gpu.py -x -q -m gpu > $OUT/pytest_park.log 2>&1; echo "park tests exit $?"; tail -3 $OUT/pytest_park.log
timeout 900 python -m pytest tests/test_batch_gpu.py tests/test_tpot_gpu.py tests/test_sweep_cli.py -x -q -m gpu > $OUT/pytest_batch.log 2>&1; echo "batch tests exit $?"; tail -2 $OUT/pytest_batch.log
bash scripts/gpu_ab.sh r2h/ab build/ab/libA_base.so 2368
