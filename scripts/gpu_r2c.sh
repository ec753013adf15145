OUT=gpurun_out/r2c; mkdir -p $OUT
timeout 900 python -m pytest tests/test_unit_probe.py tests/test_callers.py tests/test_tpot_gpu.py tests/test_multi_device.py -q -m gpu > $OUT/pytest_new.log 2>&1; echo "pytest new exit $?"; tail -30 $OUT/pytest_new.log | cut -c1-400
