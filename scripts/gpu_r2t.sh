bash scripts/gpu_abn.sh r2t 2368 build/ab/libI_heap.so build/ab/libJ_nlog.so
OUT=gpurun_out/r2t; mkdir -p $OUT
timeout 1800 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1; echo "pytest exit $?"; tail -3 $OUT/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke exit $?"
