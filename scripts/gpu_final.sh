# Round-end evidence: parity suite, smoke, default bench + reference arm,
# launch list, DRAM traffic of the default config, ncu --set full at 1184.
OUT=gpurun_out/$1; mkdir -p $OUT
timeout 1500 python -m pytest tests -m gpu -q > $OUT/pytest_gpu.log 2>&1; echo "pytest exit $?"; tail -2 $OUT/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke exit $?"; tail -1 $OUT/smoke.log
bash scripts/gpu_bench_default.sh $1 | grep -v "^{" 
python -c "import json; d=json.loads(open('$OUT/bench.json').read().strip().splitlines()[-1]); print('value', d['value'], 'e2e', d['e2e']['value'], 'frac', d['roofline']['frac'])"
bash scripts/gpu_ncu_full.sh $1 1184
