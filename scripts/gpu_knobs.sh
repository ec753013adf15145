OUT=gpurun_out/r1g; mkdir -p $OUT
run() { # label envs...
  lab=$1; shift
  env "$@" timeout 300 python bench.py --replicas 2368 --steps 2 --warmup 1 --no-cpu-baseline > $OUT/$lab.json 2>$OUT/$lab.err
  python -c "import json; d=json.loads(open('$OUT/$lab.json').read().strip().splitlines()[-1]); print('$lab', round(d['value']/1e6,1), 'M/s step', round(d['ms_per_step'],1), 'engine', round(d['roofline']['kernel_ms'],1))" 2>&1 | tail -1
}
run base
run c256 PB_CAND_SMEM=256
run c128 PB_CAND_SMEM=128
run c256_cv50 PB_CAND_SMEM=256 PB_CARVEOUT=50
run w6 PB_MAX_WARPS_PER_SM=6
run w10 PB_MAX_WARPS_PER_SM=10
run w4 PB_MAX_WARPS_PER_SM=4
