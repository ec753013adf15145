bash scripts/gpu_ncu_full.sh r2d 1184
