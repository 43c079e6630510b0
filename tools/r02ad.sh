#!/bin/bash
# ncu --set full of the fixed-cost kernels (prepare + select) on W3.
cd "$(dirname "$0")/.."
OUT=gpurun_out/r02ad; mkdir -p $OUT
timeout 900 ncu --set full --clock-control none --import-source on \
  -k "regex:k_reset|k_enumerate|k_plan|k_scatter|k_topk_select" --launch-skip 15 --launch-count 5 \
  -o $OUT/fixed_full python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-strong --e2e-steps 1 \
  > $OUT/ncu_fixed.log 2>&1
tail -3 $OUT/ncu_fixed.log
ncu -i $OUT/fixed_full.ncu-rep --page raw --csv --metrics gpu__time_duration.sum,sm__cycles_active.avg,smsp__inst_executed.sum,dram__bytes_read.sum > $OUT/fixed_raw.csv 2>&1
cut -c1-300 $OUT/fixed_raw.csv | head -10
