#!/bin/bash
# ncu --set full of the fixed-cost kernels of one W3 launch
mkdir -p gpurun_out/ncufixed
timeout 900 ncu --set full --warp-sampling-interval 0 --clock-control none --import-source on --kernel-name-base demangled \
  -k "regex:k_plan|k_topk|k_enumerate|k_scatter|k_reset" --launch-skip 10 --launch-count 5 -o gpurun_out/ncufixed/fixed \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-strong --e2e-steps 1 > gpurun_out/ncufixed/ncu.log 2>&1
tail -2 gpurun_out/ncufixed/ncu.log
