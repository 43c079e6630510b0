#!/bin/bash
# 1F1B steady-state jumps: parity (1F1B suite first) + A/B.
cd "$(dirname "$0")/.."
OUT=gpurun_out/r02ag; mkdir -p $OUT
timeout 600 python -m pytest tests/test_gpu_1f1b.py tests/test_gpu_f4.py -x -q > $OUT/pytest_f1b.log 2>&1; echo "exit $?" >> $OUT/pytest_f1b.log
tail -2 $OUT/pytest_f1b.log
timeout 900 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1; echo "exit $?" >> $OUT/pytest_gpu.log
tail -2 $OUT/pytest_gpu.log
cp paper_2111_05426_b200/libdistir.so /tmp/keep.so
for so in variants/nof1bjump.so /tmp/keep.so; do
  echo "=== $so"; cp $so paper_2111_05426_b200/libdistir.so
  timeout 300 python tools/probe_grids.py W2:mlp_1b_1f1b W4:mlp_w4_1f1b W2:mlp_1b_zero_1f1b W1:mlp_w1_1f1b W2 W3 W5 2>&1 | tail -7
done > $OUT/ab.txt 2>&1
cp /tmp/keep.so paper_2111_05426_b200/libdistir.so
cat $OUT/ab.txt
