#!/bin/bash
# 1F1B jumps with falling live memory: parity + diagnostics + A/B.
cd "$(dirname "$0")/.."
OUT=gpurun_out/r02aj; mkdir -p $OUT
timeout 900 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1; echo "exit $?" >> $OUT/pytest_gpu.log
tail -2 $OUT/pytest_gpu.log
cp paper_2111_05426_b200/libdistir.so /tmp/keep.so
for so in variants/nof1bjump.so /tmp/keep.so; do
  echo "=== $so"; cp $so paper_2111_05426_b200/libdistir.so
  timeout 300 python tools/probe_grids.py W2:mlp_1b_1f1b W4:mlp_w4_1f1b W2:mlp_1b_zero_1f1b W1:mlp_w1_1f1b 2>&1 | tail -4
done > $OUT/ab.txt 2>&1
cp variants/instr.so paper_2111_05426_b200/libdistir.so
timeout 300 python tools/probe_jump.py W2:mlp_1b_1f1b W4:mlp_w4_1f1b >> $OUT/ab.txt 2>&1
cp /tmp/keep.so paper_2111_05426_b200/libdistir.so
cat $OUT/ab.txt
