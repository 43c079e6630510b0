#!/bin/bash
# MLP walk-or-cache cost model: parity + A/B over crossing costs (GPipe and 1F1B grids).
cd "$(dirname "$0")/.."
OUT=gpurun_out/r02ac; mkdir -p $OUT
timeout 900 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1; echo "exit $?" >> $OUT/pytest_gpu.log
tail -2 $OUT/pytest_gpu.log
cp paper_2111_05426_b200/libdistir.so /tmp/keep.so
for so in variants/cross0.so variants/cross200.so /tmp/keep.so variants/cross1500.so; do
  echo "=== $so"; cp $so paper_2111_05426_b200/libdistir.so
  timeout 300 python tools/probe_grids.py W1 W2 W4 W5 W2:mlp_1b_1f1b W4:mlp_w4_1f1b W2:mlp_1b_zero W3 PM_1B 2>&1 | tail -9
  timeout 300 python tools/probe_longpole.py "mlpw4 P64 K128" 2>&1 | tail -1
done > $OUT/ab.txt 2>&1
cp /tmp/keep.so paper_2111_05426_b200/libdistir.so
cat $OUT/ab.txt
