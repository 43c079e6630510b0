#!/bin/bash
# 1F1B jumps over 4-period windows; tail copy in the e2e path: parity + A/B + bench.
cd "$(dirname "$0")/.."
OUT=gpurun_out/r02ah; mkdir -p $OUT
timeout 600 python -m pytest tests/test_gpu_1f1b.py tests/test_gpu_f4.py tests/test_gpu_parity.py -x -q > $OUT/pytest_f1b.log 2>&1; echo "exit $?" >> $OUT/pytest_f1b.log
tail -2 $OUT/pytest_f1b.log
cp paper_2111_05426_b200/libdistir.so /tmp/keep.so
for so in variants/nof1bjump.so /tmp/keep.so; do
  echo "=== $so"; cp $so paper_2111_05426_b200/libdistir.so
  timeout 300 python tools/probe_grids.py W2:mlp_1b_1f1b W4:mlp_w4_1f1b W2:mlp_1b_zero_1f1b W3 2>&1 | tail -4
done > $OUT/ab.txt 2>&1
cp /tmp/keep.so paper_2111_05426_b200/libdistir.so
cat $OUT/ab.txt
timeout 600 python bench.py --no-cpu-baseline --no-strong > $OUT/bench.json 2> $OUT/bench.err
python -c "import json;d=json.load(open('$OUT/bench.json'));print(d['ms_per_step'], d['e2e'], d['time_to_best_ms'])"
