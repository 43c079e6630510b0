#!/bin/bash
# shared GPT-2 cost divisions, MLP jumps off: parity + A/B.
cd "$(dirname "$0")/.."
OUT=gpurun_out/r02ab; mkdir -p $OUT
timeout 900 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1; echo "exit $?" >> $OUT/pytest_gpu.log
tail -2 $OUT/pytest_gpu.log
PROBE_TAIL=15 bash tools/ab_so.sh variants/noshared.so variants/mlpjump.so paper_2111_05426_b200/libdistir.so > $OUT/ab.txt 2>&1
cat $OUT/ab.txt
