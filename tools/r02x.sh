#!/bin/bash
# fused prepare + PDL + GPipe jumps: GPU parity, A/B of the launch options
# and of the GPT-2 plain-walk variants, bench.
cd "$(dirname "$0")/.."
OUT=gpurun_out/r02x; mkdir -p $OUT
timeout 900 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1; echo "exit $?" >> $OUT/pytest_gpu.log
tail -2 $OUT/pytest_gpu.log
for v in "DISTIR_PDL=0 DISTIR_FUSED_PREP=0" "DISTIR_PDL=0" "DISTIR_FUSED_PREP=0" "X=1"; do
  echo "=== env $v"; env $v timeout 300 python tools/probe_longpole.py 2>&1 | tail -8
done > $OUT/ab_env.txt 2>&1
cat $OUT/ab_env.txt
PROBE_TAIL=15 bash tools/ab_so.sh variants/plain4.so variants/plain16.so > $OUT/ab_plain.txt 2>&1
cat $OUT/ab_plain.txt
timeout 600 python bench.py --no-cpu-baseline > $OUT/bench.json 2> $OUT/bench.err
cut -c1-600 $OUT/bench.json
