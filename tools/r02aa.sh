#!/bin/bash
# K-gated jumps + 32-bit setup divisions: parity, A/B, instrumented probe.
cd "$(dirname "$0")/.."
OUT=gpurun_out/r02aa; mkdir -p $OUT
timeout 900 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1; echo "exit $?" >> $OUT/pytest_gpu.log
tail -2 $OUT/pytest_gpu.log
PROBE_TAIL=15 bash tools/ab_so.sh variants/nojump.so variants/jk32.so paper_2111_05426_b200/libdistir.so > $OUT/ab.txt 2>&1
cat $OUT/ab.txt
PROBE_GRIDS=1 bash tools/instr_probe.sh $OUT > /dev/null 2>&1; cat $OUT/instr.txt
