#!/bin/bash
# PDL on/off in the unprofiled bench loop, k_plan split budget, GPT-2 plain walks.
cd "$(dirname "$0")/.."
OUT=gpurun_out/r02y; mkdir -p $OUT
timeout 900 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1; echo "exit $?" >> $OUT/pytest_gpu.log
tail -2 $OUT/pytest_gpu.log
for i in 1 2; do
  for v in "DISTIR_PDL=0" "DISTIR_PDL=1"; do
    env $v timeout 300 python bench.py --no-cpu-baseline --no-strong --e2e-steps 20 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$v', 'ms/step %.4f' % d['ms_per_step'], d['kernel_ms_per_step'], 'e2e', d['e2e']['value'])"
  done
done > $OUT/pdl.txt 2>&1
cat $OUT/pdl.txt
for x in 1 1.5 2 4; do
  echo "=== PLAN_BUDGET_X $x"; DISTIR_PLAN_BUDGET_X=$x timeout 300 python tools/probe_longpole.py 2>&1 | tail -5
done > $OUT/plan.txt 2>&1
cat $OUT/plan.txt
PROBE_TAIL=15 bash tools/ab_so.sh paper_2111_05426_b200/libdistir.so variants/plain8.so variants/plain16.so > $OUT/ab_plain.txt 2>&1
cat $OUT/ab_plain.txt
