#!/bin/bash
# GPU box: instrumented probe (variants/instr.so, built with
# tools/variants.sh "instr:-DDISTIR_INSTR") + the long-pole probe of the
# current library.  usage: tools/instr_probe.sh OUTDIR
cd "$(dirname "$0")/.."
OUT=${1:-gpurun_out/instr}
mkdir -p "$OUT"
timeout 300 python tools/probe_longpole.py > "$OUT/longpole.txt" 2>&1
cp paper_2111_05426_b200/libdistir.so /tmp/keep.so
cp variants/instr.so paper_2111_05426_b200/libdistir.so
DISTIR_PLAN_BUDGET_X=${PLAN_X:-1} timeout 300 python tools/probe_instr.py > "$OUT/instr.txt" 2>&1
cp /tmp/keep.so paper_2111_05426_b200/libdistir.so
cat "$OUT/longpole.txt" "$OUT/instr.txt"
