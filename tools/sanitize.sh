#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck / initcheck on the grids
# of tools/sanitize.py (GPU box).  usage: tools/sanitize.sh OUTDIR
cd "$(dirname "$0")/.."
OUT=${1:-gpurun_out/sanitize}
mkdir -p "$OUT"
export DISTIR_NO_GRAPH=1
for tool in memcheck racecheck synccheck initcheck; do
  for g in W1 W4 W4_1F1B W2_ZERO W2_1F1B SYN W3; do
    echo "=== $tool $g" >> "$OUT/summary.txt"
    timeout 900 compute-sanitizer --tool $tool --error-exitcode 9 --print-limit 20 \
      python tools/sanitize.py $g > "$OUT/${tool}_$g.log" 2>&1
    echo "exit $?" >> "$OUT/summary.txt"
    grep -E "ERROR SUMMARY|RACECHECK SUMMARY|merge ok" "$OUT/${tool}_$g.log" >> "$OUT/summary.txt"
  done
done
cat "$OUT/summary.txt"
