#!/bin/bash
# GPU-box pass for a kernel change: parity tests, long-pole probes, bench.
#   usage: tools/perf_round.sh TAG [extra pytest args]
TAG=${1:-perf}
OUT=gpurun_out/$TAG
mkdir -p "$OUT"
timeout 900 python -m pytest tests -m gpu -x -q ${2:-} > "$OUT/pytest_gpu.log" 2>&1
echo "pytest_gpu exit $?" >> "$OUT/pytest_gpu.log"
timeout 300 python tools/probe_longpole.py > "$OUT/longpole.txt" 2>&1
timeout 600 python bench.py --no-cpu-baseline > "$OUT/bench.json" 2> "$OUT/bench.err"
tail -3 "$OUT/pytest_gpu.log"; cat "$OUT/longpole.txt"; cat "$OUT/bench.json" | cut -c1-400
if [ "$3" = "ncu" ]; then
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file "$OUT/launches.csv" python bench.py --steps 5 --warmup 3 --no-cpu-baseline \
    --e2e-steps 1 > "$OUT/ncu_launch_bench.log" 2>&1
  python tools/ncu_summary.py "$OUT/launches.csv" "bench.py --steps 5 --warmup 3 (W3, B200)"
fi
