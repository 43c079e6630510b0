#!/bin/bash
# One GPU-box pass (run under gpurun from the repo root): GPU tests, smoke,
# the default bench line, the ncu launch list of the same command, and one
# `ncu --set full` capture of the dominant kernel.  Outputs in gpurun_out/$TAG.
#   usage: tools/gpu_round.sh TAG [skip-tests] [skip-ncu]
TAG=${1:-r01}
OUT=gpurun_out/$TAG
mkdir -p "$OUT"
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > "$OUT/gpu.txt" 2>&1
nproc > "$OUT/nproc.txt"; lscpu | head -20 >> "$OUT/nproc.txt"
if [ "$2" != "skip-tests" ]; then
  timeout 1200 python -m pytest tests -m gpu -x -q > "$OUT/pytest_gpu.log" 2>&1
  echo "pytest_gpu exit $?" >> "$OUT/pytest_gpu.log"
  timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > "$OUT/smoke.log" 2>&1
  echo "smoke exit $?" >> "$OUT/smoke.log"
fi
timeout 900 python bench.py > "$OUT/bench.json" 2> "$OUT/bench.err"
echo "bench exit $?" >> "$OUT/bench.err"
if [ "$3" != "skip-ncu" ]; then
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file "$OUT/launches.csv" python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-strong \
    --e2e-steps 1 > "$OUT/ncu_launch_bench.log" 2>&1
  timeout 900 ncu --set full --clock-control none --import-source on --warp-sampling-interval 2 \
    --kernel-name-base demangled -k "regex:k_simulate<.int.1, .int.3>" --launch-skip 2 --launch-count 2 -o "$OUT/simulate_full" \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-strong --e2e-steps 1 \
    > "$OUT/ncu_full.log" 2>&1
  python tools/ncu_capture.py "$OUT/simulate_full.ncu-rep" "$OUT/ncu_simulate_summary.json" \
    "k_simulate<1,3> on W3 x TB200 (bench.py --steps 2 --warmup 3, launches 3-4)" > "$OUT/ncu_capture.log" 2>&1
  python tools/ncu_summary.py "$OUT/launches.csv" "bench.py --steps 5 --warmup 3 (W3, B200)" \
    > "$OUT/launches_summary.csv" 2>&1
fi
ls -la "$OUT"
