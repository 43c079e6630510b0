#!/bin/bash
# The full GPU round of the current tree: tests, smoke, bench, ncu launch
# list, ncu --set full of k_simulate<1,3>, and the per-grid report.
#   usage: tools/final_round.sh TAG
cd "$(dirname "$0")/.."
TAG=${1:-final}
bash tools/gpu_round.sh $TAG
tail -2 gpurun_out/$TAG/pytest_gpu.log; cat gpurun_out/$TAG/smoke.log; cut -c1-300 gpurun_out/$TAG/bench.json
timeout 1500 python tools/grid_report.py gpurun_out/$TAG/grid_report.json > gpurun_out/$TAG/grid_report.md 2> gpurun_out/$TAG/grid_report.err
tail -20 gpurun_out/$TAG/grid_report.md
