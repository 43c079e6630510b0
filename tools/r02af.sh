#!/bin/bash
# full GPU round of the current tree + the per-grid report.
cd "$(dirname "$0")/.."
bash tools/gpu_round.sh r02af
tail -2 gpurun_out/r02af/pytest_gpu.log; cat gpurun_out/r02af/smoke.log; cut -c1-300 gpurun_out/r02af/bench.json
timeout 1500 python tools/grid_report.py gpurun_out/r02af/grid_report.json > gpurun_out/r02af/grid_report.md 2> gpurun_out/r02af/grid_report.err
tail -25 gpurun_out/r02af/grid_report.md
