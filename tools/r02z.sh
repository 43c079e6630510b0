#!/bin/bash
# jumps gated + plain walks: A/B against no jumps, then the full GPU round
# (tests, smoke, bench, ncu launch list, ncu --set full of k_simulate<1,3>).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out/r02z
PROBE_TAIL=15 bash tools/ab_so.sh variants/nojump.so paper_2111_05426_b200/libdistir.so > gpurun_out/r02z/ab.txt 2>&1
cat gpurun_out/r02z/ab.txt
bash tools/gpu_round.sh r02z
tail -2 gpurun_out/r02z/pytest_gpu.log; cat gpurun_out/r02z/smoke.log; cut -c1-300 gpurun_out/r02z/bench.json
