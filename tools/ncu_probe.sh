#!/bin/bash
# ncu --set full of one simulate launch of a single-configuration probe
#   usage: tools/ncu_probe.sh TAG "probe name" "kernel regex"
TAG=$1; NAME=$2; KRE=${3:-k_simulate<.int.1, .int.3>}
mkdir -p gpurun_out/$TAG
timeout 900 ncu --set full --warp-sampling-interval 0 --clock-control none --import-source on --kernel-name-base demangled \
  -k "regex:$KRE" --launch-skip 3 --launch-count 1 -o gpurun_out/$TAG/probe \
  python tools/probe_longpole.py "$NAME" > gpurun_out/$TAG/ncu.log 2>&1
tail -3 gpurun_out/$TAG/ncu.log
