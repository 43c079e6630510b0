#!/bin/bash
# A/B on one box: simulate kernels at 1, 2, 3 resident blocks per SM
for b in 3 2 1; do
  echo "=== blocks/SM $b"
  DISTIR_SIM_BLOCKS_PER_SM=$b timeout 300 python tools/probe_longpole.py 2>&1 | tail -5
done
