#!/bin/bash
for x in 1 2 4 8; do
  echo "=== plan budget x$x"
  DISTIR_PLAN_BUDGET_X=$x timeout 300 python tools/probe_longpole.py 2>&1 | tail -5
done
