#!/bin/bash
PROBE_TAIL=16 bash tools/variants.sh "base:" "cross1+noinline:-DDISTIR_CROSS1=1 -DDISTIR_COLD_NOINLINE=1" "noinline:-DDISTIR_COLD_NOINLINE=1"
