#!/bin/bash
PROBE_TAIL=16 bash tools/variants.sh "base:" "unroll:-DDISTIR_UNROLL_SEG=1" "unroll+cross1:-DDISTIR_UNROLL_SEG=1 -DDISTIR_CROSS1=1"
