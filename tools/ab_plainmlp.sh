#!/bin/bash
PROBE_TAIL=16 bash tools/variants.sh "base:" "mlp1:-DDISTIR_PLAIN_AFTER_MLP=1" "all1:-DDISTIR_PLAIN_AFTER=1"
