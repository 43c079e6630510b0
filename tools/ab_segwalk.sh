#!/bin/bash
PROBE_TAIL=16 bash tools/variants.sh "base:" "segwalk:-DDISTIR_SEGWALK=1" "base2:"
