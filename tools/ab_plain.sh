#!/bin/bash
PROBE_TAIL=16 bash tools/variants.sh "nos1:-DDISTIR_PLAIN_S1=0" "s1:-DDISTIR_PLAIN_S1=1" "s1x2:-DDISTIR_PLAIN_S1=2"
