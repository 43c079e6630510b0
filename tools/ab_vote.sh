#!/bin/bash
PROBE_TAIL=16 bash tools/variants.sh "vote:-DDISTIR_VOTE=1" "novote:-DDISTIR_VOTE=0"
