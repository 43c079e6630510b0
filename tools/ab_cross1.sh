timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
PROBE_TAIL=16 bash tools/variants.sh "nocross:-DDISTIR_CROSS1=0" "cross1:-DDISTIR_CROSS1=1"
