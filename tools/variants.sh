#!/bin/bash
# Build compile-time variants of libdistir.so and probe each (GPU box).
# usage: tools/variants.sh "NAME:-DFLAG=1 -DX=2" ...
cd "$(dirname "$0")/.."
cp paper_2111_05426_b200/libdistir.so /tmp/libdistir.keep.so
for spec in "$@"; do
  name="${spec%%:*}"; flags="${spec#*:}"
  nvcc -gencode arch=compute_100a,code=sm_100a -lineinfo -O3 -fmad=false -std=c++17 \
    -Xcompiler -fPIC -shared $flags -o paper_2111_05426_b200/libdistir.so \
    paper_2111_05426_b200/csrc/distir.cu -ldl || { echo "build $name failed"; continue; }
  echo "=== $name ($flags)"
  timeout 300 python tools/probe_longpole.py ${PROBE_ONLY:-} 2>&1 | tail -${PROBE_TAIL:-7}
done
cp /tmp/libdistir.keep.so paper_2111_05426_b200/libdistir.so
