#!/bin/bash
# Build compile-time variants of libdistir.so HERE (cross-compiled, ~45 s
# each, in parallel TUs) into variants/NAME.so; on the GPU box
# tools/ab_so.sh variants/*.so times them, and
#   tools/ab_so.sh --test variants/X.so   runs the GPU parity suite on one.
# usage: tools/variants.sh "NAME:-DFLAG=1 -DX=2" ...
cd "$(dirname "$0")/.."
mkdir -p variants
for spec in "$@"; do
  name="${spec%%:*}"; flags="${spec#*:}"
  python paper_2111_05426_b200/csrc/build_lib.py $flags -o "variants/$name.so" \
    || { echo "build $name failed"; continue; }
done
