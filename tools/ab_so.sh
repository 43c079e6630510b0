#!/bin/bash
# A/B two prebuilt libraries on one box: tools/ab_so.sh A.so B.so
cp paper_2111_05426_b200/libdistir.so /tmp/keep.so
for so in "$@"; do
  echo "=== $so"; cp "$so" paper_2111_05426_b200/libdistir.so
  timeout 300 python tools/probe_longpole.py 2>&1 | tail -${PROBE_TAIL:-6}
done
cp /tmp/keep.so paper_2111_05426_b200/libdistir.so
