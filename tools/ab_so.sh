#!/bin/bash
# A/B prebuilt libraries on one GPU box: tools/ab_so.sh [--test] A.so B.so ...
# Each library is swapped in, probed (tools/probe_longpole.py) and, with
# --test, run through the GPU parity suite; the original is restored.
cd "$(dirname "$0")/.."
TEST=0
if [ "$1" = "--test" ]; then TEST=1; shift; fi
cp paper_2111_05426_b200/libdistir.so /tmp/keep.so; set -- "${@/paper_2111_05426_b200\/libdistir.so//tmp/keep.so}"
for so in "$@"; do
  echo "=== $so"; [ "$so" -ef paper_2111_05426_b200/libdistir.so ] || cp "$so" paper_2111_05426_b200/libdistir.so
  timeout 300 python tools/probe_longpole.py ${PROBE_ONLY:-} 2>&1 | tail -${PROBE_TAIL:-6}
  if [ $TEST = 1 ]; then
    timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
  fi
done
cp /tmp/keep.so paper_2111_05426_b200/libdistir.so
