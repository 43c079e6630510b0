#!/bin/bash
cp paper_2111_05426_b200/libdistir.so /tmp/keep.so
for spec in "s1:-DDISTIR_F1B_SENDS=1" "s2:-DDISTIR_F1B_SENDS=2" "s3:-DDISTIR_F1B_SENDS=3"; do
  name="${spec%%:*}"; flags="${spec#*:}"
  nvcc -gencode arch=compute_100a,code=sm_100a -lineinfo -O3 -fmad=false -std=c++17 -Xcompiler -fPIC -shared $flags -o paper_2111_05426_b200/libdistir.so paper_2111_05426_b200/csrc/distir.cu -ldl
  echo "=== $name"; (cd tools && timeout 300 python probe_f1b.py 2>&1 | tail -3)
done
cp /tmp/keep.so paper_2111_05426_b200/libdistir.so
timeout 900 python -m pytest tests/test_gpu_1f1b.py tests/test_gpu_f4.py tests/test_gpu_regression.py -x -q 2>&1 | tail -2
