OUT=gpurun_out/${1:-r02o}; mkdir -p $OUT
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_1f1b.py tests/test_gpu_f4.py -x -q > $OUT/pytest.log 2>&1; tail -2 $OUT/pytest.log
for so in paper_2111_05426_b200/libdistir.so variants/pm16.so variants/pm64.so variants/pm128.so; do
  [ -f /tmp/keep_done ] || { cp paper_2111_05426_b200/libdistir.so /tmp/keep.so; touch /tmp/keep_done; }
  [ "$so" -ef paper_2111_05426_b200/libdistir.so ] || cp "$so" paper_2111_05426_b200/libdistir.so
  echo "=== $so"; timeout 300 python tools/probe_grids.py W1:mlp_w1_1f1b W2:mlp_1b_1f1b W4:mlp_w4_1f1b W2 W4 W3 W5 W2:mlp_1b_zero
  cp /tmp/keep.so paper_2111_05426_b200/libdistir.so
done
