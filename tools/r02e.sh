OUT=gpurun_out/${1:-r02e}; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q > $OUT/pytest.log 2>&1; tail -2 $OUT/pytest.log
PROBE_TAIL=16 bash tools/ab_so.sh paper_2111_05426_b200/libdistir.so variants/plain0.so > $OUT/ab.txt 2>&1
cp paper_2111_05426_b200/libdistir.so /tmp/k.so
cp variants/instr.so paper_2111_05426_b200/libdistir.so; PROBE_GRIDS=1 timeout 300 python tools/probe_instr.py > $OUT/instr.txt 2>&1
cp /tmp/k.so paper_2111_05426_b200/libdistir.so
for c in "gpt2_xl 16 128" "gpt2_xl 2 2"; do
  tag=$(echo $c | tr ' ' _)
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_simulate --launch-skip 3 --launch-count 1 \
    -o $OUT/one_$tag python tools/probe_one.py $c > $OUT/ncu_$tag.log 2>&1
done
cat $OUT/ab.txt
