OUT=gpurun_out/r02b; mkdir -p $OUT
timeout 900 python -m pytest tests -m gpu -x -q > $OUT/pytest.log 2>&1; tail -3 $OUT/pytest.log
bash tools/ab_so.sh paper_2111_05426_b200/libdistir.so variants/noquick.so > $OUT/ab.txt 2>&1
cp paper_2111_05426_b200/libdistir.so /tmp/k.so
for v in instr instr_noquick; do cp variants/$v.so paper_2111_05426_b200/libdistir.so; timeout 300 python tools/probe_instr.py > $OUT/$v.txt 2>&1; done
cp /tmp/k.so paper_2111_05426_b200/libdistir.so
cat $OUT/ab.txt
