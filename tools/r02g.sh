OUT=gpurun_out/${1:-r02g}; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_merge.py -x -q > $OUT/pytest.log 2>&1; tail -2 $OUT/pytest.log
PROBE_TAIL=16 bash tools/ab_so.sh --test paper_2111_05426_b200/libdistir.so variants/minb3.so variants/nolo.so > $OUT/ab.txt 2>&1
cp paper_2111_05426_b200/libdistir.so /tmp/k.so
cp variants/instr.so paper_2111_05426_b200/libdistir.so; PROBE_GRIDS=1 timeout 300 python tools/probe_instr.py > $OUT/instr.txt 2>&1
cp /tmp/k.so paper_2111_05426_b200/libdistir.so
cat $OUT/ab.txt
