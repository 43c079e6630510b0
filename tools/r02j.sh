OUT=gpurun_out/${1:-r02j}; mkdir -p $OUT
PROBE_TAIL=16 bash tools/ab_so.sh --test paper_2111_05426_b200/libdistir.so variants/ties0.so variants/ties2.so > $OUT/ab.txt 2>&1
cat $OUT/ab.txt
