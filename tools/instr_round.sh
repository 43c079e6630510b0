mkdir -p gpurun_out/instr2
nvcc -gencode arch=compute_100a,code=sm_100a -lineinfo -O3 -fmad=false -std=c++17 -Xcompiler -fPIC -shared -DDISTIR_INSTR -o paper_2111_05426_b200/libdistir.so paper_2111_05426_b200/csrc/distir.cu -ldl && timeout 300 python tools/probe_instr.py > gpurun_out/instr2/instr.txt 2>&1
cat gpurun_out/instr2/instr.txt
