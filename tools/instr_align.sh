nvcc -gencode arch=compute_100a,code=sm_100a -lineinfo -O3 -fmad=false -std=c++17 -Xcompiler -fPIC -shared -DDISTIR_INSTR -o paper_2111_05426_b200/libdistir.so paper_2111_05426_b200/csrc/distir.cu -ldl
DISTIR_PLAN_BUDGET_X=0 PROBE_GRIDS=0 timeout 300 python tools/probe_instr.py 2>&1
