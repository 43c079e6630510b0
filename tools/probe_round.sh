mkdir -p gpurun_out/probe1
timeout 300 python tools/probe_longpole.py > gpurun_out/probe1/longpole.txt 2>&1
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:k_simulate<.int.1, .int.3>" --launch-skip 2 --launch-count 1 -o gpurun_out/probe1/simulate_full python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/probe1/ncu_full.log 2>&1
nvcc -gencode arch=compute_100a,code=sm_100a -lineinfo -O3 -fmad=false -std=c++17 -Xcompiler -fPIC -shared -DDISTIR_INSTR -o paper_2111_05426_b200/libdistir.so paper_2111_05426_b200/csrc/distir.cu -ldl && timeout 300 python tools/probe_instr.py > gpurun_out/probe1/instr.txt 2>&1
ls -la gpurun_out/probe1
