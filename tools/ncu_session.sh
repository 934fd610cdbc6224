#!/bin/bash
# ncu --set full captures of the top kernels (one GPU, one kernel each)
mkdir -p gpurun_out
ncu --set full --clock-control none --import-source on -k regex:"cgemm_fused4" -c 1 -f \
    -o gpurun_out/cgemm1024_full python tools/kbench.py cgemm 1024 1 > gpurun_out/ncu_c1full.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"cgemm_fused4" -c 1 -f \
    -o gpurun_out/cgemm8192_full python tools/kbench.py cgemm 8192 1 > gpurun_out/ncu_cfull.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_matmul" -s 2 -c 1 -f \
    -o gpurun_out/matmul_s4_3x3_full python tools/kbench.py matmul 49 512 4608 3 > gpurun_out/ncu_mmfull.log 2>&1
ls -la gpurun_out/*.ncu-rep
