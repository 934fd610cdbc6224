mkdir -p gpurun_out
ncu --set full --clock-control none --import-source on -k regex:"k_matmul" -s 3 -c 1 -f \
    -o gpurun_out/mm4608_full python tools/kbench.py matmul 49 512 4608 3 > gpurun_out/ncu_mm4608.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_matmul" -s 3 -c 1 -f \
    -o gpurun_out/mm2304_full python tools/kbench.py matmul 196 256 2304 3 > gpurun_out/ncu_mm2304.log 2>&1
ls -la gpurun_out/*.ncu-rep
