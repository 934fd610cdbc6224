mkdir -p gpurun_out
{
timeout 120 python tools/kbench.py cgemm 8192 5
timeout 120 python tools/kbench.py cgemm 1024 20
timeout 300 python tools/kbench.py resnet 10
} > gpurun_out/cg_kbench.txt 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_cgemm_fused4 -s 1 -c 1 -o gpurun_out/cg8192_r2 python tools/kbench.py cgemm 8192 1 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_cgemm_fused4 -s 1 -c 1 -o gpurun_out/cg1024_r2 python tools/kbench.py cgemm 1024 1 > /dev/null 2>&1
cat gpurun_out/cg_kbench.txt
