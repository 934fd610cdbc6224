mkdir -p gpurun_out
{
timeout 900 python -m pytest tests/test_gpu_kernels.py -m gpu -q -p no:cacheprovider -k "matmul or resnet or builtins" 2>&1 | tail -3
timeout 300 python tools/kbench.py resnet 10 | grep -E "^matmul|sum of"
echo "== dev lib, chain kernel off"; KAAS_MATMUL_LK=0 KAAS_B200_LIB=paper_2212_08146_b200/libkaas_b200_dev.so timeout 300 python tools/kbench.py resnet 10 | grep -E "sum of"
echo "== dev lib, chain kernel on everywhere k%4==0"; KAAS_MATMUL_LK=1 KAAS_B200_LIB=paper_2212_08146_b200/libkaas_b200_dev.so timeout 300 python tools/kbench.py resnet 10 | grep -E "^matmul|sum of"
} > gpurun_out/mmtest.txt 2>&1
cat gpurun_out/mmtest.txt
