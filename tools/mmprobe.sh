L=paper_2212_08146_b200/libkaas_b200_dev.so
{
echo "== loads"; KAAS_B200_LIB=$L timeout 300 python tools/kbench.py resnet 10 | grep -E "^matmul|sum of"
echo "== no loads (compute only)"; KAAS_MM_NOLOAD=1 KAAS_B200_LIB=$L timeout 300 python tools/kbench.py resnet 10 | grep -E "^matmul|sum of"
} > gpurun_out/mmprobe.txt 2>&1
cat gpurun_out/mmprobe.txt
