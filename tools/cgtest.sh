{
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_executor.py -m gpu -q -p no:cacheprovider -k "cgemm or fresh or replays" 2>&1 | tail -3
for n in 1024 2048 4096 8192; do timeout 120 python tools/kbench.py cgemm $n 10; done
echo "== whole tiles only (dev)"; for n in 1024 2048; do KAAS_CGEMM_STREAMK=0 KAAS_B200_LIB=paper_2212_08146_b200/libkaas_b200_dev.so timeout 120 python tools/kbench.py cgemm $n 10; done
} > gpurun_out/cgtest.txt 2>&1
cat gpurun_out/cgtest.txt
