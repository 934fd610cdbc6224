mkdir -p gpurun_out
out=gpurun_out/jq.txt; : > $out
timeout 600 python -m pytest tests/test_gpu_kernels.py -m gpu -q -p no:cacheprovider -x -k "jacobi" >> $out 2>&1
for i in 1 2; do timeout 120 python tools/kbench.py jacobi 4096 500 5 >> $out 2>&1; done
timeout 300 python tools/jspan.py 2>&1 | tail -5 >> $out
cat $out
