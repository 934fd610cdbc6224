# 3xFP16 cGEMM: parity + kernel timing + per-kernel launch list
mkdir -p gpurun_out
{
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_executor.py -m gpu -q -p no:cacheprovider -s -k "cgemm or fresh or replays" 2>&1 | grep -v "^$" | tail -12
for n in 1024 2048 4096 8192; do timeout 120 python tools/kbench.py cgemm $n 10; done
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed --clock-control none --csv python tools/kbench.py cgemm 8192 1 2>/dev/null | grep -v "^==" | tail -40
timeout 300 ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed --clock-control none --csv python tools/kbench.py cgemm 1024 1 2>/dev/null | grep -v "^==" | tail -20
} > gpurun_out/cg16.txt 2>&1
tail -60 gpurun_out/cg16.txt
