#!/bin/bash
# One GPU session: tests, bench (both arms), launch list, ncu captures of the top kernels.
mkdir -p gpurun_out
python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1
python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
python bench.py --impl reference --steps 5 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 2 --warmup 3 --no-extras --cpu-seconds 0 > gpurun_out/ncu_bench.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"jacobi_(rows|cols)" -s 2 -c 1 \
    -o gpurun_out/jacobi_full python bench.py --steps 1 --warmup 3 --no-extras --cpu-seconds 0 > gpurun_out/ncu_jfull.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"cgemm_(tf32|fused)" -c 1 \
    -o gpurun_out/cgemm8192_full python tools/kbench.py cgemm 8192 1 > gpurun_out/ncu_cfull.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"cgemm_(tf32|fused)" -c 1 \
    -o gpurun_out/cgemm1024_full python tools/kbench.py cgemm 1024 1 > gpurun_out/ncu_c1full.log 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
tail -3 gpurun_out/gpu_tests.log; cat gpurun_out/smoke.log; cat gpurun_out/bench.json
