# session-3 final evidence: smoke, GPU tests, bench (both arms), launch list, ncu of the Jacobi chain and the run kernel
mkdir -p gpurun_out
timeout 180 python __graft_entry__.py smoke > gpurun_out/smoke_s3f.txt 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke_s3f.txt
timeout 2400 python -m pytest tests -m gpu -q --durations=15 -p no:cacheprovider -s > gpurun_out/gputest_s3f.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/gputest_s3f.txt
timeout 900 python bench.py > gpurun_out/bench_s3f.json 2> gpurun_out/bench_s3f.err; echo "bench rc=$?" >> gpurun_out/bench_s3f.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref_s3f.json 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 1200 --csv --log-file gpurun_out/launches_s3f.csv python bench.py --steps 2 --warmup 3 --no-extras --cpu-seconds 0.5 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_jacobi_tmem -c 1 -o gpurun_out/ncu_jacobi_s3f python tools/kbench.py jacobi 4096 500 1 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_cgemm_fused4 -c 1 -o gpurun_out/ncu_cgemm8192_s3f python tools/kbench.py cgemm 8192 1 > /dev/null 2>&1
tail -3 gpurun_out/gputest_s3f.txt; tail -2 gpurun_out/smoke_s3f.txt; tail -2 gpurun_out/bench_s3f.err
