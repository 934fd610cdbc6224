# bench (ours) + launch list of the bench + ncu full capture of cgemm 8192 (traffic)
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/bench_s3.json 2> gpurun_out/bench_s3.err; echo "bench rc=$?" >> gpurun_out/bench_s3.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 1200 --csv --log-file gpurun_out/launches_s3.csv python bench.py --steps 2 --warmup 3 --no-extras --cpu-seconds 0.5 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_cgemm_fused4 -c 1 -o gpurun_out/ncu_cgemm8192_f16 python tools/kbench.py cgemm 8192 1 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_cgemm -c 1 -o gpurun_out/ncu_cgemm1024_f16 python tools/kbench.py cgemm 1024 1 > /dev/null 2>&1
tail -2 gpurun_out/bench_s3.err; ls -la gpurun_out/*.ncu-rep
