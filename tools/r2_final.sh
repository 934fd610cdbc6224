# round-2 evidence session: GPU tests, smoke, bench (ours + reference arm), launch list
mkdir -p gpurun_out
timeout 180 python __graft_entry__.py smoke > gpurun_out/smoke_final.txt 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke_final.txt
timeout 2400 python -m pytest tests -m gpu -q --durations=20 -p no:cacheprovider -s > gpurun_out/gputest_final.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/gputest_final.txt
timeout 900 python bench.py > gpurun_out/bench_final.json 2> gpurun_out/bench_final.err; echo "bench rc=$?" >> gpurun_out/bench_final.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref_final.json 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 1200 --csv --log-file gpurun_out/launches_final.csv python bench.py --steps 2 --warmup 3 --no-extras --cpu-seconds 0.5 > /dev/null 2>&1
tail -3 gpurun_out/gputest_final.txt; cat gpurun_out/smoke_final.txt | tail -2; tail -2 gpurun_out/bench_final.err
