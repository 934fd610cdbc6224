# round-2 GPU session: tests, bench, Jacobi trace (dev build)
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q --durations=30 -p no:cacheprovider -s > gpurun_out/gputest.txt 2>&1; echo pytest rc=$? >> gpurun_out/gputest.txt
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench rc=$? >> gpurun_out/bench.err
timeout 300 python tools/jtrace.py > gpurun_out/jtrace.txt 2>&1
tail -3 gpurun_out/gputest.txt
