# dev: invocation-run kernel -- parity + ResNet chain timing (product lib, and the dev lib with runs off) + trace
mkdir -p gpurun_out
out=gpurun_out/rn_quick.txt; : > $out
timeout 900 python -m pytest tests/test_gpu_runs.py tests/test_gpu_kernels.py -m gpu -q -p no:cacheprovider -x -k "${TESTK:-runs or resnet or builtins or matmul or saxpy}" >> $out 2>&1
echo "pytest rc=$?" >> $out
for lib in prod off; do
  if [ $lib = off ]; then export KAAS_B200_LIB=paper_2212_08146_b200/libkaas_b200_dev.so KAAS_RUN=0; fi
  echo "== resnet chain ($lib)" >> $out
  timeout 300 python -c "
import bench, json
r = bench.measure_resnet(0, steps=20)
print(json.dumps({k: r[k] for k in ('req_per_s','p50_ms','device_ms','kernel_ms','tmacs')}))
" >> $out 2>&1
done
unset KAAS_RUN
timeout 300 python tools/rtrace.py > gpurun_out/rtrace.txt 2>&1
tail -1 gpurun_out/rtrace.txt >> $out
cat $out
