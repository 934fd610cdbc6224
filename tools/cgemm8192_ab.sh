# dev: warm cGEMM 8192 request A/B of build/var libs (same box, alternating)
mkdir -p gpurun_out
out=gpurun_out/cg8_ab.txt; : > $out
run() { timeout 600 python -c "
import sys, json; sys.path.insert(0, '.')
import bench
r = bench.measure_cgemm(8192, 5, 0, False)
print('$1', json.dumps({k: round(r[k], 3) for k in ('warm_req_per_s', 'warm_p50_ms', 'kernel_ms')}))
"; }
for i in 1 2; do
  run default >> $out 2>&1
  for v in build/var/*.so; do KAAS_B200_LIB=$v run $(basename $v .so) >> $out 2>&1; done
done
cat $out
