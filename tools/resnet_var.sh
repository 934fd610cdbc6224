# dev: ResNet chain A/B of build/var libs (bit-exact subset first)
mkdir -p gpurun_out
out=gpurun_out/rnv2.txt; : > $out
run() { timeout 300 python -c "
import sys, json; sys.path.insert(0, '.')
import bench
r = bench.measure_resnet(0, steps=10)
print('$1', json.dumps({k: round(r[k], 4) for k in ('req_per_s', 'kernel_ms')}))
"; }
for v in build/var/*.so; do echo "== parity $v" >> $out; KAAS_B200_LIB=$v timeout 300 python -m pytest tests -m gpu -q -p no:cacheprovider -x -k "matmul or resnet or builtins" 2>&1 | tail -1 >> $out; done
for i in 1 2 3; do
  run default >> $out 2>&1
  for v in build/var/*.so; do KAAS_B200_LIB=$v run $(basename $v .so) >> $out 2>&1; done
done
cat $out
