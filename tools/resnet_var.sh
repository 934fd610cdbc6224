mkdir -p gpurun_out
run() { timeout 300 python -c "
import sys, json; sys.path.insert(0, '.')
import bench
r = bench.measure_resnet(0, steps=10)
print('$1', json.dumps({k: r[k] for k in ('req_per_s', 'kernel_ms')}))
"; }
run default > gpurun_out/rnv2.txt 2>&1
for v in build/var/*.so; do KAAS_B200_LIB=$v run $(basename $v .so) >> gpurun_out/rnv2.txt 2>&1; done
cat gpurun_out/rnv2.txt
