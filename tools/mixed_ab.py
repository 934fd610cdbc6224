import sys, json, os
sys.path.insert(0, '.')
import bench
for i in range(2):
    r = bench.measure_mixed(0)
    print(os.environ.get("KAAS_JACOBI_TMEM", "1"), json.dumps({k: r[k] for k in ("req_per_s", "p50_ms", "p99_ms", "device_span_sum_over_wall", "hit_rate", "evictions", "h2d_gbs")}), flush=True)
