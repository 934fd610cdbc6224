"""Dev: peer-fill measurement after each other bench workload (order effects)."""
import json
import sys

sys.path.insert(0, ".")
import bench  # noqa: E402

which = sys.argv[1:] or ["none"]
for w in which:
    if w == "resnet":
        bench.measure_resnet(0)
    elif w == "mixed":
        bench.measure_mixed(0)
    elif w == "cgemm8192":
        bench.measure_cgemm(8192, 5, 0, True)
    elif w.startswith("sleep"):
        import time
        time.sleep(float(w[5:]))
    elif w == "cgemm1024":
        bench.measure_cgemm(1024, 20, 0, True)
    if w.startswith("sleep"):
        continue
    r = bench.measure_peer_fill(0)
    import subprocess
    smi = subprocess.run(["nvidia-smi", "--query-gpu=clocks.sm,clocks.mem,power.draw,clocks_event_reasons.active",
                          "--format=csv,noheader"], capture_output=True, text=True).stdout.strip()
    print(w, json.dumps({k: round(r[k], 1) for k in ("h2d_gbs", "p2p_gbs")}), smi, flush=True)

if "timeline" in sys.argv:
    import subprocess
    import time
    from paper_2212_08146_b200 import native
    bench.measure_cgemm(8192, 5, 0, True)
    s = native.Stream(0)
    a = native.malloc_async(s, 1 << 30)
    b = native.malloc_async(s, 1 << 30)
    e0, e1 = native.Event(0, True), native.Event(0, True)
    t0 = time.perf_counter()
    for i in range(24):
        e0.record(s)
        native.d2d_async(b, a, 1 << 30, s)
        e1.record(s)
        e1.sync()
        smi = subprocess.run(["nvidia-smi", "--query-gpu=clocks.sm,clocks.mem,power.draw,temperature.gpu,"
                              "temperature.memory,clocks_event_reasons.active", "--format=csv,noheader"],
                             capture_output=True, text=True).stdout.strip()
        print(f"t={time.perf_counter() - t0:5.2f}s D2D {(1 << 30) / (e0.elapsed_ms(e1) * 1e6):7.1f} GB/s  {smi}",
              flush=True)
        time.sleep(0.25)
