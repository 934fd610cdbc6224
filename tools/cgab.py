"""Interleaved A/B of cGEMM variants under sustained load (dev lib: the
variant switches are read per launch).  Prints ms/launch and the median SM
clock / power over each block of launches.

    KAAS_B200_LIB=paper_2212_08146_b200/libkaas_b200_dev.so python tools/cgab.py n reps rounds
"""
import os
import sys
import threading
import time

import numpy as np

sys.path.insert(0, ".")
from paper_2212_08146_b200 import native  # noqa: E402
from paper_2212_08146_b200.api import LaunchDims, i32  # noqa: E402
from paper_2212_08146_b200.kernels import default_registry, fill_desc  # noqa: E402
from tools.kbench import dev_buf, timed  # noqa: E402

VARIANTS = [("pair g8", {"KAAS_CGEMM_PAIR": "1", "KAAS_CGEMM_GROUPM": "8"}),
            ("pair g4", {"KAAS_CGEMM_PAIR": "1", "KAAS_CGEMM_GROUPM": "4"}),
            ("1cta g8", {"KAAS_CGEMM_PAIR": "0", "KAAS_CGEMM_GROUPM": "8"}),
            ("1cta g16", {"KAAS_CGEMM_PAIR": "0", "KAAS_CGEMM_GROUPM": "16"})]


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
    reps = int(sys.argv[2]) if len(sys.argv) > 2 else 20
    rounds = int(sys.argv[3]) if len(sys.argv) > 3 else 3
    import pynvml
    pynvml.nvmlInit()
    h = pynvml.nvmlDeviceGetHandleByIndex(0)
    k = default_registry().get("cgemm")
    s = native.Stream(0)
    rng = np.random.default_rng(0)
    pA = dev_buf(s, rng.standard_normal(2 * n * n, dtype=np.float32).tobytes())
    pB = dev_buf(s, rng.standard_normal(2 * n * n, dtype=np.float32).tobytes())
    pC = native.malloc_async(s, 8 * n * n)
    d = (native.LaunchDesc * 1)()
    fill_desc(d[0], k, LaunchDims(grid_x=n * n), (i32(n), i32(n), i32(n)), [pA, pB, pC], [8 * n * n] * 3)
    variants = VARIANTS
    if os.environ.get("CGAB_ONLY"):
        variants = [v for v in VARIANTS if v[0] in os.environ["CGAB_ONLY"].split(",")]
    res = {name: [] for name, _ in variants}
    for r in range(rounds):
        for name, env in (variants if r % 2 == 0 else variants[::-1]):
            os.environ.update(env)
            samples, stop = [], threading.Event()

            def sample():
                while not stop.is_set():
                    samples.append((pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM),
                                    pynvml.nvmlDeviceGetPowerUsage(h) / 1000))
                    time.sleep(0.005)
            t = threading.Thread(target=sample)
            t.start()
            ms = timed(s, lambda: native.launch_batch(0, s, d), reps)
            stop.set()
            t.join()
            clk = float(np.median([a for a, _ in samples])) if samples else 0
            pw = float(np.median([b for _, b in samples])) if samples else 0
            res[name].append(ms)
            useful = 8.0 * n ** 3
            print(f"round {r} {name:9s} n={n}: {ms:8.3f} ms  tf32-issued {3 * useful / ms / 1e9:6.1f} TFLOP/s  "
                  f"sm {clk:.0f} MHz  {pw:.0f} W", flush=True)
    for name, v in res.items():
        print(f"{name:9s} median {np.median(v):.3f} ms  min {min(v):.3f}")


if __name__ == "__main__":
    main()
