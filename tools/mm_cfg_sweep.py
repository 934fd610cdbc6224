"""Dev: every bit-exact matmul config on each distinct ResNet-50 layer shape
(all configs give the same bytes; only speed differs) vs the cost model's pick.

    python tools/mm_cfg_sweep.py        (KAAS_MATMUL_CFG=i forces config i)
"""
import os
import subprocess
import sys

sys.path.insert(0, ".")
from paper_2212_08146_b200.workloads import resnet50_gemms  # noqa: E402

shapes = []
for _, m, n, k in resnet50_gemms():
    if (m, n, k) not in shapes:
        shapes.append((m, n, k))
tot_model, tot_best = 0.0, 0.0
for m, n, k in shapes:
    def run(cfg):
        env = dict(os.environ)
        env["KAAS_B200_LIB"] = "paper_2212_08146_b200/libkaas_b200_dev.so"
        env["KAAS_MATMUL_LK"] = "0"
        if cfg is not None:
            env["KAAS_MATMUL_CFG"] = str(cfg)
        out = subprocess.run([sys.executable, "tools/kbench.py", "matmul", str(m), str(n), str(k), "10"],
                             capture_output=True, text=True, env=env).stdout
        return float(out.split(":")[1].split("us")[0])
    model = run(None)
    times = [run(c) for c in range(14)]
    best = min(times)
    tot_model += model
    tot_best += best
    print(f"{m:6d}x{n:5d}x{k:5d}: model {model:7.1f} us  best {best:7.1f} us (cfg {times.index(best)})  "
          + " ".join(f"{t:.0f}" for t in times), flush=True)
print(f"sum over distinct shapes: model {tot_model:.1f} us, best {tot_best:.1f} us")
