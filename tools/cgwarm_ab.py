"""Dev: warm cGEMM 8192^3 request latency (bench.measure_cgemm) under raster
group / write-back panel settings (dev build: KAAS_CGEMM_GROUPM, KAAS_CGEMM_PANELM)."""
import json
import os
import sys

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_2212_08146_b200 import native  # noqa: E402

native.init_device(0)
N = int(os.environ.get("CG_N", "8192"))
r = bench.measure_cgemm(N, 12 if N >= 4096 else 200, 0, False)
print(json.dumps({"n": N, "group": os.environ.get("KAAS_CGEMM_GROUPM", "def"), "panel": os.environ.get("KAAS_CGEMM_PANELM", "def"),
                  **{k: round(r[k], 3) for k in ("warm_req_per_s", "warm_p50_ms", "warm_device_ms", "kernel_ms")}}))
