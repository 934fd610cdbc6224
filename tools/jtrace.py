"""Dev: per-CTA phase timestamps of the Jacobi column kernel (sweeps 100..131).

    make -C paper_2212_08146_b200/csrc dev   # the trace exists only in the dev build
    python tools/jtrace.py [n]

Stamps (globaltimer, ns): t0 = CTA's warp 0 has its x, t1 = warp 0's row
partials done, t2 = the CTA's rows published.  Prints the per-sweep spread
of each phase across CTAs and the critical path from publish to the next
sweep's x arrival.
"""

import ctypes as C
import os
import sys

import numpy as np

sys.path.insert(0, ".")
os.environ.setdefault("KAAS_JACOBI_TRACE", "1")
os.environ.setdefault("KAAS_B200_LIB", "paper_2212_08146_b200/libkaas_b200_dev.so")
from paper_2212_08146_b200 import native  # noqa: E402
sys.argv = [sys.argv[0], "jacobi"] + sys.argv[1:2] + ["500", "1"]
sys.path.insert(0, "tools")
import kbench  # noqa: E402

n = int(sys.argv[2]) if len(sys.argv) > 2 else 4096
kbench.jacobi(n, 500, 1)
buf = (C.c_uint * (32 * 148 * 3))()
rc = native.load().kaas_dev_jacobi_trace(buf, C.sizeof(buf))
assert rc == 0, rc
t = np.frombuffer(buf, dtype=np.uint32).astype(np.int64).reshape(32, 148, 3)
t -= t[0, :, 0].min()
t %= 1 << 32
for s in range(0, 31, 6):
    a, b, c = t[s, :, 0], t[s, :, 1], t[s, :, 2]
    nxt = t[s + 1, :, 0]
    print(f"sweep {100 + s}: x-arrival spread {a.max() - a.min():5d} ns | compute (t1-t0) "
          f"p50 {np.median(b - a):5.0f} max {np.max(b - a):5d} | tail (t2-t1) p50 {np.median(c - b):5.0f} "
          f"max {np.max(c - b):5d} | last publish -> next arrival p50 {np.median(nxt - c.max()):5.0f} "
          f"| sweep period {np.median(nxt - a):5.0f}")
per = (t[31, :, 0] - t[0, :, 0]) / 31
print(f"mean sweep period {per.mean():.0f} ns")
