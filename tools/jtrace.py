"""Dev: per-CTA phase timestamps of the Jacobi column kernel (sweeps 100..131).

    make -C paper_2212_08146_b200/csrc dev   # the trace exists only in the dev build
    python tools/jtrace.py [n]

Stamps (globaltimer, ns), warp 0 of each CTA: poll start, x arrived,
register + shared-memory rows done, TMEM rows + reductions done, rows
published.  Prints per-phase medians and the critical path from the last
publish to the next sweep's x arrival.
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
NW = 32 * 148 * 5 + 148 * 8
buf = (C.c_uint * (NW + 32 * 148 * 8))()
rc = native.load().kaas_dev_jacobi_trace(buf, C.sizeof(buf))
assert rc == 0, rc
raw = np.frombuffer(buf, dtype=np.uint32).astype(np.int64)
t = raw[:32 * 148 * 5].reshape(32, 148, 5)
wa = raw[NW:].reshape(32, 148, 8)
t0 = t[0, :, 1].min()
t -= t0
t %= 1 << 32
wa = (wa - t0) % (1 << 32)
# stamps (warp 0 of each CTA): 0 poll start, 1 x arrived, 2 register+smem rows
# done, 3 TMEM rows + reductions done, 4 published
rows = []
for s in range(0, 31):
    p0, xa, mid, cd, pub = (t[s, :, i] for i in range(5))
    nxt = t[s + 1, :, 1]
    rows.append((np.median(xa - p0), np.median(mid - xa), np.median(cd - mid), np.median(pub - cd),
                 np.median(nxt - pub.max()), pub.max() - pub.min(), xa.max() - xa.min(),
                 np.median(nxt - xa)))
r = np.array(rows)
names = ["wait for x (poll)", "reg+smem rows", "TMEM rows+reduce", "CTA reduce+publish",
         "last publish->next arrival", "publish spread", "arrival spread", "sweep period"]
for i, nm in enumerate(names):
    print(f"{nm:28s} median over sweeps {np.median(r[:, i]):7.0f} ns   (min {r[:, i].min():6.0f}, max {r[:, i].max():6.0f})")
per = (t[31, :, 1] - t[0, :, 1]) / 31
print(f"mean sweep period {per.mean():.0f} ns")

# per-warp x arrival relative to the CTA's last publish of the previous sweep
lag = []
for s in range(1, 31):
    pub_prev = t[s - 1, :, 4]  # warp 0's publish, per CTA
    for w in range(8):
        lag.append((w, np.median(wa[s, :, w] - pub_prev)))
lag = np.array(lag)
for w in range(8):
    print(f"warp {w}: x arrives {np.median(lag[lag[:, 0] == w, 1]):6.0f} ns after its CTA's previous publish")
last = np.argmax(wa[1:31], axis=2).ravel()
print("last warp to get its x (share of CTA-sweeps):", np.bincount(last, minlength=8) / last.size)
