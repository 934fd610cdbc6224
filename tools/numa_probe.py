"""Dev: pinned H2D bandwidth vs the NUMA node of the host pages (first touch
by a thread bound to that node's cores)."""
import os
import statistics
import subprocess
import sys

sys.path.insert(0, ".")
from paper_2212_08146_b200 import native  # noqa: E402
from paper_2212_08146_b200.hoststore import PinnedBlob  # noqa: E402

print(subprocess.run(["nvidia-smi", "topo", "-m"], capture_output=True, text=True).stdout)
print(subprocess.run(["lscpu"], capture_output=True, text=True).stdout[-900:])
nodes = {}
base = "/sys/devices/system/node"
for d in sorted(os.listdir(base)):
    if d.startswith("node"):
        with open(f"{base}/{d}/cpulist") as fh:
            nodes[d] = fh.read().strip()
print("nodes", nodes)


def parse(cpulist):
    out = []
    for part in cpulist.split(","):
        if "-" in part:
            a, b = part.split("-")
            out += range(int(a), int(b) + 1)
        elif part:
            out.append(int(part))
    return out


native.init_device(0)
s = native.Stream(0)
d = native.malloc_async(s, 256 << 20)
allowed = os.sched_getaffinity(0)
for name, cl in nodes.items():
    cpus = set(parse(cl)) & allowed
    if not cpus:
        continue
    os.sched_setaffinity(0, cpus)
    blob = PinnedBlob(256 << 20)
    C = __import__("ctypes")
    C.memset(blob.addr, 1, 256 << 20)  # first touch on this node
    e0, e1 = native.Event(0, True), native.Event(0, True)
    v = []
    for _ in range(5):
        e0.record(s)
        native.h2d_async(d, blob.addr, 256 << 20, s)
        e1.record(s)
        e1.sync()
        v.append((256 << 20) / (e0.elapsed_ms(e1) * 1e6))
    w = []
    for _ in range(5):
        e0.record(s)
        native.d2h_async(blob.addr, d, 256 << 20, s)
        e1.record(s)
        e1.sync()
        w.append((256 << 20) / (e0.elapsed_ms(e1) * 1e6))
    print(f"{name} ({len(cpus)} cpus): H2D {statistics.median(v):.1f} GB/s  D2H {statistics.median(w):.1f} GB/s")
os.sched_setaffinity(0, allowed)
