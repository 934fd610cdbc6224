"""Dev: Jacobi 500-sweep chain time vs how long the GPU sat idle before the
launch (after an L2-flushing memset), host spin-waits of 0..2000 us."""
import sys
import time

sys.path.insert(0, ".")
sys.path.insert(0, "tools")
import jgap  # noqa: E402  (builds the chain; prints its own table first)
from paper_2212_08146_b200 import native  # noqa: E402


def spin(us):
    t = time.perf_counter() + us * 1e-6
    while time.perf_counter() < t:
        pass


def pre(us):
    native.memset_async(jgap.flush, 0, 256 << 20, jgap.s)
    jgap.s.sync()
    spin(us)


for rnd in range(2):
    for us in (0, 10, 25, 50, 100, 200, 500, 1000, 2000):
        jgap.one(lambda: pre(us))
        v = sorted(jgap.one(lambda: pre(us)) for _ in range(15))
        print(f"round {rnd} idle {us:5d} us: us/sweep p50 {v[7]:.3f} min {v[0]:.3f}  chain p50 {v[7] * 500:.1f} us")
