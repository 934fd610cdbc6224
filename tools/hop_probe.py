"""Dev: latency of the small copies around a Jacobi request (one B200).

Device-timed (events), medians of 50:
  a) 16 KiB H2D alone
  b) 16 KiB H2D on s_in, event, s_exec waits, 4-byte memset on s_exec
  c) the same H2D + memset both on s_exec
  d) 4-byte memset on s_exec, event, s_out waits, 16 KiB D2H on s_out
  e) memset + D2H both on s_exec

    python tools/hop_probe.py
"""
import statistics
import sys

sys.path.insert(0, ".")
from paper_2212_08146_b200 import native  # noqa: E402

native.init_device(0)
s_in, s_exec, s_out = native.Stream(0), native.Stream(0), native.Stream(0)
host = native.host_alloc(16384)
dev = native.malloc_async(s_exec, 16384)
flag = native.malloc_async(s_exec, 256)
s_exec.sync()


def timed(fn, start_stream, end_stream, reps=50):
    ts = []
    for _ in range(reps):
        e0, e1 = native.Event(0, True), native.Event(0, True)
        e0.record(start_stream)
        fn()
        e1.record(end_stream)
        e1.sync()
        ts.append(e0.elapsed_ms(e1) * 1e3)
    return statistics.median(ts[5:])


def a():
    native.h2d_async(dev, host, 16384, s_in)


def b():
    native.h2d_async(dev, host, 16384, s_in)
    ev = native.Event(0).record(s_in)
    s_exec.wait(ev)
    native.memset_async(flag, 0, 4, s_exec)


def c():
    native.h2d_async(dev, host, 16384, s_exec)
    native.memset_async(flag, 0, 4, s_exec)


def d():
    native.memset_async(flag, 0, 4, s_exec)
    ev = native.Event(0).record(s_exec)
    s_out.wait(ev)
    native.d2h_async(host, dev, 16384, s_out)


def e():
    native.memset_async(flag, 0, 4, s_exec)
    native.d2h_async(host, dev, 16384, s_exec)


print(f"a) H2D 16 KiB alone                 {timed(a, s_in, s_in):7.1f} us")
print(f"b) H2D on s_in -> event -> s_exec   {timed(b, s_in, s_exec):7.1f} us")
print(f"c) H2D + memset on s_exec           {timed(c, s_exec, s_exec):7.1f} us")
print(f"d) s_exec -> event -> D2H on s_out  {timed(d, s_exec, s_out):7.1f} us")
print(f"e) memset + D2H on s_exec           {timed(e, s_exec, s_exec):7.1f} us")
