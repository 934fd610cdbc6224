"""Invocation runs (csrc/runs.cu): consecutive builtin invocations of a
request execute as one persistent cooperative launch with dependency
counters.  Results must be exactly what one launch per invocation in request
order gives -- the reference's sequential model (backend.py:258-266,
executor.py:356-369) -- so every case here is compared bit-exactly
(NaN-canonical) with the CPU oracle, together with the response.

The random requests mix every builtin over shared buffers: read-after-write
chains, write-after-read reuse, exact aliasing (matmul(c, c, c) goes through a
temporary; elementwise ops in place), partial coverage, long and ragged
shapes, const weights (prepared transposed B: filled on the first request,
reused on the repeat), and matmuls the run kernel cannot take (k % 4 != 0),
which split a run in two.
"""

import random

import numpy as np
import pytest

from helpers import canon
from oracle.executor import DictStore, OracleExecutor
from paper_2212_08146_b200.api import BufferArg, KaasRequest, KernelInvocation, LaunchDims, f32, i32
from paper_2212_08146_b200.gpu_executor import ExecutorConfig, GpuExecutor
from paper_2212_08146_b200.hoststore import PinnedStore

pytestmark = pytest.mark.gpu

S = 64 * 1024  # floats per working buffer


def _grid(cells, rng):
    cells = max(1, cells)
    r = rng.random()
    if r < 0.2:  # partial coverage
        return LaunchDims(grid_x=max(1, cells - rng.randint(0, cells - 1)))
    return LaunchDims(grid_x=cells + rng.randint(0, 5))


def _seed(stores, rng, nprng, tag):
    keys = {}
    for i in range(3):
        d = (nprng.standard_normal(S) * 4).astype("<f4")
        if rng.random() < 0.3:
            d[rng.randrange(S)] = rng.choice((np.inf, -np.inf, np.nan, -0.0))
        keys[f"in{i}"] = f"runs/{tag}/in{i}"
        for st in stores:
            st.put(keys[f"in{i}"], d.tobytes())
    for i in range(2):
        n = rng.choice((256, 1024, 4096, S))
        d = (nprng.standard_normal(n) * 0.5).astype("<f4")
        keys[f"w{i}"] = f"runs/{tag}/w{i}"
        for st in stores:
            st.put(keys[f"w{i}"], d.tobytes())
    return keys


def _request(rng, keys, tag, wsizes):
    bufs = [BufferArg("in0", 4 * S, "input", key=keys["in0"]),
            BufferArg("in1", 4 * S, "input", key=keys["in1"], is_const=True),
            BufferArg("in2", 4 * S, "inout", key=keys["in2"])]
    bufs += [BufferArg(f"w{i}", 4 * wsizes[i], "input", key=keys[f"w{i}"], is_const=True) for i in range(2)]
    bufs += [BufferArg(f"e{i}", 4 * S, "inout", is_ephemeral=True) for i in range(3)]
    bufs += [BufferArg(f"o{i}", 4 * S, "output", key=f"runs/{tag}/o{i}") for i in range(2)]
    readable = ["in0", "in1", "in2", "e0", "e1", "e2", "o0", "o1"]
    writable = ["in2", "e0", "e1", "e2", "o0", "o1"]
    invs = []
    for _ in range(rng.randint(2, 12)):
        kind = rng.choice(("vadd", "saxpy", "fill", "reduce", "mm", "mm", "mm", "mm_alias", "mm_w"))
        if kind in ("vadd", "saxpy"):
            n = rng.choice((1, 3, 4, 1000, 8192, 8193, S))
            x, y = rng.choice(readable), rng.choice(readable)
            o = rng.choice(writable + [x] if x in writable else writable)
            lits = (i32(n),) if kind == "vadd" else (i32(n), f32(rng.uniform(-2, 2)))
            invs.append(KernelInvocation("vector_add" if kind == "vadd" else "saxpy", _grid(n, rng), lits,
                                         (x, y, o)))
        elif kind == "fill":
            n = rng.choice((1, 5, 4096, 20000, S))
            invs.append(KernelInvocation("fill", _grid(n, rng), (i32(n), f32(rng.uniform(-3, 3))),
                                         (rng.choice(writable),)))
        elif kind == "reduce":
            n = rng.choice((0, 1, 17, 4096, S))
            invs.append(KernelInvocation("reduce_sum", LaunchDims(), (i32(n),),
                                         (rng.choice(readable), rng.choice(writable))))
        else:
            if kind == "mm_w":  # const weight as B: prepared transposed copy
                wi = rng.randrange(2)
                k = rng.choice([d for d in (4, 8, 16, 64, 256) if wsizes[wi] % d == 0])
                m = wsizes[wi] // k
                m = min(m, S // k)
                n = rng.choice((1, 7, 49, 64, 100))
                n = max(1, min(n, S // max(k, m)))
                b = f"w{wi}"
            else:
                k = rng.choice((4, 8, 12, 64, 68, 256, 3, 5))  # 3, 5: not a run matmul
                m = rng.choice((1, 4, 16, 33, 64, 200, 256))
                n = rng.choice((1, 2, 49, 64, 65, 256))
                while n * k > S or k * m > S or n * m > S:
                    n = max(1, n // 2)
                    m = max(1, m // 2)
                b = rng.choice(readable)
            a = rng.choice(readable)
            o = a if kind == "mm_alias" else rng.choice(writable)
            if kind == "mm_alias":
                if a not in writable:
                    a = o = rng.choice(writable)
                b = rng.choice((a, b))
            invs.append(KernelInvocation("matmul", _grid(n * m, rng), (i32(n), i32(m), i32(k)), (a, b, o)))
    return KaasRequest(f"runs-{tag}", tuple(bufs), tuple(invs))


@pytest.fixture(scope="module")
def pair(cuda):
    store, ostore = PinnedStore(), DictStore()
    ex = GpuExecutor(ExecutorConfig(capacity=1 << 30), store)
    oex = OracleExecutor(1 << 30, ostore)
    yield ex, store, oex, ostore
    ex.close()


@pytest.mark.parametrize("seed", range(24))
def test_random_runs_bit_exact(pair, seed):
    ex, store, oex, ostore = pair
    rng = random.Random(1000 + seed)
    nprng = np.random.default_rng(1000 + seed)
    tag = f"s{seed}"
    keys = _seed((store, ostore), rng, nprng, tag)
    wsizes = [len(ostore.get(keys["w0"])) // 4, len(ostore.get(keys["w1"])) // 4]
    req = _request(rng, keys, tag, wsizes)
    for rep in range(2):  # the repeat runs on cache hits and prepared weights
        g, o = ex.execute(req), oex.execute(req)
        assert g == o, (rep, g.status, o.status)
        for k in ostore.keys():
            if k.startswith(f"runs/{tag}/"):
                assert canon(store.get(k)) == canon(ostore.get(k)), (rep, k, req.invocations)


def test_run_of_many_invocations_splits_across_launches(pair):
    """More tasks than one launch holds (128): the run continues in a second
    launch, still in order."""
    ex, store, oex, ostore = pair
    for st in (store, ostore):
        st.put("runs/long/x", np.arange(1024, dtype="<f4").tobytes())
    invs = []
    for i in range(300):
        if i % 3 == 0:
            invs.append(KernelInvocation("saxpy", LaunchDims(grid_x=1024), (i32(1024), f32(1.0001)), ("a", "x", "a")))
        elif i % 3 == 1:
            invs.append(KernelInvocation("vector_add", LaunchDims(grid_x=1000), (i32(1000),), ("a", "a", "b")))
        else:
            invs.append(KernelInvocation("matmul", LaunchDims(grid_x=32 * 32), (i32(32), i32(32), i32(32)),
                                         ("b", "a", "a")))
    req = KaasRequest("runs-long", (BufferArg("x", 4096, "input", key="runs/long/x"),
                                    BufferArg("a", 4096, "inout", is_ephemeral=True),
                                    BufferArg("b", 4096, "output", key="runs/long/b")), tuple(invs))
    g, o = ex.execute(req), oex.execute(req)
    assert g == o
    assert canon(store.get("runs/long/b")) == canon(ostore.get("runs/long/b"))
