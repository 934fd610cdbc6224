"""GPU executor parity: the B200 path reproduces the reference executor.

* golden streams recorded from the real reference: every response (status,
  message, IoStats, per-invocation virtual times, total virtual time), the
  cache state after every request, the removal sequence, and every store
  write (NaN-canonical bytes) must be identical;
* fresh streams from tests/fuzzgen.py (incl. cgemm / jacobi_sweep) against
  the CPU oracle: decisions bit-exact, data bit-exact for builtins and within
  the north-star tolerances for cgemm (rel. Frobenius <= 1e-4) and
  jacobi_sweep (max abs <= 1e-5).
"""

import numpy as np
import pytest

from fuzzgen import make_stream
from helpers import cache_digest, canon, load_golden, replay
from oracle.executor import DictStore, OracleExecutor
from paper_2212_08146_b200.api import response_to_doc
from paper_2212_08146_b200.gpu_executor import ExecutorConfig, GpuExecutor
from paper_2212_08146_b200.hoststore import MemoryStore, PinnedStore

pytestmark = pytest.mark.gpu

STREAMS = ["executor_fuzz31337.json.gz", "executor_fuzz77.json.gz",
           "executor_tight.json.gz", "executor_fuzzfa22.json.gz"]


def gpu_factory(capacity, store_cls, debug=True):
    made = []

    def make(initial):
        store = store_cls()
        for k, v in initial.items():
            store.put(k, v)
        ex = GpuExecutor(ExecutorConfig(capacity=capacity, debug=debug), store)
        removed = []
        orig = ex.cache.remove

        def spy(key):
            removed.append(key)
            return orig(key)

        ex.cache.remove = spy
        made.append(ex)
        snap = lambda: [(k, *v) for k, v in ex.cache.snapshot().items()]  # noqa: E731
        return ex, store, snap, removed
    return make, made


@pytest.mark.parametrize("store_cls", [PinnedStore, MemoryStore])
@pytest.mark.parametrize("name", STREAMS)
def test_gpu_replays_reference_stream(cuda, name, store_cls):
    stream = load_golden(name)
    make, made = gpu_factory(stream["capacity"], store_cls)
    n = 0
    for i, step, resp, digest, removed, writes in replay(stream, make):
        assert resp == step["response"], f"step {i}: {resp} != {step['response']}"
        assert digest == step["cache"], f"step {i} cache"
        assert removed == step["removed"], f"step {i} removals"
        assert writes == step["writes"], f"step {i} store writes"
        ex = made[0]
        assert ex.cache.ephemeral_bytes == 0
        assert all(b.pinned == 0 and not b.dirty for b in ex.cache.entries.values())
        n += 1
    assert n == len(stream["steps"])
    ex = made[0]
    final = sorted([k, b.size, b.last_use] for k, b in ex.cache.entries.items())
    assert final == stream["final_cache"]
    ex.close()


def _compare_key(key, got, want):
    if key.startswith("c/"):
        g = np.frombuffer(bytes(got), "<c8").astype(np.complex128)
        w = np.frombuffer(bytes(want), "<c8").astype(np.complex128)
        den = np.linalg.norm(w)
        err = np.linalg.norm(g - w) / den if den else np.linalg.norm(g - w)
        assert err <= 1e-4, f"{key}: rel. Frobenius {err:.3e}"
    elif key.startswith("j/"):
        g = np.frombuffer(bytes(got), "<f4").astype(np.float64)
        w = np.frombuffer(bytes(want), "<f4").astype(np.float64)
        if g.size == 1:  # residual: relative tolerance
            assert abs(g[0] - w[0]) <= 1e-5 * max(1.0, abs(w[0])), key
        else:
            assert np.abs(g - w).max() <= 1e-5, f"{key}: {np.abs(g - w).max():.3e}"
    else:
        assert canon(got) == canon(want), key


@pytest.mark.parametrize("seed", [1, 2, 3])
def test_gpu_matches_oracle_on_fresh_streams(cuda, seed):
    gstore, ostore = PinnedStore(), DictStore()
    reqs = make_stream(seed, 250, gstore)
    make_stream(seed, 250, ostore)  # same seed: identical store contents + requests
    cap = 2 << 20
    gex = GpuExecutor(ExecutorConfig(capacity=cap, debug=True), gstore)
    oex = OracleExecutor(cap, ostore)
    kinds = set()
    for req in reqs:
        g = gex.execute(req)
        o = oex.execute(req)
        assert response_to_doc(g) == response_to_doc(o), req.request_id
        assert cache_digest((k, *v) for k, v in gex.cache.snapshot().items()) == \
            cache_digest((k, *v) for k, v in oex.snapshot().items())
        if not g.status.ok:
            kinds.add(g.status.error_kind)
    assert gstore.keys() == ostore.keys()
    for k in ostore.keys():
        _compare_key(k, gstore.get(k), ostore.get(k))
    assert {"NotFound", "BackendFault", "UnknownKernel", "ArityMismatch"} <= kinds
    gex.close()


@pytest.mark.parametrize("depth", [2, 4])
def test_pipelined_begin_complete_matches_sequential(cuda, depth):
    """Overlapping requests (begin several, complete later) must give the
    sequential reference's responses, cache states and store bytes --
    including a request that reads (non-const) the key its predecessor is
    still writing back (read-your-writes), and evictions of buffers an
    in-flight request is still flushing (tight capacity)."""
    from paper_2212_08146_b200 import workloads as W
    from paper_2212_08146_b200.api import BufferArg, KaasRequest, KernelInvocation, LaunchDims, f32, i32
    gstore, ostore = PinnedStore(), DictStore()
    reqs = make_stream(7, 120, gstore)
    make_stream(7, 120, ostore)
    # read-after-write chain, back to back: r_i writes key k_i; r_{i+1} reads
    # k_i (non-const) while r_i may still be writing it back
    chain = []
    for i in range(12):
        n = 256 + 64 * i
        bufs = [BufferArg("o", 4 * 4096, "output", key=f"f/raw{i}")]
        invs = [KernelInvocation("fill", LaunchDims(grid_x=4096), (i32(4096), f32(0.5 + i)), ("o",))]
        if i:
            bufs.insert(0, BufferArg("x", 4 * 4096, "input", key=f"f/raw{i - 1}"))
            invs.append(KernelInvocation("vector_add", LaunchDims(grid_x=n), (i32(4096),), ("x", "o", "o")))
        chain.append(KaasRequest(f"raw/{i}", tuple(bufs), tuple(invs)))
    reqs[20:20] = chain
    W.seed_jacobi(gstore, 512, prefix="pj")
    W.seed_jacobi(ostore, 512, prefix="pj")
    for i in range(6):
        reqs.insert(15 * i + 5, W.jacobi_request(f"pj/{i}", 512, 9, "pj/A/512", "pj/b/512",
                                                 "pj/x0/512", f"j/pj{i % 2}", "j/pjr"))
    cap = 3 << 20
    gex = GpuExecutor(ExecutorConfig(capacity=cap, debug=True), gstore)
    oex = OracleExecutor(cap, ostore)
    got = {}
    gex.on_complete = lambda rec, resp: got.__setitem__(rec.req.request_id, resp)
    want = {}
    for req in reqs:
        want[req.request_id] = oex.execute(req)
        rec = gex.begin(req)
        if isinstance(rec, type(want[req.request_id])):
            got[req.request_id] = rec
        assert cache_digest((k, *v) for k, v in gex.cache.snapshot().items()) == \
            cache_digest((k, *v) for k, v in oex.snapshot().items()), req.request_id
        while gex.inflight > depth:
            gex.complete(through=next(iter(gex._inflight)))
    gex.complete()
    assert set(got) == set(want)
    for rid, resp in want.items():
        assert response_to_doc(got[rid]) == response_to_doc(resp), rid
    assert gstore.keys() == ostore.keys()
    for k in ostore.keys():
        _compare_key(k, gstore.get(k), ostore.get(k))
    gex.close()


def test_peer_fills_preserve_decisions_and_bytes(cuda):
    """Two executors sharing a PeerDirectory: on two GPUs when the box has
    them (cudaMemcpyPeerAsync over NVLink between pool allocations, peer
    access granted per pool), else on one (the same path as a D2D copy).  Fills of objects the other executor
    holds at the current store version are device-to-device copies; every
    response, cache state and store byte still equals the reference
    (two oracle executors over one store, same interleaving)."""
    from paper_2212_08146_b200.api import BufferArg, KaasRequest, KernelInvocation, LaunchDims, f32, i32
    from paper_2212_08146_b200.peers import PeerDirectory
    gstore, ostore = PinnedStore(), DictStore()
    reqs = make_stream(11, 160, gstore)
    make_stream(11, 160, ostore)
    n = 4096
    # versioned hand-offs: a output written on one executor, read (non-const) on the other
    for i in range(6):
        w = KaasRequest(f"w/{i}", (BufferArg("o", 4 * n, "output", key="f/shared"),),
                        (KernelInvocation("fill", LaunchDims(grid_x=n), (i32(n), f32(1.0 + i)), ("o",)),))
        r = KaasRequest(f"r/{i}", (BufferArg("x", 4 * n, "input", key="f/shared"),
                                   BufferArg("y", 4 * n, "output", key=f"f/copy{i}")),
                        (KernelInvocation("vector_add", LaunchDims(grid_x=n), (i32(n),), ("x", "x", "y")),))
        reqs[20 * i:20 * i] = [w, r]
    cap = 4 << 20
    peers = PeerDirectory()
    from paper_2212_08146_b200 import native
    ndev = native.device_count()
    devs = (0, 1 % ndev)  # the second executor on a second GPU when there is one: NVLink P2P
    if devs[1] != devs[0]:
        native.init_device(devs[1])
        assert native.enable_peer(devs[0], devs[1]) and native.enable_peer(devs[1], devs[0])
    gexs = [GpuExecutor(ExecutorConfig(capacity=cap, executor_id=e, debug=True, device=devs[e]), gstore)
            for e in (0, 1)]
    for g in gexs:
        g.peers = peers
    oexs = [OracleExecutor(cap, ostore) for _ in (0, 1)]
    for j, req in enumerate(reqs):
        e = j % 2
        g, o = gexs[e].execute(req), oexs[e].execute(req)
        assert response_to_doc(g) == response_to_doc(o), req.request_id
        assert cache_digest((k, *v) for k, v in gexs[e].cache.snapshot().items()) == \
            cache_digest((k, *v) for k, v in oexs[e].snapshot().items())
    assert gstore.keys() == ostore.keys()
    for k in ostore.keys():
        _compare_key(k, gstore.get(k), ostore.get(k))
    assert sum(g.dev_stats.p2p_bytes for g in gexs) > 0 and peers.lends > 0
    for g in gexs:
        g.close()


# -- the reference's direct resolve_buffer API (pkg/tests/test_executor.py:63-107)


def _direct_executor(capacity=1 << 20):
    store = PinnedStore()
    return GpuExecutor(ExecutorConfig(capacity=capacity), store), store


def test_resolve_buffer_called_directly(cuda):
    """TestResolveBuffer (test_executor.py:63-107) against the GPU executor:
    resolve_buffer works outside execute() -- zero-filled ephemerals, NotFound,
    const hits, SizeMismatch, non-const refetch -- and the bytes are final
    when it returns."""
    from paper_2212_08146_b200.api import BufferArg
    from paper_2212_08146_b200.faults import NotFoundError, SizeMismatchError
    from paper_2212_08146_b200.gpu_executor import _ReqStats

    ex, store = _direct_executor()
    try:
        buf = ex.resolve_buffer(BufferArg("tmp", 32, "inout", is_ephemeral=True))
        assert buf.key is None and buf.pinned == 1
        assert buf.snapshot() == b"\x00" * 32
        ex.cache.free_ephemeral(buf)
        with pytest.raises(NotFoundError):
            ex.resolve_buffer(BufferArg("x", 8, "input", key="absent"))
        store.put("w", bytes(range(64)))
        arg = BufferArg("w", 64, "input", key="w", is_const=True)
        first = _ReqStats()
        b1 = ex.resolve_buffer(arg, first)
        ex.cache.unpin(b1)
        assert first.store_gets == 1 and b1.snapshot() == bytes(range(64))
        second = _ReqStats()
        b2 = ex.resolve_buffer(arg, second)
        assert b2 is b1 and second.store_gets == 0 and second.cache_hits == 1
        ex.cache.unpin(b2)
        store.put("w60", bytes(60))
        with pytest.raises(SizeMismatchError):
            ex.resolve_buffer(BufferArg("w60", 64, "input", key="w60", is_const=True))
        store.put("k", b"\x01" * 8)
        karg = BufferArg("x", 8, "inout", key="k")
        b1 = ex.resolve_buffer(karg)
        ex.cache.unpin(b1)
        store.put("k", b"\x02" * 8)
        b2 = ex.resolve_buffer(karg)
        assert b2.snapshot() == b"\x02" * 8
        ex.cache.unpin(b2)
    finally:
        ex.close()


def test_failed_request_leaves_zero_output_not_leftover_memory(cuda):
    """A cgemm output's zero-fill is elided (the kernel overwrites every byte);
    if a later buffer of the same request fails to resolve, the kernel never
    runs and the output entry that stays cached (clean, as in the reference,
    SURVEY App. A.8) must read as zeros -- never as leftover pool memory."""
    from paper_2212_08146_b200.api import (BufferArg, KaasRequest, KernelInvocation,
                                           LaunchDims, i32)
    from paper_2212_08146_b200 import native

    n = 64
    store = PinnedStore()
    ostore = DictStore()
    ex = GpuExecutor(ExecutorConfig(capacity=8 << 20), store)
    oex = OracleExecutor(8 << 20, ostore)
    try:
        rng = np.random.default_rng(3)
        for s_ in (store, ostore):
            s_.put("A", (rng.standard_normal(2 * n * n).astype("<f4")).tobytes())
            s_.put("B", (rng.standard_normal(2 * n * n).astype("<f4")).tobytes())
            s_.put("Z", bytes(8 * n * n))
        # dirty the device pool with non-zero bytes the output may be carved from
        junk = [native.malloc_async(ex.s_exec, 8 * n * n) for _ in range(8)]
        for p in junk:
            native.memset_async(p, 0x7F, 8 * n * n, ex.s_exec)
        for p in junk:
            native.free_async(ex.s_exec, p)
        ex.s_exec.sync()
        bad = KaasRequest("bad", (
            BufferArg("A", 8 * n * n, "input", key="A", is_const=True),
            BufferArg("B", 8 * n * n, "input", key="B", is_const=True),
            BufferArg("C", 8 * n * n, "output", key="C"),
            BufferArg("X", 64, "input", key="missing"),
            BufferArg("R", 4, "output", is_ephemeral=True)), (
            KernelInvocation("cgemm", LaunchDims(grid_x=n * n), (i32(n), i32(n), i32(n)), ("A", "B", "C")),
            KernelInvocation("reduce_sum", LaunchDims(), (i32(16),), ("X", "R"))))
        read = KaasRequest("read", (
            BufferArg("C", 8 * n * n, "input", key="C", is_const=True),
            BufferArg("Z", 8 * n * n, "input", key="Z", is_const=True),
            BufferArg("O", 8 * n * n, "output", key="O")), (
            KernelInvocation("vector_add", LaunchDims(grid_x=2 * n * n), (i32(2 * n * n),), ("C", "Z", "O")),))
        for req in (bad, read):
            g, o = ex.execute(req), oex.execute(req)
            assert response_to_doc(g) == response_to_doc(o), req.request_id
        assert not ex.execute(bad).status.ok
        assert bytes(store.get("O")) == bytes(8 * n * n)
        assert ex.execute(read).io_stats.cache_hits == 2
    finally:
        ex.close()


POISON_SCRIPT = r"""
import sys
sys.path.insert(0, sys.argv[1])
from paper_2212_08146_b200 import native
from paper_2212_08146_b200 import workloads as W
from paper_2212_08146_b200.hoststore import PinnedStore
from paper_2212_08146_b200.pool import KaasService

store = PinnedStore()
W.seed_jacobi(store, 256, prefix="p")
req = lambda i: W.jacobi_request(f"p{i}", 256, 4, "p/A/256", "p/b/256", "p/x0/256", "p/x", "p/r")
with KaasService(store, n_executors=2, capacity=64 << 20, policy="rr", devices=[0]) as svc:
    assert svc.submit(req(0)).status.ok
    ex0 = svc.executors[0]
    native.inject_fault(ex0.s_exec)       # a trapping kernel: a sticky device fault
    r = svc.submit(req(1))                # routed to executor 1 (rr): same context -> fails
    outs = [svc.submit(req(i)) for i in range(2, 6)]
    assert all(not o.status.ok and o.status.error_kind == "Internal" for o in outs), outs
    assert all(e.poisoned for e in svc.executors), [e.poisoned for e in svc.executors]
    assert svc.router.down == {0, 1}
print("POISON-OK")
"""


def test_device_fault_poisons_executor_and_router_routes_away(cuda, tmp_path):
    """SURVEY §5 failure row: a sticky CUDA fault (fault injection: a kernel
    that traps) marks the executor poisoned; every later request on it is
    answered Internal in band without touching the device, and the router
    stops placing requests there.  Runs in a subprocess -- the fault kills
    that process's CUDA context."""
    import os
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    script = tmp_path / "poison.py"
    script.write_text(POISON_SCRIPT)
    out = subprocess.run([sys.executable, str(script), root], capture_output=True, text=True,
                         timeout=300)
    assert "POISON-OK" in out.stdout, out.stdout + out.stderr
