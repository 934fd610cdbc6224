"""The CPU oracle is pinned against the real reference's outputs.

Golden fixtures (tests/golden/*.json.gz) were produced by running the
reference package itself (tests/golden/make_golden.py).  These tests need no
GPU and no reference checkout.
"""

import math

import numpy as np
import pytest

from helpers import load_golden, replay, canon
from oracle.executor import DictStore, OracleExecutor
from oracle.kernels import KERNELS, OracleFault, k_cgemm, k_jacobi_sweep
from oracle.router import OracleRouter
from paper_2212_08146_b200.api import LaunchDims, ScalarLiteral, i32

STREAMS = ["executor_fuzz31337.json.gz", "executor_fuzz77.json.gz",
           "executor_tight.json.gz", "executor_fuzzfa22.json.gz"]


def _oracle_factory(capacity):
    def make(initial):
        store = DictStore(initial)
        ex = OracleExecutor(capacity, store)
        return ex, store, lambda: [(k, v[0], v[1], v[2], v[3]) for k, v in ex.snapshot().items()], ex.removed
    return make


@pytest.mark.parametrize("name", STREAMS)
def test_oracle_replays_reference_stream(name):
    stream = load_golden(name)
    n = 0
    for i, step, resp, digest, removed, writes in replay(stream, _oracle_factory(stream["capacity"])):
        assert resp == step["response"], f"step {i}"
        assert digest == step["cache"], f"step {i} cache"
        assert removed == step["removed"], f"step {i} removals"
        assert writes == step["writes"], f"step {i} store writes"
        n += 1
    assert n == len(stream["steps"])


def test_golden_streams_cover_every_error_kind():
    kinds = set()
    for name in STREAMS:
        for step in load_golden(name)["steps"]:
            r = step["response"]
            if r["status"] == "error":
                kinds.add(r["error"]["kind"])
    assert {"NotFound", "SizeMismatch", "OutOfDeviceMemory", "UnknownKernel",
            "ArityMismatch", "BackendFault", "InvalidRequest"} <= kinds


def _lit(t, v):
    return ScalarLiteral(t, v)


def test_oracle_kernels_match_reference_backend():
    for case in load_golden("kernels.json.gz")["cases"]:
        dims = LaunchDims(*case["dims"])
        lits = tuple(_lit(t, v) for t, v in case["literals"])
        ins = [np.frombuffer(bytes.fromhex(h), dtype=np.uint8).copy() for h in case["inputs"]]
        if case["out_init"] is not None:
            out = np.frombuffer(bytes.fromhex(case["out_init"]), dtype=np.uint8).copy()
        else:
            out = np.zeros(4 * case["out_cells"], dtype=np.uint8)
        with np.errstate(all="ignore"):
            KERNELS[case["kernel"]][3](dims, lits, ins + [out])
        assert out.tobytes() == bytes.fromhex(case["expect"]), case["kernel"]


def test_reference_known_answers():
    """pkg/tests/test_backend.py:41-95 known answers, restated."""
    f32 = np.float32
    out = np.zeros(3, f32)
    KERNELS["vector_add"][3](LaunchDims(block_x=4), (i32(3),),
                             [np.array([1, 2, 3], f32).view(np.uint8), np.array([4, 5, 6], f32).view(np.uint8),
                              out.view(np.uint8)])
    assert out.tolist() == [5.0, 7.0, 9.0]
    out = np.full(4, -1.0, f32)
    KERNELS["vector_add"][3](LaunchDims(grid_x=2), (i32(4),),
                             [np.array([1, 2, 3, 4], f32).view(np.uint8),
                              np.array([10, 20, 30, 40], f32).view(np.uint8), out.view(np.uint8)])
    assert out.tolist() == [11.0, 22.0, -1.0, -1.0]
    out = np.zeros(1, f32)
    KERNELS["reduce_sum"][3](LaunchDims(), (i32(1000),), [np.ones(1000, f32).view(np.uint8), out.view(np.uint8)])
    assert out[0] == 1000.0
    out = np.full(1, 9.0, f32)
    KERNELS["reduce_sum"][3](LaunchDims(), (i32(0),), [np.zeros(0, np.uint8), out.view(np.uint8)])
    assert out[0] == 0.0
    with pytest.raises(OracleFault):
        KERNELS["fill"][3](LaunchDims(), (i32(-3), _lit("f32", 0.0)), [np.zeros(4, np.uint8)])
    with pytest.raises(OracleFault):
        KERNELS["vector_add"][3](LaunchDims(grid_x=4), (i32(4),),
                                 [np.zeros(16, np.uint8), np.zeros(16, np.uint8), np.zeros(8, np.uint8)])


def test_oracle_cgemm_known_answers():
    rng = np.random.default_rng(1)
    n, m, k = 5, 7, 3
    A = (rng.standard_normal((n, k)) + 1j * rng.standard_normal((n, k))).astype(np.complex64)
    eye = np.eye(k, m, dtype=np.complex64)
    out = np.zeros(n * m, np.complex64)
    k_cgemm(LaunchDims(grid_x=n * m), (i32(n), i32(m), i32(k)),
            [A.view(np.uint8).ravel(), eye.view(np.uint8).ravel(), out.view(np.uint8)])
    expect = np.zeros((n, m), np.complex64)
    expect[:, :k] = A
    assert np.array_equal(out.reshape(n, m), expect)
    # (1+2i)(3-i) = 5+5i; coverage: only the first cell written
    a = np.array([1 + 2j, 0], np.complex64)
    b = np.array([3 - 1j, 0], np.complex64)
    out = np.full(4, 9 + 9j, np.complex64)
    k_cgemm(LaunchDims(), (i32(2), i32(2), i32(1)), [a.view(np.uint8), b.view(np.uint8), out.view(np.uint8)])
    assert out[0] == 5 + 5j and np.all(out[1:] == 9 + 9j)
    with pytest.raises(OracleFault):
        k_cgemm(LaunchDims(), (i32(2), i32(2), i32(2)), [a.view(np.uint8), b.view(np.uint8), out.view(np.uint8)])


def test_oracle_jacobi_converges_and_defines_residual():
    n = 64
    rng = np.random.default_rng(2)
    A = rng.random((n, n)).astype(np.float32)
    A[np.arange(n), np.arange(n)] = A.sum(1) + 1
    xt = rng.standard_normal(n)
    b = (A.astype(np.float64) @ xt).astype(np.float32)
    x = np.zeros(n, np.float32)
    nxt = np.zeros(n, np.float32)
    r = np.zeros(1, np.float32)
    for _ in range(200):
        k_jacobi_sweep(LaunchDims(grid_x=n), (i32(n),),
                       [A.view(np.uint8).ravel(), b.view(np.uint8), x.view(np.uint8), nxt.view(np.uint8),
                        r.view(np.uint8)])
        x, nxt = nxt.copy(), x
    assert np.abs(x - xt).max() < 1e-4
    assert r[0] < 1e-3
    # partial coverage leaves rows >= cov untouched
    out = np.full(n, 7.0, np.float32)
    k_jacobi_sweep(LaunchDims(grid_x=10), (i32(n),),
                   [A.view(np.uint8).ravel(), b.view(np.uint8), x.view(np.uint8), out.view(np.uint8),
                    r.view(np.uint8)])
    assert np.all(out[10:] == 7.0) and not np.any(out[:10] == 7.0)


def test_oracle_router_matches_reference_placements():
    routing = load_golden("routing.json.gz")
    from helpers import load_golden as _lg  # noqa: F401
    import random as _r  # noqa: F401
    reqs = _zipf_requests()
    for policy in ("random:1", "rr", "affinity:8", "affinity:1"):
        router = OracleRouter([0, 1, 2, 3], policy)
        seq = []
        for r in reqs:
            e = router.route(r)
            seq.append(e)
            router.complete(e, True, r)
        assert seq == routing[f"zipf_{policy}"], policy


def _zipf_requests():
    """Rebuild the reference's zipf_const stream (kaas/bench.py:77-180,
    seed 42, 2000 requests) with the product's workload builder."""
    from paper_2212_08146_b200.workloads import WorkloadSpec, build_requests
    return build_requests(WorkloadSpec("zipf_const", 2000, zipf_s=1.0, key_universe=100, seed=42))


def test_canon_only_touches_nan_words():
    words = np.array([0x7FC00001, 0xFFC00000, 0x7F800000, 0x3F800000, 0x7F800001], dtype="<u4")
    out = np.frombuffer(canon(words.tobytes()), dtype="<u4")
    assert out.tolist() == [0x7FC00000, 0x7FC00000, 0x7F800000, 0x3F800000, 0x7FC00000]
    assert math.isnan(np.frombuffer(canon(words.tobytes()), "<f4")[0])
