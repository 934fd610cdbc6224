"""Generate golden fixtures by running the REAL reference implementation.

Run in the build container, where the reference is mounted read-only:

    python tests/golden/make_golden.py [/root/reference]

It imports ``kaas`` from ``<ref>/pkg/src`` and the reference's own test
generators (``genreq``, ``oracles``) from ``<ref>/pkg/tests``, replays the
reference test streams, and writes gzip'd JSON fixtures next to this file.
Nothing here is imported at test time; the GPU box never sees the reference.

Fixture contents (all bytes hex, NaN-canonicalised hashes where noted):
  executor_<name>.json.gz   initial store, request stream (wire JSON),
                            per-request response + cache snapshot digest +
                            eviction victims + store writes
  kernels.json.gz           reference-backend outputs for random builtin cases
  routing.json.gz           placement sequences + bench reports
"""

from __future__ import annotations

import gzip
import hashlib
import json
import os
import random
import sys

import numpy as np

REF = sys.argv[1] if len(sys.argv) > 1 else "/root/reference"
sys.path.insert(0, os.path.join(REF, "pkg", "src"))
sys.path.insert(0, os.path.join(REF, "pkg", "tests"))

from kaas.backend import SimulatedBackend  # noqa: E402
from kaas.bench import WorkloadSpec, build_requests, gen_data, run_bench  # noqa: E402
from kaas.executor import CacheState, Executor, ExecutorConfig  # noqa: E402
from kaas.protocol import LaunchDims, encode_request, encode_response, f32, i32  # noqa: E402
from kaas.router import Router, parse_policy  # noqa: E402
from kaas.store import MemoryStore  # noqa: E402

import genreq  # noqa: E402  (reference test generator)

HERE = os.path.dirname(os.path.abspath(__file__))


def canon_hash(data: bytes) -> str:
    """sha256 of the bytes with every f32-NaN word replaced by 0x7fc00000.

    NaN payloads are not specified by IEEE 754 and numpy's x86 loops pick
    them by element position; parity is bit-exact on everything else."""
    if len(data) % 4 == 0 and data:
        w = np.frombuffer(data, dtype="<u4").copy()
        nan = ((w & 0x7F800000) == 0x7F800000) & ((w & 0x007FFFFF) != 0)
        w[nan] = 0x7FC00000
        data = w.tobytes()
    return hashlib.sha256(data).hexdigest()


def snap_digest(cache: CacheState) -> str:
    items = sorted((k, b.size, b.last_use, b.pinned, b.dirty) for k, b in cache.entries.items())
    return hashlib.sha256(json.dumps(items).encode()).hexdigest()


def dump(name: str, doc) -> None:
    path = os.path.join(HERE, name)
    with gzip.open(path, "wt", encoding="utf-8") as fh:
        json.dump(doc, fh, separators=(",", ":"), sort_keys=True)
    print(f"wrote {path} ({os.path.getsize(path)} bytes)")


def record_stream(name, seed, n_keys, sizes, capacity, n_requests, debug=True):
    rng = random.Random(seed)
    store = MemoryStore()
    pool = []
    for i in range(n_keys):
        size = rng.choice(sizes)
        store.put(f"k{i}", rng.randbytes(size))
        pool.append((f"k{i}", size))
    initial = {k: store.get(k).hex() for k in store.keys()}
    ex = Executor(ExecutorConfig(capacity=capacity, executor_id=0, debug=debug), store,
                  SimulatedBackend())
    victims: list[str] = []
    orig_remove = ex.cache.remove

    def spy_remove(key):
        victims.append(key)
        return orig_remove(key)

    ex.cache.remove = spy_remove
    steps = []
    for i in range(n_requests):
        req, fault = genreq.fuzz_request(rng, pool, i)
        before = dict(store._objects)
        victims.clear()
        resp = ex.execute(req)
        writes = {k: canon_hash(v) for k, v in store._objects.items() if before.get(k) is not v}
        steps.append({
            "request": json.loads(encode_request(req)),
            "fault": fault,
            "response": json.loads(encode_response(resp)),
            "cache": snap_digest(ex.cache),
            "removed": list(victims),
            "writes": writes,
            "tick": ex.cache.tick,
            "used": ex.cache.used_bytes,
        })
    final_cache = sorted([k, b.size, b.last_use] for k, b in ex.cache.entries.items())
    dump(f"executor_{name}.json.gz", {
        "seed": seed, "capacity": capacity, "initial_store": initial, "steps": steps,
        "final_cache": final_cache,
        "final_store": {k: canon_hash(store.get(k)) for k in store.keys()},
        "stats": ex.stats(),
    })


def record_kernels():
    backend = SimulatedBackend()
    rng = random.Random(20240917)
    nprng = np.random.default_rng(20240917)
    cases = []

    def run(kid, dims, lits, inputs, out_cells, out_init=None):
        out = np.zeros(max(1, out_cells), dtype="<f4") if out_init is None else out_init.copy()
        views = [a.copy().view(np.uint8) for a in inputs] + [out.view(np.uint8)]
        backend.launch(kid, dims, lits, views)
        cases.append({
            "kernel": kid, "dims": list(dims.__dict__.values()),
            "literals": [[l.type, l.value] for l in lits],
            "inputs": [a.tobytes().hex() for a in inputs],
            "out_init": (out_init.tobytes().hex() if out_init is not None else None),
            "out_cells": max(1, out_cells),
            "expect": out.tobytes().hex(),
        })

    for _ in range(60):
        n = rng.randint(1, 64)
        x = (nprng.standard_normal(n) * 100).astype("<f4")
        y = (nprng.standard_normal(n) * 100).astype("<f4")
        cov = rng.randint(1, n + 3)
        dims = LaunchDims(grid_x=cov, block_x=1)
        run("vector_add", dims, (i32(n),), [x, y], n)
        a = float(nprng.standard_normal())
        run("saxpy", dims, (i32(n), f32(a)), [x, y], n)
        run("reduce_sum", dims, (i32(n),), [x], 1)
        run("fill", dims, (i32(n), f32(a)), [], n, out_init=np.full(n, -1.0, "<f4"))
    for _ in range(40):
        n, m, k = (rng.randint(1, 40) for _ in range(3))
        a = (nprng.standard_normal(n * k) * 10).astype("<f4")
        b = (nprng.standard_normal(k * m) * 10).astype("<f4")
        cov = rng.randint(1, n * m + 5)
        run("matmul", LaunchDims(grid_x=cov), (i32(n), i32(m), i32(k)), [a, b], n * m)
    # special values: NaN/Inf/-0.0/denormals through every builtin
    specials = np.array([0.0, -0.0, np.inf, -np.inf, np.nan, 1e-45, -1e-45, 3.4e38, -3.4e38,
                         1.0, -1.0, 1e-38], dtype="<f4")
    x = np.resize(specials, 48).astype("<f4")
    y = np.roll(x, 5)
    dims = LaunchDims(grid_x=48)
    run("vector_add", dims, (i32(48),), [x, y], 48)
    run("saxpy", dims, (i32(48), f32(-2.5)), [x, y], 48)
    run("reduce_sum", dims, (i32(48),), [x], 1)
    run("matmul", LaunchDims(grid_x=36), (i32(6), i32(6), i32(8)), [x[:48], y[:48]], 36)
    run("reduce_sum", LaunchDims(), (i32(1),), [np.array([-0.0], "<f4")], 1)
    run("matmul", LaunchDims(grid_x=4), (i32(2), i32(2), i32(0)), [np.zeros(0, "<f4"), np.zeros(0, "<f4")], 4,
        out_init=np.full(4, 7.0, "<f4"))
    dump("kernels.json.gz", {"cases": cases})


def record_routing():
    out = {}
    # placement sequence of the fixed-seed zipf stream, sequential submitter
    spec = WorkloadSpec("zipf_const", 2000, zipf_s=1.0, key_universe=100, seed=42)
    reqs = build_requests(spec)
    for policy in ("random:1", "rr", "affinity:8", "affinity:1"):
        router = Router([0, 1, 2, 3], parse_policy(policy))
        seq = []
        from kaas.protocol import IoStats, KaasResponse, Status
        ok = KaasResponse("r", Status.make_ok(), io_stats=IoStats())
        for r in reqs:
            e = router.route(r)
            seq.append(e)
            router.update_digest(e, ok, r)
        out[f"zipf_{policy}"] = seq
    # full benches (executor + router + service), byte-stable reports
    rep = run_bench(WorkloadSpec("zipf_const", 5000, zipf_s=1.0, key_universe=100, seed=42),
                    ["random:1", "affinity:8"], n_executors=4, capacity=30 * 64 * 1024)
    out["bench_zipf_const"] = rep
    rep2 = run_bench(WorkloadSpec("mixed", 300, seed=7), ["random:3", "rr", "affinity:8"],
                     n_executors=4, warm_repeat=True)
    out["bench_mixed"] = rep2
    rep3 = run_bench(WorkloadSpec("matmul_chain", 6, matrix_dim=16, seed=5), ["rr"],
                     n_executors=2, warm_repeat=True)
    out["bench_matmul_chain"] = rep3
    dump("routing.json.gz", out)


def main():
    record_stream("fuzz31337", 31337, 8, (16, 64, 256, 1024), 1 << 18, 300)
    record_stream("fuzz77", 77, 12, (16, 64, 256, 1024, 4096), 1 << 20, 500)
    record_stream("fuzzfa22", 0xFA22, 12, (16, 64, 256, 1024, 4096, 16384), 1 << 20, 2000)
    # tight capacity: heavy eviction / OOM traffic
    record_stream("tight", 4242, 16, (64, 256, 1024, 4096), 24 * 1024, 600)
    record_kernels()
    record_routing()


if __name__ == "__main__":
    main()
