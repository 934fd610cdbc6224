"""Bench report v1 over the GPU pool (``pkg/src/kaas/bench.py:234-355``).

``run_bench`` drives a fresh ``KaasService`` per policy with the reference's
request streams and aggregates exactly the reference's report fields (hit
rate, store traffic, virtual mean / nearest-rank p95 latency, per-executor
counts, busy fraction, virtual makespan).  Those are pure functions of the
cache and routing decisions, so a GPU run's report is byte-identical to the
reference's for a single submitter.  ``measured`` adds what the reference
cannot report: wall-clock req/s, p50/p99 wall latency and per-GPU device
time / copy volumes (kept outside the v1 fields).
"""

from __future__ import annotations

import json
import math
import statistics
import time
from dataclasses import asdict

from .hoststore import MemoryStore
from .workloads import WorkloadSpec, build_requests, default_capacity, gen_data

REPORT_VERSION = 1


def percentile(values, q: float):
    """Nearest-rank percentile (bench.py:234-237 uses q = 0.95)."""
    ordered = sorted(values)
    if not ordered:
        return 0
    rank = math.ceil(q * len(ordered))
    return ordered[max(0, rank - 1)]


def run_stream(service, requests, clients: int):
    """Submit ``requests``; returns (responses, wall latencies in s)."""
    lat = [0.0] * len(requests)

    def one(i):
        t = time.perf_counter()
        r = service.submit(requests[i])
        lat[i] = time.perf_counter() - t
        return r

    if clients <= 1:
        return [one(i) for i in range(len(requests))], lat
    import concurrent.futures as cf
    with cf.ThreadPoolExecutor(max_workers=clients) as pool:
        return list(pool.map(one, range(len(requests)))), lat


def aggregate(responses, service, compute_ns_total: int) -> dict:
    hits = sum(r.io_stats.cache_hits for r in responses)
    misses = sum(r.io_stats.cache_misses for r in responses)
    lats = [r.simulated_total_time for r in responses]
    makespan = max((e.clock.now_ns for e in service.executors), default=0)
    busy = compute_ns_total / (len(service.executors) * makespan) if makespan else 0.0
    return {
        "requests": len(responses),
        "errors": sum(0 if r.status.ok else 1 for r in responses),
        "hit_rate": hits / (hits + misses) if hits + misses else 0.0,
        "cache_hits": hits,
        "cache_misses": misses,
        "store_gets": sum(r.io_stats.store_gets for r in responses),
        "store_puts": sum(r.io_stats.store_puts for r in responses),
        "mean_latency_ns": statistics.fmean(lats) if lats else 0.0,
        "p95_latency_ns": percentile(lats, 0.95) if lats else 0,
        "per_executor_requests": [e.requests_served for e in service.executors],
        "gpu_busy_fraction": busy,
        "simulated_makespan_ns": makespan,
    }


def run_bench(spec: WorkloadSpec, policies, n_executors: int = 4, capacity: int | None = None,
              timing=None, clients: int = 1, warm_repeat: bool = False, digest_cap: int = 1024,
              service_factory=None, store_factory=MemoryStore, measured: bool = False) -> dict:
    """One fresh service per policy; returns the v1 report (plus ``measured``
    side fields when asked)."""
    problems = spec.validate()
    if problems:
        raise ValueError("; ".join(problems))
    cap = capacity if capacity is not None else default_capacity(spec)
    report = {
        "report_version": REPORT_VERSION, "workload": asdict(spec), "executors": n_executors,
        "capacity": cap, "clients": clients, "warm_repeat": warm_repeat, "over_http": False,
        "policies": {},
    }
    if service_factory is None:
        from .pool import KaasService

        def service_factory(store, policy):
            return KaasService(store, n_executors=n_executors, capacity=cap, policy=policy,
                               timing=timing, digest_cap=digest_cap)
    side = {}
    for policy in policies:
        store = store_factory()
        gen_data(spec, store)
        reqs = build_requests(spec)
        service = service_factory(store, policy)
        try:
            t0 = time.perf_counter()
            responses, lat = run_stream(service, reqs, clients)
            wall = time.perf_counter() - t0
            compute = sum(s.simulated_compute_time for r in responses for s in r.per_invocation)
            entry = aggregate(responses, service, compute)
            if warm_repeat:
                base = [e.requests_served for e in service.executors]
                again, _ = run_stream(service, reqs, clients)
                compute2 = sum(s.simulated_compute_time for r in again for s in r.per_invocation)
                entry["repeat"] = aggregate(again, service, compute + compute2)
                entry["repeat"]["per_executor_requests"] = [
                    e.requests_served - b for e, b in zip(service.executors, base)]
                entry["repeat"]["requests"] = len(again)
            report["policies"][policy] = entry
            side[policy] = {"wall_s": wall, "req_per_s": len(reqs) / wall if wall else 0.0,
                            "p50_ms": percentile(lat, 0.50) * 1e3,
                            "p99_ms": percentile(lat, 0.99) * 1e3}
        finally:
            service.close()
    if measured:
        report["measured"] = side
    return report


def report_json(report: dict) -> str:
    return json.dumps(report, indent=2, sort_keys=True) + "\n"
