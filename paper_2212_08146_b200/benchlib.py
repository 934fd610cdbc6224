"""Bench harness over the GPU pool (``pkg/src/kaas/bench.py:234-355``,
``pkg/src/kaas/cli.py:108-170``): report v1 and v2, table, CLI.

``run_bench`` drives a fresh ``KaasService`` per policy with the reference's
request streams and aggregates exactly the reference's report fields (hit
rate, store traffic, virtual mean / nearest-rank p95 latency, per-executor
counts, busy fraction, virtual makespan).  Those are pure functions of the
cache and routing decisions, so a GPU run's report is byte-identical to the
reference's for a single submitter.  ``measured`` adds what the reference
cannot report: wall-clock req/s, p50/p99 wall latency and per-GPU device
time / copy volumes (kept outside the v1 fields).  Report v2
(``version=2``) is v1 with ``report_version`` 2 and those measurements
always present under ``measured``; every v1 field keeps its name and value.

    python -m paper_2212_08146_b200.benchlib run --workload mixed --requests 300 \
        --policies random:3,rr,affinity:8 --gpus 8 --v2 --out report.json
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


class _HttpClient:
    """Drive the pool through a real socket (reference ``_HttpClient``):
    the HTTP front end on ``host:port`` (port 0 = any), one connection per
    client thread."""

    def __init__(self, service, host: str, port: int):
        import threading

        from .frontend import start
        self._srv, self.port = start(service, host, port)
        self.host = host
        self._local = threading.local()

    def submit(self, req):
        import http.client

        from .api import decode_response, encode_request
        conn = getattr(self._local, "conn", None)
        if conn is None:
            conn = self._local.conn = http.client.HTTPConnection(self.host, self.port, timeout=300)
        conn.request("POST", "/v1/invoke", encode_request(req),
                     {"Content-Type": "application/json"})
        r = conn.getresponse()
        body = r.read()
        if r.status != 200:
            raise RuntimeError(f"HTTP {r.status}: {body[:200]!r}")
        return decode_response(body)

    def close(self):
        self._srv.shutdown()
        self._srv.server_close()


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
              service_factory=None, store_factory=MemoryStore, measured: bool = False,
              over_http: str | None = None, version: int = 1, devices=None) -> dict:
    """One fresh service per policy; returns the v1 report (plus ``measured``
    side fields when asked), or the v2 report (``version=2``).  ``over_http``
    = "host:port" drives the requests through the HTTP front end."""
    problems = spec.validate()
    if problems:
        raise ValueError("; ".join(problems))
    cap = capacity if capacity is not None else default_capacity(spec)
    if version not in (1, 2):
        raise ValueError(f"unknown report version {version}")
    measured = measured or version == 2
    report = {
        "report_version": version, "workload": asdict(spec), "executors": n_executors,
        "capacity": cap, "clients": clients, "warm_repeat": warm_repeat,
        "over_http": over_http is not None, "policies": {},
    }
    if service_factory is None:
        from .pool import KaasService

        def service_factory(store, policy):
            return KaasService(store, n_executors=n_executors, capacity=cap, policy=policy,
                               timing=timing, digest_cap=digest_cap, devices=devices)
    side = {}
    for policy in policies:
        store = store_factory()
        gen_data(spec, store)
        reqs = build_requests(spec)
        service = service_factory(store, policy)
        client = service
        if over_http:
            host, _, port = over_http.partition(":")
            client = _HttpClient(service, host or "127.0.0.1", int(port or 0))
        try:
            t0 = time.perf_counter()
            responses, lat = run_stream(client, reqs, clients)
            wall = time.perf_counter() - t0
            compute = sum(s.simulated_compute_time for r in responses for s in r.per_invocation)
            entry = aggregate(responses, service, compute)
            if warm_repeat:
                base = [e.requests_served for e in service.executors]
                again, _ = run_stream(client, reqs, clients)
                compute2 = sum(s.simulated_compute_time for r in again for s in r.per_invocation)
                entry["repeat"] = aggregate(again, service, compute + compute2)
                entry["repeat"]["per_executor_requests"] = [
                    e.requests_served - b for e, b in zip(service.executors, base)]
                entry["repeat"]["requests"] = len(again)
            report["policies"][policy] = entry
            side[policy] = {"wall_s": wall, "req_per_s": len(reqs) / wall if wall else 0.0,
                            "p50_ms": percentile(lat, 0.50) * 1e3,
                            "p99_ms": percentile(lat, 0.99) * 1e3}
            if version == 2:
                side[policy]["devices"] = [
                    e.device_stats() for e in service.executors if hasattr(e, "device_stats")]
        finally:
            if client is not service:
                client.close()
            service.close()
    if measured:
        report["measured"] = side
    return report


def report_json(report: dict) -> str:
    return json.dumps(report, indent=2, sort_keys=True) + "\n"


def render_table(report: dict) -> str:
    """The reference's table (bench.py:330-351), plus wall-clock columns
    when the report carries measurements."""
    cols = ["policy", "hit_rate", "gets", "puts", "mean_lat_ms", "p95_lat_ms", "busy", "errors"]
    meas = report.get("measured") or {}
    if meas:
        cols += ["req/s", "p50_ms", "p99_ms"]
    rows = [cols]
    for policy, e in report["policies"].items():
        row = [policy, f"{e['hit_rate']:.4f}", str(e["store_gets"]), str(e["store_puts"]),
               f"{e['mean_latency_ns'] / 1e6:.3f}", f"{e['p95_latency_ns'] / 1e6:.3f}",
               f"{e['gpu_busy_fraction']:.4f}", str(e["errors"])]
        if meas:
            m = meas.get(policy, {})
            row += [f"{m.get('req_per_s', 0.0):.1f}", f"{m.get('p50_ms', 0.0):.3f}",
                    f"{m.get('p99_ms', 0.0):.3f}"]
        rows.append(row)
    widths = [max(len(r[i]) for r in rows) for i in range(len(cols))]
    lines = []
    for i, row in enumerate(rows):
        lines.append("  ".join(c.ljust(w) for c, w in zip(row, widths)).rstrip())
        if i == 0:
            lines.append("  ".join("-" * w for w in widths))
    return "\n".join(lines)


def bench_main(argv=None) -> int:
    """``kaas-bench run`` (cli.py:108-170) over the GPU pool; extra flags:
    --gpus (devices to use), --store (pinned | mem), --v2."""
    import argparse
    import sys

    from .frontend import parse_capacity
    from .hoststore import PinnedStore
    from .timing import TimingModel
    ap = argparse.ArgumentParser(prog="kaas-bench", description="KaaS benchmark on B200")
    sub = ap.add_subparsers(dest="command", required=True)
    p = sub.add_parser("run", help="run a workload against each policy")
    p.add_argument("--workload", required=True, choices=["matmul_chain", "zipf_const", "mixed"])
    p.add_argument("--seed", type=int, default=0)
    p.add_argument("--requests", type=int, default=1000)
    p.add_argument("--policies", default="random:1,affinity:8")
    p.add_argument("--out", metavar="PATH")
    p.add_argument("--over-http", metavar="ADDR", dest="over_http")
    p.add_argument("--clients", type=int, default=1)
    p.add_argument("--warm-repeat", action="store_true")
    p.add_argument("--matrix-dim", type=int, default=4)
    p.add_argument("--zipf-s", type=float, default=1.0)
    p.add_argument("--key-universe", type=int, default=100)
    p.add_argument("--executors", type=int, default=4)
    p.add_argument("--capacity", default=None)
    p.add_argument("--timing", help="TimingModel JSON file (reference format)")
    p.add_argument("--gpus", type=int, default=0, help="GPUs to spread executors over (0 = all)")
    p.add_argument("--store", choices=("pinned", "mem"), default="pinned")
    p.add_argument("--v2", action="store_true", help="report_version 2 (v1 + measurements)")
    a = ap.parse_args(argv)
    spec = WorkloadSpec(kind=a.workload, request_count=a.requests, matrix_dim=a.matrix_dim,
                        zipf_s=a.zipf_s, key_universe=a.key_universe, seed=a.seed)
    problems = spec.validate()
    if a.clients < 1:
        problems.append("--clients must be >= 1")
    if a.executors < 1:
        problems.append("--executors must be >= 1")
    try:
        capacity = parse_capacity(a.capacity) if a.capacity else None
        timing = TimingModel.from_file(a.timing) if a.timing else None
    except (ValueError, OSError) as exc:
        problems.append(str(exc))
        capacity, timing = None, None
    if problems:
        print(f"kaas-bench: invalid workload: {'; '.join(problems)}", file=sys.stderr)
        return 2
    from .pool import visible_devices
    devs = visible_devices()
    if a.gpus:
        devs = devs[: a.gpus]
    report = run_bench(spec, [s.strip() for s in a.policies.split(",") if s.strip()],
                       n_executors=a.executors, capacity=capacity, timing=timing,
                       clients=a.clients, warm_repeat=a.warm_repeat, over_http=a.over_http,
                       version=2 if a.v2 else 1, measured=True, devices=devs,
                       store_factory=PinnedStore if a.store == "pinned" else MemoryStore)
    if not a.v2:
        report.pop("measured", None)  # v1: the reference's fields only
    print(render_table(report))
    if a.out:
        with open(a.out, "w", encoding="utf-8") as fh:
            fh.write(report_json(report))
        print(f"report written to {a.out}")
    return 0


if __name__ == "__main__":
    raise SystemExit(bench_main())
