"""Pool + router + bench harness against the reference's own bench reports.

The product service is driven with oracle-backed executors (CPU), so these
tests pin the host-side routing / queueing / aggregation logic without a GPU;
tests/test_gpu_service.py repeats them with the B200 executors.
"""

import json

import pytest

from helpers import load_golden
from oracle.executor import OracleExecutor
from paper_2212_08146_b200.benchlib import report_json, run_bench
from paper_2212_08146_b200.faults import NotFoundError
from paper_2212_08146_b200.pool import KaasService
from paper_2212_08146_b200.workloads import WorkloadSpec


class _StoreView:
    """Oracle expects KeyError for a missing key."""

    def __init__(self, store):
        self.store = store

    def get(self, key):
        try:
            return self.store.get(key)
        except NotFoundError:
            raise KeyError(key) from None

    def put(self, key, payload):
        self.store.put(key, payload)


class _Clock:
    def __init__(self, ex):
        self.ex = ex

    @property
    def now_ns(self):
        return self.ex.now


class OracleBacked:
    def __init__(self, i, store, capacity):
        self.executor_id = i
        self.inner = OracleExecutor(capacity, _StoreView(store))
        self.clock = _Clock(self.inner)

    def execute(self, req):
        return self.inner.execute(req)

    @property
    def requests_served(self):
        return self.inner.served

    def stats(self):
        return {"executor_id": self.executor_id, "requests": self.inner.served}


def oracle_service(n_executors, capacity):
    def factory(store, policy):
        return KaasService(store, n_executors=n_executors, policy=policy,
                           executor_factory=lambda i: OracleBacked(i, store, capacity))
    return factory


def _strip(rep):
    rep = json.loads(report_json(rep))
    rep.pop("measured", None)
    return rep


@pytest.mark.parametrize("key,spec,policies,n_exec,cap,warm", [
    ("bench_zipf_const", WorkloadSpec("zipf_const", 5000, zipf_s=1.0, key_universe=100, seed=42),
     ["random:1", "affinity:8"], 4, 30 * 64 * 1024, False),
    ("bench_mixed", WorkloadSpec("mixed", 300, seed=7), ["random:3", "rr", "affinity:8"], 4, None, True),
    ("bench_matmul_chain", WorkloadSpec("matmul_chain", 6, matrix_dim=16, seed=5), ["rr"], 2, None, True),
])
def test_report_matches_reference(key, spec, policies, n_exec, cap, warm):
    golden = load_golden("routing.json.gz")[key]
    from paper_2212_08146_b200.workloads import default_capacity
    capacity = cap if cap is not None else default_capacity(spec)
    rep = run_bench(spec, policies, n_executors=n_exec, capacity=cap, warm_repeat=warm,
                    service_factory=oracle_service(n_exec, capacity))
    assert _strip(rep) == golden


def test_affinity_margin_gate():
    """test_acceptance.py:270-288: affinity beats random by >= 0.30."""
    rep = load_golden("routing.json.gz")["bench_zipf_const"]
    margin = rep["policies"]["affinity:8"]["hit_rate"] - rep["policies"]["random:1"]["hit_rate"]
    assert margin >= 0.30


def test_multi_client_service_completes_and_balances():
    spec = WorkloadSpec("zipf_const", 800, key_universe=40, seed=3)
    from paper_2212_08146_b200.workloads import default_capacity
    cap = default_capacity(spec)
    rep = run_bench(spec, ["affinity:8", "static", "exclusive"], n_executors=4, clients=8,
                    service_factory=oracle_service(4, cap))
    for policy, entry in rep["policies"].items():
        assert entry["requests"] == 800 and entry["errors"] == 0, policy
        assert sum(entry["per_executor_requests"]) == 800


def test_report_over_http_and_v2():
    """The v1 report through the HTTP front end (reference ``--over-http``)
    equals the golden report except for the ``over_http`` flag; v2 keeps
    every v1 field and adds the measurements."""
    golden = load_golden("routing.json.gz")["bench_matmul_chain"]
    spec = WorkloadSpec("matmul_chain", 6, matrix_dim=16, seed=5)
    from paper_2212_08146_b200.workloads import default_capacity
    capacity = default_capacity(spec)
    rep = run_bench(spec, ["rr"], n_executors=2, warm_repeat=True, over_http="127.0.0.1:0",
                    service_factory=oracle_service(2, capacity))
    rep = _strip(rep)
    assert rep.pop("over_http") is True
    g = dict(golden)
    assert g.pop("over_http") is False
    assert rep == g
    v2 = run_bench(spec, ["rr"], n_executors=2, warm_repeat=True, version=2,
                   service_factory=oracle_service(2, capacity))
    v2 = json.loads(report_json(v2))
    meas = v2.pop("measured")
    assert v2.pop("report_version") == 2 and meas["rr"]["req_per_s"] > 0
    g2 = dict(golden)
    g2.pop("report_version")
    assert v2 == g2


def test_bench_cli_validates_like_the_reference(capsys):
    from paper_2212_08146_b200.benchlib import bench_main
    assert bench_main(["run", "--workload", "mixed", "--requests", "0"]) == 2
    assert "invalid workload" in capsys.readouterr().err


class _FakePipelined:
    """GPU-executor-shaped stand-in (begin / complete / inflight / execute):
    records the order in which requests reach it, and sleeps a little so the
    pool's inline and worker paths interleave."""

    def __init__(self, eid):
        import threading
        self.executor_id = eid
        self.order = []
        self._inflight = {}
        self._seq = 0
        self._lock = threading.Lock()
        self.on_complete = None
        self.poisoned = None

    @property
    def inflight(self):
        return len(self._inflight)

    def _resp(self, req):
        from paper_2212_08146_b200.api import KaasResponse, Status
        return KaasResponse(req.request_id, Status.make_ok())

    def execute(self, req):
        import time
        with self._lock:
            self.order.append(req.request_id)
        time.sleep(0.0003)
        return self._resp(req)

    def begin(self, req):
        from types import SimpleNamespace
        with self._lock:
            self.order.append(req.request_id)
        self._seq += 1
        rec = SimpleNamespace(seq=self._seq, response=self._resp(req))
        self._inflight[self._seq] = rec
        return rec

    def complete(self, through=None, block=True):
        import time
        done = 0
        for seq in sorted(self._inflight):
            if through is not None and seq > through:
                break
            time.sleep(0.0002)
            rec = self._inflight.pop(seq)
            if self.on_complete is not None:
                self.on_complete(rec, rec.response)
            done += 1
        return done


@pytest.mark.parametrize("policy", ["rr", "affinity:8", "random:7", "exclusive"])
def test_each_executor_runs_requests_in_routing_order(policy):
    """Many client threads through submit(): every executor sees its requests
    in the order the router placed them (the inline fast path may not
    overtake a request routed earlier), so a decision log replays against a
    FIFO executor (tests/test_gpu_service.py)."""
    import threading
    from paper_2212_08146_b200 import workloads as W

    reqs = [W.cgemm_request(f"t{i % 16}/r{i}", 8, f"k/A{i % 5}", f"k/B{i % 3}", f"k/C{i % 7}")
            for i in range(600)]
    svc = KaasService(None, n_executors=4, policy=policy, executor_factory=_FakePipelined,
                      log_decisions=True)
    try:
        it = iter(range(len(reqs)))
        lock = threading.Lock()

        def client():
            while True:
                with lock:
                    i = next(it, None)
                if i is None:
                    return
                assert svc.submit(reqs[i]).status.ok

        threads = [threading.Thread(target=client) for _ in range(16)]
        for t in threads:
            t.start()
        for t in threads:
            t.join()
        decisions = list(svc.router.decisions)
    finally:
        svc.close()
    assert len(decisions) == len(reqs)
    for e in svc.executors:
        routed = [rid for rid, chosen, _ in decisions if chosen == e.executor_id]
        assert e.order == routed
