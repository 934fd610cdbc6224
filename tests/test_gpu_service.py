"""The GPU pool reproduces the reference's bench reports byte for byte.

Four executors share the one GPU of the test box (each with its own ledger
and streams); routing, cache decisions and virtual timings are bit-exact, so
the v1 report equals the reference's (tests/golden/routing.json.gz)."""

import json

import pytest

from helpers import load_golden
from paper_2212_08146_b200.benchlib import report_json, run_bench
from paper_2212_08146_b200.hoststore import PinnedStore
from paper_2212_08146_b200.pool import KaasService
from paper_2212_08146_b200.workloads import WorkloadSpec, default_capacity

pytestmark = pytest.mark.gpu


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
def test_gpu_pool_report_matches_reference(cuda, key, spec, policies, n_exec, cap, warm):
    golden = load_golden("routing.json.gz")[key]
    capacity = cap if cap is not None else default_capacity(spec)

    def factory(store, policy):
        return KaasService(store, n_executors=n_exec, capacity=capacity, policy=policy,
                           devices=[0])

    rep = run_bench(spec, policies, n_executors=n_exec, capacity=cap, warm_repeat=warm,
                    service_factory=factory, store_factory=PinnedStore, measured=True)
    assert rep["measured"]
    assert _strip(rep) == golden


def test_gpu_pool_concurrent_clients(cuda):
    spec = WorkloadSpec("mixed", 400, seed=9)
    cap = default_capacity(spec)
    rep = run_bench(spec, ["affinity:8", "static", "exclusive"], n_executors=4, clients=16,
                    service_factory=lambda s, p: KaasService(s, n_executors=4, capacity=cap,
                                                             policy=p, devices=[0]),
                    store_factory=PinnedStore)
    for policy, entry in rep["policies"].items():
        assert entry["errors"] == 0, policy
        assert sum(entry["per_executor_requests"]) == 400


def test_http_front_end_over_gpu_pool(cuda):
    """Wire clients -> front end -> GPU pool: a cGEMM and a Jacobi request
    over HTTP, results fetched back through /v1/objects."""
    import http.client

    import numpy as np

    from paper_2212_08146_b200 import workloads as W
    from paper_2212_08146_b200.api import decode_response, encode_request
    from paper_2212_08146_b200.frontend import start

    store = PinnedStore()
    svc = KaasService(store, n_executors=2, capacity=256 << 20, policy="affinity:8", devices=[0])
    srv, port = start(svc)

    def call(method, path, body=None):
        c = http.client.HTTPConnection("127.0.0.1", port, timeout=60)
        c.request(method, path, body=body)
        r = c.getresponse()
        data = r.read()
        c.close()
        return r.status, data

    try:
        A, B = W.cgemm_data(64, seed=3)
        assert call("PUT", "/v1/objects/h/A", A.tobytes())[0] == 200
        assert call("PUT", "/v1/objects/h/B", B.tobytes())[0] == 200
        code, body = call("POST", "/v1/invoke",
                          encode_request(W.cgemm_request("h1", 64, "h/A", "h/B", "h/C")))
        assert code == 200 and decode_response(body, strict=True).status.ok
        code, data = call("GET", "/v1/objects/h/C")
        got = np.frombuffer(data, "<c8").astype(np.complex128).reshape(64, 64)
        truth = A.astype(np.complex128) @ B.astype(np.complex128)
        assert np.linalg.norm(got - truth) / np.linalg.norm(truth) <= 1e-4
        from oracle.executor import DictStore, OracleExecutor
        W.seed_jacobi(store, 256, prefix="hj")
        ostore = DictStore()
        W.seed_jacobi(ostore, 256, prefix="hj")
        jreq = W.jacobi_request("h2", 256, 50, "hj/A/256", "hj/b/256", "hj/x0/256", "hj/x", "hj/r")
        code, body = call("POST", "/v1/invoke", encode_request(jreq))
        assert code == 200 and decode_response(body).status.ok
        OracleExecutor(1 << 30, ostore).execute(jreq)
        x = np.frombuffer(call("GET", "/v1/objects/hj/x")[1], "<f4").astype(np.float64)
        ox = np.frombuffer(ostore.get("hj/x"), "<f4").astype(np.float64)
        assert np.abs(x - ox).max() <= 1e-5
    finally:
        srv.shutdown()
        srv.server_close()
        svc.close()


def test_gpu_report_v2_over_http(cuda):
    """Report v2 through the HTTP front end over the GPU pool: the v1 fields
    are the reference's (modulo the over_http flag) and every GPU executor's
    device measurements are attached."""
    golden = load_golden("routing.json.gz")["bench_matmul_chain"]
    spec = WorkloadSpec("matmul_chain", 6, matrix_dim=16, seed=5)

    def factory(store, policy):
        return KaasService(store, n_executors=2, capacity=default_capacity(spec), policy=policy,
                           devices=[0])

    rep = run_bench(spec, ["rr"], n_executors=2, warm_repeat=True, over_http="127.0.0.1:0",
                    version=2, service_factory=factory, store_factory=PinnedStore)
    rep = json.loads(report_json(rep))
    meas = rep.pop("measured")
    assert rep.pop("report_version") == 2 and rep.pop("over_http") is True
    g = dict(golden)
    g.pop("report_version"), g.pop("over_http")
    assert rep == g
    devs = meas["rr"]["devices"]
    assert len(devs) == 2 and all(d["kernel_launches"] > 0 for d in devs)


def _decisions_only_kernels():
    """The oracle's kernel table with the numerics dropped: same literal
    types, arity, writes and FMA counts (virtual time), no data -- decisions
    do not depend on kernel outputs."""
    from oracle.kernels import KERNELS

    def fma(kid):
        if kid == "cgemm":
            return lambda d, l, v: 4 * l[0].value * l[1].value * l[2].value
        if kid == "jacobi_sweep":
            return lambda d, l, v: l[0].value * l[0].value
        raise KeyError(kid)
    return {kid: (spec[0], spec[1], spec[2], fma(kid)) for kid, spec in KERNELS.items()
            if kid in ("cgemm", "jacobi_sweep")}


class _SizedStore:
    """Oracle-side store: only object sizes matter for decisions."""

    def __init__(self, sizes):
        self.sizes = dict(sizes)

    def get(self, key):
        if key not in self.sizes:
            raise KeyError(key)
        return memoryview(bytearray(self.sizes[key]))

    def put(self, key, payload):
        self.sizes[key] = len(payload)


@pytest.mark.parametrize("policy", ["affinity:2", "static", "exclusive", "rr"])
def test_sixteen_client_mixed_decisions_replay(cuda, policy):
    """BASELINE configs[3] (shrunk): 16 client threads, mixed cGEMM + Jacobi
    under LRU pressure, 4 executors.  Every logged routing decision is
    replayed through the oracle policy on the logged state (SURVEY §7.3
    #10), and each executor's request sequence through an oracle executor:
    statuses, IoStats, per-invocation and total virtual times identical."""
    import threading

    from oracle.executor import OracleExecutor
    from oracle.router import OracleRouter
    from paper_2212_08146_b200 import workloads as W
    from paper_2212_08146_b200.api import response_to_doc

    store = PinnedStore()
    uni = W.mixed_universe(store, n_cgemm=6, cg_n=512, n_jacobi=6, jac_n=1024, seed=3)
    reqs = W.mixed_requests(uni, 160, sweeps=20, seed=5)
    cap = 3 * 4 * 1024 * 1024 + 2 * 2 * 1024 * 1024  # ~5 const matrices per executor: evictions
    sizes = {k: len(store.get(k)) for k in store.keys()}
    got = {}
    with KaasService(store, n_executors=4, capacity=cap, policy=policy, devices=[0],
                     log_decisions=True) as svc:
        lock = threading.Lock()
        it = iter(range(len(reqs)))

        def client():
            while True:
                with lock:
                    i = next(it, None)
                if i is None:
                    return
                got[reqs[i].request_id] = svc.submit(reqs[i])

        threads = [threading.Thread(target=client) for _ in range(16)]
        for t in threads:
            t.start()
        for t in threads:
            t.join()
        decisions = list(svc.router.decisions)
    assert len(decisions) == len(reqs) and all(r.status.ok for r in got.values())
    by_id = {r.request_id: r for r in reqs}
    # 1. decision function: the oracle policy on the logged state
    orc = OracleRouter([0, 1, 2, 3], policy)
    per_exec = {e: [] for e in range(4)}
    for rid, chosen, state in decisions:
        for e, (depth, items) in state.items():
            orc.depth[e] = depth
            orc.keys[e].clear()
            orc.keys[e].update(items)
        assert orc.pick(by_id[rid]) == chosen, rid
        per_exec[chosen].append(rid)
    # 2. each executor's sequence (FIFO per executor = routing order)
    kernels = _decisions_only_kernels()
    for e, rids in per_exec.items():
        oex = OracleExecutor(cap, _SizedStore(sizes), kernels=kernels)
        for rid in rids:
            want = response_to_doc(oex.execute(by_id[rid]))
            assert response_to_doc(got[rid]) == want, (e, rid)
