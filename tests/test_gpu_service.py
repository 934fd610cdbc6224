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
