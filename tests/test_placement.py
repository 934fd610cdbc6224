"""Router decisions: the reference's exact sequences (pkg/tests/test_router.py)
plus the two new policies against the oracle restatement."""

import pytest

from helpers import load_golden
from oracle.router import OracleRouter
from paper_2212_08146_b200.api import BufferArg, IoStats, KaasRequest, KaasResponse, Status
from paper_2212_08146_b200.faults import NoExecutorsError, UnknownExecutorError
from paper_2212_08146_b200.placement import (
    AffinityPolicy,
    RandomPolicy,
    RoundRobinPolicy,
    Router,
    parse_policy,
)
from paper_2212_08146_b200.workloads import WorkloadSpec, build_requests


def const_request(*keys, size=64, rid="r"):
    return KaasRequest(rid, buffers=tuple(
        BufferArg(f"b{i}", size, "input", key=k, is_const=True) for i, k in enumerate(keys)))


OK = KaasResponse("r", Status.make_ok(), io_stats=IoStats())


def test_round_robin_cycles():
    r = Router([0, 1, 2], RoundRobinPolicy())
    seq = []
    for _ in range(6):
        e = r.route(const_request("w"))
        seq.append(e)
        r.update_digest(e, OK, const_request("w"))
    assert seq == [0, 1, 2, 0, 1, 2]


def test_random_seed_deterministic():
    def run(seed):
        r = Router([0, 1, 2, 3], RandomPolicy(seed))
        out = []
        for _ in range(20):
            e = r.route(const_request("w"))
            out.append(e)
            r.update_digest(e, OK, const_request("w"))
        return out
    assert run(9) == run(9) and run(9) != run(10)


def test_affinity_reference_sequences():
    r = Router([0, 1, 2, 3], AffinityPolicy(q_max=1))
    warm = const_request("hot")
    e = r.route(warm)
    r.update_digest(e, OK, warm)
    assert [r.route(const_request("hot", rid=f"r{i}")) for i in range(6)] == [0, 0, 1, 2, 3, 1]
    r = Router([0, 1, 2, 3], AffinityPolicy(8))
    seq = []
    for i in range(8):
        q = const_request(f"cold{i}", rid=f"r{i}")
        e = r.route(q)
        seq.append(e)
        r.update_digest(e, OK, q)
    assert seq == [0, 1, 2, 3, 0, 1, 2, 3]


def test_affinity_scores_bytes_and_spills():
    r = Router([0, 1], AffinityPolicy(8))
    big = const_request("big", size=1024, rid="b")
    r.route(big)
    r.update_digest(0, OK, big)
    smalls = const_request("s1", "s2", size=64, rid="s")
    e = r.route(smalls)
    r.update_digest(e, OK, smalls)
    mixed = KaasRequest("m", buffers=(
        BufferArg("x", 1024, "input", key="big", is_const=True),
        BufferArg("y", 64, "input", key="s1", is_const=True),
        BufferArg("z", 64, "input", key="s2", is_const=True)))
    assert r.route(mixed) == 0
    r2 = Router([0, 1], AffinityPolicy(q_max=2))
    w = const_request("w")
    r2.route(w)
    r2.update_digest(0, OK, w)
    r2.digests[0].queue_depth = 3
    assert r2.route(w) == 1


def test_digest_cap_and_errors():
    r = Router([0], RoundRobinPolicy(), digest_cap=3)
    for i in range(5):
        q = const_request(f"k{i}")
        r.route(q)
        r.update_digest(0, OK, q)
    assert list(r.digests[0].keys) == ["k2", "k3", "k4"]
    assert r.digests[0].used_bytes == 3 * 64
    with pytest.raises(UnknownExecutorError):
        r.update_digest(9, OK, const_request("x"))
    with pytest.raises(NoExecutorsError):
        Router([], RoundRobinPolicy()).route(const_request("x"))


def test_failed_response_does_not_update_digest():
    r = Router([0, 1], AffinityPolicy(8))
    q = const_request("w")
    e = r.route(q)
    r.update_digest(e, KaasResponse("r", Status.make_error("NotFound", "x")), q)
    assert r.digests[e].queue_depth == 0 and not r.digests[e].keys


@pytest.mark.parametrize("policy", ["random:1", "rr", "affinity:8", "affinity:1"])
def test_zipf_placements_match_reference(policy):
    golden = load_golden("routing.json.gz")[f"zipf_{policy}"]
    reqs = build_requests(WorkloadSpec("zipf_const", 2000, zipf_s=1.0, key_universe=100, seed=42))
    r = Router([0, 1, 2, 3], parse_policy(policy))
    seq = []
    for q in reqs:
        e = r.route(q)
        seq.append(e)
        r.update_digest(e, OK, q)
    assert seq == golden


@pytest.mark.parametrize("policy", ["static", "exclusive", "affinity:2", "random:5", "rr"])
def test_policies_match_oracle_with_inflight_depths(policy):
    """Interleaved route/complete (requests in flight) against the oracle."""
    import random as _r
    rng = _r.Random(99)
    reqs = build_requests(WorkloadSpec("mixed", 600, key_universe=30, seed=4))
    reqs = [KaasRequest(f"tenant{rng.randrange(5)}/{q.request_id}", q.buffers, q.invocations)
            for q in reqs]
    r = Router([0, 1, 2, 3, 4, 5], parse_policy(policy))
    o = OracleRouter([0, 1, 2, 3, 4, 5], policy)
    inflight = []
    for q in reqs:
        e1, e2 = r.route(q), o.route(q)
        assert e1 == e2
        inflight.append((e1, q))
        while inflight and rng.random() < 0.6:
            e, done = inflight.pop(rng.randrange(len(inflight)))
            ok = rng.random() < 0.9
            r.update_digest(e, OK if ok else KaasResponse("r", Status.make_error("NotFound", "x")), done)
            o.complete(e, ok, done)


def test_parse_policy_spellings():
    assert str(parse_policy("rr")) == "rr"
    assert str(parse_policy("random:3")) == "random:3"
    assert str(parse_policy("affinity:4")) == "affinity:4"
    assert str(parse_policy("static")) == "static"
    assert str(parse_policy("exclusive")) == "exclusive"
    for bad in ("nope", "random:", "affinity:x"):
        with pytest.raises(ValueError):
            parse_policy(bad)
    with pytest.raises(ValueError):
        AffinityPolicy(0)


def test_exclusive_isolates_tenants_and_static_is_stable():
    r = Router([0, 1, 2], parse_policy("exclusive"))
    homes = {}
    for i in range(30):
        t = f"t{i % 4}"
        e = r.route(KaasRequest(f"{t}/{i}"))
        homes.setdefault(t, e)
        assert homes[t] == e
    assert sorted(homes.values()) == [0, 0, 1, 2]
    s = Router([0, 1, 2, 3], parse_policy("static"))
    q = const_request("w1", "w2")
    assert len({s.route(q) for _ in range(20)}) == 1


def test_new_policies_route_malformed_requests_instead_of_raising():
    """A request with a non-str id (or non-str const keys) is routed -- the
    executor then answers InvalidRequest in band, as with the reference's
    own policies -- never an exception out of Router.route."""
    from paper_2212_08146_b200.api import BufferArg, KaasRequest
    from paper_2212_08146_b200.placement import Router, parse_policy

    bad = [KaasRequest(5), KaasRequest(None), KaasRequest(""),
           KaasRequest("r", (BufferArg("a", 4, "input", key=7, is_const=True),))]
    for spec in ("static", "exclusive"):
        r = Router([0, 1, 2], parse_policy(spec))
        for req in bad:
            assert r.route(req) in (0, 1, 2)


def test_router_skips_executors_marked_down():
    from paper_2212_08146_b200.api import KaasRequest
    from paper_2212_08146_b200.placement import Router, parse_policy

    r = Router([0, 1, 2], parse_policy("rr"))
    r.mark_down(1)
    assert [r.route(KaasRequest(f"q{i}")) for i in range(4)] == [0, 2, 0, 2]
    r.mark_down(0)
    r.mark_down(2)
    assert r.route(KaasRequest("all-down")) in (0, 1, 2)  # still answered (in band)
