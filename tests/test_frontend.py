"""HTTP front end (CPU): the reference server's endpoint contract
(pkg/tests/test_server.py) over the pool, with oracle-backed executors."""

import http.client
import json

import numpy as np
import pytest

from paper_2212_08146_b200.api import decode_response, encode_request
from paper_2212_08146_b200.frontend import parse_capacity, start
from paper_2212_08146_b200.hoststore import MemoryStore
from paper_2212_08146_b200.pool import KaasService
from paper_2212_08146_b200.workloads import matmul_chain_request
from test_service_cpu import OracleBacked


@pytest.fixture
def server():
    store = MemoryStore()
    svc = KaasService(store, n_executors=2, policy="affinity:8",
                      executor_factory=lambda i: OracleBacked(i, store, 1 << 20))
    srv, port = start(svc)
    yield port, store
    srv.shutdown()
    srv.server_close()
    svc.close()


def call(port, method, path, body=None, headers=None):
    c = http.client.HTTPConnection("127.0.0.1", port, timeout=30)
    c.request(method, path, body=body, headers=headers or {})
    r = c.getresponse()
    data = r.read()
    c.close()
    return r.status, data, r.getheader("Connection")


def test_health_stats_and_objects(server):
    port, store = server
    assert call(port, "GET", "/v1/health")[:2] == (200, b"ok")
    code, body, _ = call(port, "PUT", "/v1/objects/a%2Fb", b"\x01\x02\x03\x04")
    assert code == 200 and json.loads(body) == {"key": "a/b", "size": 4}
    assert call(port, "GET", "/v1/objects/a%2Fb")[:2] == (200, b"\x01\x02\x03\x04")
    code, body, conn = call(port, "GET", "/v1/objects/missing")
    assert code == 404 and json.loads(body)["error"]["kind"] == "NotFound" and conn == "close"
    code, body, _ = call(port, "GET", "/v1/stats")
    assert code == 200 and len(json.loads(body)["executors"]) == 2
    assert call(port, "GET", "/v1/nope")[0] == 404


def test_invoke_roundtrip_matches_direct_execution(server):
    port, store = server
    rng = np.random.default_rng(1234)
    a = rng.standard_normal(64).astype("<f4")
    b = rng.standard_normal(64).astype("<f4")
    for k, v in (("A", a), ("B", b)):
        assert call(port, "PUT", f"/v1/objects/{k}", v.tobytes())[0] == 200
    req = matmul_chain_request("http-1", 8)
    code, body, _ = call(port, "POST", "/v1/invoke", encode_request(req),
                         {"Content-Type": "application/json"})
    assert code == 200
    resp = decode_response(body, strict=True)
    assert resp.status.ok and resp.io_stats.store_puts == 1
    A, B = a.reshape(8, 8), b.reshape(8, 8)
    ab = np.zeros((8, 8), "<f4")
    for kk in range(8):
        ab += A[:, kk:kk + 1] * B[kk:kk + 1, :]
    d = np.zeros((8, 8), "<f4")
    for kk in range(8):
        d += ab[:, kk:kk + 1] * ab[kk:kk + 1, :]
    assert call(port, "GET", "/v1/objects/D")[1] == d.tobytes()


def test_decode_errors_are_400_and_close(server):
    port, _ = server
    code, body, conn = call(port, "POST", "/v1/invoke", b"{nope")
    assert code == 400 and json.loads(body)["error"]["kind"] == "ParseError" and conn == "close"
    code, body, _ = call(port, "POST", "/v1/invoke", b'{"request_id": 5}')
    assert code == 400 and json.loads(body)["error"]["kind"] == "SchemaError"
    # semantic errors travel in-band with 200
    code, body, _ = call(port, "POST", "/v1/invoke",
                         b'{"request_id":"","buffers":[],"invocations":[]}')
    assert code == 200 and decode_response(body).status.error_kind == "InvalidRequest"


def test_parse_capacity():
    assert parse_capacity("256MiB") == 256 << 20
    assert parse_capacity("2GiB") == 2 << 30
    assert parse_capacity("4096") == 4096


def test_reference_sdk_drives_the_front_end(server):
    """The reference's own client SDK (kaas_client) against this front end:
    its acceptance flow (pkg/sdk/tests/test_acceptance.py:30-50, matmul
    chain n=8 seed 1234, bit-exact) -- where the reference checkout exists."""
    import os
    import sys
    sdk = "/root/reference/pkg/sdk/src"
    if not os.path.isdir(sdk):
        pytest.skip("reference SDK not present")
    sys.path.insert(0, sdk)
    try:
        from kaas_client import ClientSession
        from kaas_client.builder import matmul_chain
    except ImportError:
        pytest.skip("kaas_client not importable")
    port, _ = server
    sess = ClientSession(f"127.0.0.1:{port}", strict=True)
    assert sess.health()
    n = 8
    rng = np.random.default_rng(1234)
    a = (rng.standard_normal(n * n) * 3).astype("<f4")
    b = (rng.standard_normal(n * n) * 3).astype("<f4")
    sess.put_object("acc/A", a.tobytes())
    sess.put_object("acc/B", b.tobytes())
    res = sess.invoke(matmul_chain("acc/A", "acc/B", "acc/D", n, request_id="acc-chain"))
    assert res.ok and res.io_stats.store_gets == 2 and res.io_stats.store_puts == 1

    def ref(x, y):
        out = np.zeros(n * n, "<f4")
        for i in range(n):
            for j in range(n):
                acc = np.float32(0.0)
                for k in range(n):
                    acc = np.float32(acc + x[i * n + k] * y[k * n + j])
                out[i * n + j] = acc
        return out
    ab = ref(a, b)
    assert sess.get_object("acc/D") == ref(ab, ab).tobytes()
