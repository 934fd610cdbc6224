"""Wire codec (CPU): the decode fast path is indistinguishable from the
checked decoder (pkg/src/kaas/protocol.py:314-567 restated in api.py) --
same requests, same errors -- and interns resent kernel graphs."""

import json
import math

import pytest

from paper_2212_08146_b200 import workloads as W
from paper_2212_08146_b200.api import (ParseError, SchemaError, _loads, decode_request,
                                       encode_request, request_from_doc)


def _both(body, strict=False):
    """(fast result or exception, checked result or exception)"""
    out = []
    for fn in (lambda: decode_request(body, strict), lambda: request_from_doc(_loads(body), strict)):
        try:
            out.append(("ok", fn()))
        except (ParseError, SchemaError) as exc:
            out.append((type(exc).__name__, str(exc)))
    return out


def _jacobi_doc():
    return json.loads(encode_request(W.jacobi_request("j", 64, 6, "A", "b", "x0", "x", "r")))


def test_fast_path_equals_checked_decoder_and_interns_graphs():
    for strict in (False, True):
        body = encode_request(W.jacobi_request("j1", 4096, 500, "A", "b", "x0", "x", "r"))
        (k1, a), (k2, b) = _both(body, strict)
        assert k1 == k2 == "ok" and a == b
        again = decode_request(body.replace(b'"j1"', b'"j2"'), strict)
        assert again.request_id == "j2"
        assert again.invocations is a.invocations and again.buffers is a.buffers


@pytest.mark.parametrize("mutate", [
    lambda d: d["invocations"][3]["dims"].__setitem__("grid_x", True),
    lambda d: d["invocations"][3]["dims"].__setitem__("grid_x", 2.0),
    lambda d: d["invocations"][2]["literals"][0].__setitem__("value", 7.5),
    lambda d: d["invocations"][2]["literals"][0].__setitem__("type", "u8"),
    lambda d: d["invocations"][2]["literals"][0].pop("value"),
    lambda d: d["invocations"][1].__setitem__("args", ["A", 3]),
    lambda d: d["invocations"][1].pop("dims"),
    lambda d: d["invocations"][0].__setitem__("extra", 1),
    lambda d: d["invocations"][0]["dims"].__setitem__("grid_w", 1),
    lambda d: d.__setitem__("invocations", {}),
    lambda d: d["buffers"][0].__setitem__("size", "64"),
    lambda d: d.__setitem__("extra", 0),
    lambda d: d.pop("request_id"),
    lambda d: d["invocations"].append(5),
])
def test_malformed_inputs_fail_identically(mutate):
    for strict in (False, True):
        doc = _jacobi_doc()
        mutate(doc)
        body = json.dumps(doc).encode()
        fast, slow = _both(body, strict)
        assert fast == slow, (strict, fast, slow)


def test_float_literals_keep_their_bits_and_words():
    doc = _jacobi_doc()
    inv = doc["invocations"][0]
    variants = [0.0, -0.0, 1, 2.5, "NaN", "Infinity", "-Infinity"]
    got = []
    for v in variants:
        inv2 = dict(inv, kernel_id="fill", literals=[{"type": "i32", "value": 4},
                                                     {"type": "f32", "value": v}])
        d = dict(doc, invocations=[inv2])
        (k1, a), (k2, b) = _both(json.dumps(d).encode())
        assert k1 == k2 == "ok" and a == b
        got.append(a.invocations[0].literals[1].value)
    assert math.copysign(1.0, got[0]) == 1.0 and math.copysign(1.0, got[1]) == -1.0
    assert isinstance(got[2], float) and got[2] == 1.0
    assert math.isnan(got[4]) and got[5] == math.inf and got[6] == -math.inf
