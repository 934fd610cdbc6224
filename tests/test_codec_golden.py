"""Request API parity against the REAL reference codec (CPU).

``golden/codec.json.gz`` holds the reference's outcomes
(``golden/make_codec_golden.py``) for 2,500 ``genreq.wire_random_request``
bodies x (original + 4 mutations) x {lenient, strict}, 800 x 4 wire
responses, ``valid_store_key`` on edge keys and ``ScalarLiteral`` equality.
Every case must come out of ``paper_2212_08146_b200.api`` identically: the
same accepted request (re-encoded) and violations, or the same exception
class and message.  When the reference is mounted (the build container), a
further 20,000 fresh documents are compared live.
"""

from __future__ import annotations

import os
import random
import sys

import pytest

from paper_2212_08146_b200 import api as A

import codec_cases as C
from helpers import load_golden

REF = "/root/reference"


def _req_outcome(body, strict):
    def dec():
        req = A.decode_request(body, strict)
        return [A.encode_request(req).decode(), A.validate_request(req)]
    return list(C.outcome(dec))


def _slow_outcome(body, strict):
    def dec():
        req = A.request_from_doc(A._loads(body), strict)
        return [A.encode_request(req).decode(), A.validate_request(req)]
    return list(C.outcome(dec))


def _resp_outcome(body, strict):
    return list(C.outcome(lambda: A.encode_response(A.decode_response(body, strict)).decode()))


@pytest.fixture(scope="module")
def golden():
    return load_golden("codec.json.gz")


def _norm(o):
    return [o[0], o[1]] if o[0] != "ok" else ["ok", [o[1][0], list(o[1][1])]]


def test_request_decode_matches_reference(golden):
    bad = []
    for seed, rec in enumerate(golden["requests"]):
        body = rec["body"].encode()
        cases = [body] + C.mutations(body, seed)
        for ci, (case, want) in enumerate(zip(cases, rec["outcomes"])):
            for mode, strict in enumerate((False, True)):
                got = _norm(_req_outcome(case, strict))
                if got != want[mode] or _norm(_slow_outcome(case, strict)) != want[mode]:
                    bad.append((seed, ci, strict, got, want[mode]))
    assert not bad, f"{len(bad)} mismatches, first: {bad[:3]}"


def test_response_decode_matches_reference(golden):
    bad = []
    for seed, rec in enumerate(golden["responses"]):
        for ci, (case, want) in enumerate(zip(C.response_docs(seed), rec)):
            for mode, strict in enumerate((False, True)):
                got = list(_resp_outcome(case, strict))
                if got != want[mode]:
                    bad.append((seed, ci, strict, got, want[mode]))
    assert not bad, f"{len(bad)} mismatches, first: {bad[:3]}"


def test_store_keys_and_literal_equality_match_reference(golden):
    for key, want in golden["store_keys"]:
        assert A.valid_store_key(key) is want, repr(key)
    for key, want in golden["key_violations"]:
        got = A.validate_request(A.KaasRequest("r", (A.BufferArg("x", 4, "input", key=key),), ()))
        assert got == want, repr(key)
    lits = C.LITERAL_VALUES
    got = [[A.ScalarLiteral(t, a) == A.ScalarLiteral(t, b) for b in lits for t in ("f32", "i32")]
           for a in lits]
    assert got == golden["literal_eq"]


def test_trailing_newline_key_round_trips_like_the_reference():
    req = A.KaasRequest("r", (A.BufferArg("x", 4, "input", key="k\n"),), ())
    assert A.validate_request(req) == []
    assert A.decode_request(A.encode_request(req)) == req


@pytest.mark.skipif(not os.path.isdir(os.path.join(REF, "pkg", "src")),
                    reason="reference not mounted (golden fixture still pins the codec)")
def test_live_differential_against_reference():
    """20,000 fresh reference-generated documents (seeds disjoint from the
    fixture's) through both codecs: zero kind / message / validation
    mismatches."""
    sys.path.insert(0, os.path.join(REF, "pkg", "src"))
    sys.path.insert(0, os.path.join(REF, "pkg", "tests"))
    try:
        from kaas import protocol as P
        import genreq
    finally:
        del sys.path[:2]

    def ref(body, strict):
        def dec():
            req = P.decode_request(body, strict)
            return [P.encode_request(req).decode(), P.validate_request(req)]
        return _norm(list(C.outcome(dec)))

    n, bad = 0, []
    for seed in range(100_000, 104_000):
        body = P.encode_request(genreq.wire_random_request(random.Random(seed)))
        for case in [body] + C.mutations(body, seed):
            strict = bool(n & 1)
            n += 1
            got, want = _norm(_req_outcome(case, strict)), ref(case, strict)
            if got != want:
                bad.append((seed, strict, got, want))
    assert n == 20_000
    assert not bad, f"{len(bad)} mismatches, first: {bad[:3]}"
