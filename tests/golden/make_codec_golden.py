"""Record the REAL reference codec's behaviour on the edge-case corpus.

Run in the build container (the reference is mounted read-only there):

    python tests/golden/make_codec_golden.py [/root/reference]

Base requests come from the reference's own generator
(``pkg/tests/genreq.py:52-89`` ``wire_random_request``, seeds 0..N-1),
encoded by the reference (``protocol.py:314-338``).  Each body and its
mutations (``tests/codec_cases.py``) are decoded by the reference in lenient
and strict mode (``protocol.py:454-511``); an accepted request is recorded as
its re-encoding plus ``validate_request``'s violations (``protocol.py:209-281``),
a rejected one as the exception's class and message.  Wire responses
(``protocol.py:514-567``), ``valid_store_key`` (``protocol.py:42-47``) and
``ScalarLiteral`` equality (``protocol.py:80-89``) are recorded the same way.
Output: ``codec.json.gz`` next to this file.
"""

from __future__ import annotations

import gzip
import json
import os
import random
import sys

REF = sys.argv[1] if len(sys.argv) > 1 else "/root/reference"
HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.join(REF, "pkg", "src"))
sys.path.insert(0, os.path.join(REF, "pkg", "tests"))
sys.path.insert(0, os.path.dirname(HERE))

from kaas import protocol as P  # noqa: E402

import codec_cases as C  # noqa: E402
import genreq  # noqa: E402  (reference test generator)

N_REQUESTS = 2500
N_RESPONSES = 800


def _req_outcome(body, strict):
    def dec():
        req = P.decode_request(body, strict)
        return [P.encode_request(req).decode(), P.validate_request(req)]
    return list(C.outcome(dec))


def _resp_outcome(body, strict):
    return list(C.outcome(lambda: P.encode_response(P.decode_response(body, strict)).decode()))


def main():
    requests = []
    for seed in range(N_REQUESTS):
        body = P.encode_request(genreq.wire_random_request(random.Random(seed)))
        cases = [body] + C.mutations(body, seed)
        requests.append({
            "body": body.decode(),
            "outcomes": [[_req_outcome(c, s) for s in (False, True)] for c in cases],
        })
    responses = []
    for seed in range(N_RESPONSES):
        responses.append([[_resp_outcome(c, s) for s in (False, True)]
                          for c in C.response_docs(seed)])
    keys = [[k, P.valid_store_key(k)] for k in C.STORE_KEYS]
    key_violations = [[k, P.validate_request(P.KaasRequest(
        "r", (P.BufferArg("x", 4, "input", key=k),), ()))] for k in C.STORE_KEYS]
    lits = C.LITERAL_VALUES
    eq = [[P.ScalarLiteral(t, a) == P.ScalarLiteral(t, b) for b in lits for t in ("f32", "i32")]
          for a in lits]
    out = {"generator": "genreq.wire_random_request + tests/codec_cases.py",
           "n_requests": N_REQUESTS, "requests": requests, "responses": responses,
           "store_keys": keys, "key_violations": key_violations, "literal_eq": eq}
    path = os.path.join(HERE, "codec.json.gz")
    with gzip.open(path, "wt", compresslevel=9) as f:
        json.dump(out, f, separators=(",", ":"))
    n = sum(len(r["outcomes"]) for r in requests)
    print(f"wrote {path}: {n} request cases x 2 modes, {len(responses) * 4} response cases, "
          f"{os.path.getsize(path)} bytes")


if __name__ == "__main__":
    main()
