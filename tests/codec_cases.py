"""Deterministic codec edge-case corpus (shared by the golden generator and
the CPU codec tests).

``mutations(body, seed)`` derives malformed / unusual variants of one wire
request: wrong JSON types at any depth, missing and unknown fields, unknown
enum words, bad float words, +-0 / NaN / out-of-range literals, store keys
with a trailing newline or foreign characters, and byte-level damage
(truncation, invalid UTF-8).  ``response_docs(seed)`` does the same for wire
responses.  Nothing here imports the reference: ``golden/make_codec_golden.py``
runs these cases through the real reference codec (``protocol.py:390-567``)
and records every outcome; ``test_codec_golden.py`` replays them through
``paper_2212_08146_b200.api``.
"""

from __future__ import annotations

import json
import random

_ODD_VALUES = (True, False, None, 0, 1, -1, 2.5, -0.0, "x", "", [], {}, [1], {"a": 1},
               1 << 31, -(1 << 31) - 1, 1 << 63, 10 ** 30, "NaN", "Infinity", "-Infinity",
               "nan", "inf")
_ODD_KEYS = ("k\n", "k\n\n", "\nk", "a b", "a\tb", "é", "k" * 256, "k" * 257, "", "a/b.c-d_e",
             "a\r", "k\x00")
_FLOATS = (0.0, -0.0, "NaN", "Infinity", "-Infinity", 1e308, -1e-310, 3, -7, True, "1.5",
           1e39, -1e39)


def _paths(doc, prefix=()):
    """Every (path, value) in a JSON document, containers included."""
    out = [(prefix, doc)]
    if isinstance(doc, dict):
        for k, v in doc.items():
            out.extend(_paths(v, prefix + (k,)))
    elif isinstance(doc, list):
        for i, v in enumerate(doc):
            out.extend(_paths(v, prefix + (i,)))
    return out


def _set(doc, path, value):
    cur = doc
    for p in path[:-1]:
        cur = cur[p]
    cur[path[-1]] = value


def _del(doc, path):
    cur = doc
    for p in path[:-1]:
        cur = cur[p]
    del cur[path[-1]]


def _mutate_doc(doc, rng: random.Random):
    doc = json.loads(json.dumps(doc))
    paths = [p for p, _ in _paths(doc) if p]
    kind = rng.randrange(9)
    if kind == 0 and paths:                      # a value of the wrong type
        _set(doc, rng.choice(paths), rng.choice(_ODD_VALUES))
    elif kind == 1:                              # a field goes missing
        cands = [p for p in paths if isinstance(p[-1], str)]
        if cands:
            _del(doc, rng.choice(cands))
    elif kind == 2:                              # an unknown field appears
        objs = [p for p, v in _paths(doc) if isinstance(v, dict)]
        tgt = rng.choice(objs)
        cur = doc
        for p in tgt:
            cur = cur[p]
        cur[rng.choice(("extra", "zz", "a"))] = rng.choice(_ODD_VALUES)
    elif kind == 3:                              # an unknown enum word
        cands = [p for p in paths if p[-1] in ("direction", "type", "kernel_id")]
        if cands:
            _set(doc, rng.choice(cands), rng.choice(("INPUT", "u8", "f16", "", "inout ", "output")))
    elif kind == 4:                              # float literal edge values
        cands = [p for p in paths if p[-1] == "value"]
        if cands:
            p = rng.choice(cands)
            _set(doc, p[:-1] + ("type",), rng.choice(("f32", "f64", "i32", "i64")))
            _set(doc, p, rng.choice(_FLOATS))
    elif kind == 5:                              # store key edge cases
        cands = [p for p in paths if p[-1] == "key"]
        if cands:
            _set(doc, rng.choice(cands), rng.choice(_ODD_KEYS))
    elif kind == 6:                              # integers at / past the ranges
        cands = [p for p, v in _paths(doc) if p and type(v) is int]
        if cands:
            _set(doc, rng.choice(cands), rng.choice((0, -1, 1 << 31, (1 << 31) - 1, 1 << 32,
                                                     (1 << 63) - 1, 1 << 63, -(1 << 63), 1 << 70)))
    elif kind == 7:                              # a container replaced wholesale
        cands = [p for p, v in _paths(doc) if p and isinstance(v, (list, dict))]
        if cands:
            _set(doc, rng.choice(cands), rng.choice(([], {}, "[]", None, [[]], [{}])))
    else:                                        # nothing: the document as is
        pass
    return doc


def mutations(body: bytes, seed: int, count: int = 4):
    """``count`` variants of one encoded request (bytes, or a non-bytes
    value for the type check)."""
    rng = random.Random(seed)
    doc = json.loads(body)
    out = []
    for _ in range(count):
        roll = rng.random()
        if roll < 0.06:                          # byte-level damage
            cut = rng.randrange(max(1, len(body)))
            out.append(rng.choice((body[:cut], body[:cut] + b"\xff" + body[cut:],
                                   body + b"x", b"", b"[]", b"null", b'"s"')))
        elif roll < 0.07:
            out.append(body.decode("utf-8"))      # str, not bytes: ParseError
        else:
            out.append(json.dumps(_mutate_doc(doc, rng)).encode())
    return out


_KINDS = ("InvalidRequest", "UnknownKernel", "ArityMismatch", "NotFound", "SizeMismatch",
          "OutOfDeviceMemory", "BufferBusy", "BackendFault", "Internal")


def response_docs(seed: int):
    """A well-formed wire response and three mutations of it."""
    rng = random.Random(seed)
    ok = rng.random() < 0.6
    doc = {"request_id": f"r{seed}", "status": "ok" if ok else "error"}
    if not ok:
        doc["error"] = {"kind": rng.choice(_KINDS + ("Nope",)), "message": "m"}
    doc["per_invocation"] = [{"kernel_id": rng.choice(("fill", "matmul")),
                              "simulated_compute_time": rng.randrange(1 << 20),
                              "launch_overhead": 10000} for _ in range(rng.randrange(3))]
    doc["io_stats"] = {n: rng.randrange(100) for n in (
        "store_gets", "store_puts", "bytes_fetched", "bytes_flushed", "cache_hits",
        "cache_misses")}
    doc["simulated_total_time"] = rng.randrange(1 << 30)
    if ok and rng.random() < 0.1:
        doc["error"] = {"kind": "Internal", "message": ""}
    base = json.dumps(doc).encode()
    out = [base]
    for _ in range(3):
        if rng.random() < 0.15:
            out.append(json.dumps(_mutate_doc(doc, rng)).encode().replace(b'"ok"', b'"error"'))
        else:
            out.append(json.dumps(_mutate_doc(doc, rng)).encode())
    return out


STORE_KEYS = ("k", "k\n", "k\n\n", "\nk", "k\r", "k\r\n", "a b", "A.z/0-9_", "k" * 256,
              "k" * 256 + "\n", "k" * 257, "", "é", "k\x00", "-", ".", "/", "k\t", "K\n")

LITERAL_VALUES = (0.0, -0.0, float("nan"), -float("nan"), float("inf"), -float("inf"), 1.0, 1,
                  True, 0, -1, 2.5)


def outcome(fn, *args):
    """(status, detail) of one call: the exception's class name and message,
    or ``('ok', value)``."""
    try:
        return ("ok", fn(*args))
    except Exception as exc:  # noqa: BLE001 -- every exception kind is compared
        return (type(exc).__name__, str(exc))
