"""Shared test helpers: golden fixtures, canonical hashing, stream replay."""

from __future__ import annotations

import gzip
import hashlib
import json
import os

import numpy as np

from paper_2212_08146_b200.api import request_from_doc, response_to_doc

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def load_golden(name: str):
    with gzip.open(os.path.join(GOLDEN, name), "rt", encoding="utf-8") as fh:
        return json.load(fh)


def canon(data) -> bytes:
    """Bytes with every f32-NaN word replaced by the canonical quiet NaN.

    IEEE 754 leaves NaN payload propagation open and numpy's x86 SIMD/tail
    loops pick payloads by element position, so 'bit-exact' is defined on
    every non-NaN word and NaN-for-NaN elsewhere."""
    data = bytes(data)
    if len(data) % 4 == 0 and data:
        w = np.frombuffer(data, dtype="<u4").copy()
        nan = ((w & 0x7F800000) == 0x7F800000) & ((w & 0x007FFFFF) != 0)
        w[nan] = 0x7FC00000
        data = w.tobytes()
    return data


def canon_hash(data) -> str:
    return hashlib.sha256(canon(data)).hexdigest()


def cache_digest(items) -> str:
    """items: iterable of (key, size, last_use, pinned, dirty)."""
    return hashlib.sha256(json.dumps(sorted(list(i) for i in items)).encode()).hexdigest()


def replay(stream: dict, make_executor, limit: int | None = None):
    """Run a golden executor stream through ``make_executor(store_objects)``.

    ``make_executor`` returns (executor, store, snapshot_fn, removed_list).
    Yields (step_index, golden_step, response_doc, cache_digest, removed, writes)."""
    initial = {k: bytes.fromhex(v) for k, v in stream["initial_store"].items()}
    ex, store, snap, removed = make_executor(initial)
    for i, step in enumerate(stream["steps"]):
        if limit is not None and i >= limit:
            break
        req = request_from_doc(step["request"])
        before = {k: store.get(k) for k in store.keys()}
        removed.clear()
        resp = ex.execute(req)
        writes = {}
        for k in store.keys():
            v = store.get(k)
            if k not in before or before[k] is not v:
                writes[k] = canon_hash(v)
        yield i, step, response_to_doc(resp), cache_digest(snap()), list(removed), writes
