"""Oracle placement policies -- TEST INFRASTRUCTURE ONLY.

Restates ``pkg/src/kaas/router.py:19-159`` (random / round-robin / affinity,
LRU-capped digests, depth accounting) and defines the two policies the
north star adds (``static``, ``exclusive``) as plain functions of the same
state, so the product router can be checked decision by decision.
"""

from __future__ import annotations

import random
import zlib
from collections import OrderedDict


class OracleRouter:
    def __init__(self, ids, spec: str, digest_cap: int = 1024):
        self.ids = sorted(ids)
        self.spec = spec
        self.cap = digest_cap
        self.keys = {e: OrderedDict() for e in self.ids}
        self.depth = {e: 0 for e in self.ids}
        self._rr = 0
        self._rng = random.Random(int(spec.split(":", 1)[1])) if spec.startswith("random:") else None
        self._tenants: dict[str, int] = {}

    def _bytes(self, e):
        return sum(self.keys[e].values())

    def pick(self, req) -> int:
        ids = self.ids
        s = self.spec
        if s in ("rr", "round_robin"):
            e = ids[self._rr % len(ids)]
            self._rr += 1
            return e
        if s.startswith("random:"):
            return ids[self._rng.randrange(len(ids))]
        if s.startswith("affinity:"):
            q_max = int(s.split(":", 1)[1])
            want = {b.key for b in req.buffers if b.is_const and b.key is not None}

            def score(e):
                d = self.keys[e]
                return sum(d[k] for k in want if k in d)

            best = min(ids, key=lambda e: (-score(e), self.depth[e], self._bytes(e), e))
            if self.depth[best] > q_max:
                best = min(ids, key=lambda e: (self.depth[e], e))
            return best
        if s == "static":
            consts = {b.key for b in req.buffers if b.is_const and b.key is not None}
            if any(not isinstance(k, str) for k in consts):
                return ids[0]  # malformed request: routed anywhere fixed, rejected in band
            token = "\x00".join(sorted(consts)) if consts else req.request_id
            if not isinstance(token, str):
                return ids[0]
            return ids[zlib.crc32(token.encode("utf-8", "surrogatepass")) % len(ids)]
        if s == "exclusive":
            if not isinstance(req.request_id, str):
                return ids[0]
            tenant = req.request_id.split("/", 1)[0]
            if tenant not in self._tenants:
                self._tenants[tenant] = ids[len(self._tenants) % len(ids)]
            return self._tenants[tenant]
        raise ValueError(s)

    def route(self, req) -> int:
        e = self.pick(req)
        self.depth[e] += 1
        return e

    def complete(self, e, ok: bool, req) -> None:
        self.depth[e] -= 1
        if not ok:
            return
        d = self.keys[e]
        for b in req.buffers:
            if b.key is None:
                continue
            if b.is_const or b.direction in ("output", "inout"):
                d[b.key] = b.size
                d.move_to_end(b.key)
        while len(d) > self.cap:
            d.popitem(last=False)
