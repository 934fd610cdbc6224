"""The KaaS request API, unchanged from the reference.

A ``KaasRequest`` is a buffer table (``BufferArg``: named, sized, keyed by
object-store names; input / output / inout, const or ephemeral) plus an
ordered list of ``KernelInvocation``s over that namespace.  The GPU executor
accepts exactly these values, so clients of the reference executor switch
without change.

Reference: ``pkg/src/kaas/protocol.py`` -- types ``54-202``,
``validate_request`` ``209-281``, wire format ``292-567``.  Field names,
defaults, equality (NaN-equal literals, ``protocol.py:80-89``),
``referenced_buffers`` order (``150-157``) and the violation messages are
kept identical because they are observable in responses.
"""

from __future__ import annotations

import json
import math
import re
from dataclasses import dataclass, field
from functools import cached_property

from .faults import WIRE_ERROR_KINDS

MAX_TOTAL_THREADS = 1 << 32
I32_RANGE = (-(1 << 31), (1 << 31) - 1)
I64_RANGE = (-(1 << 63), (1 << 63) - 1)
STORE_KEY_MAX_LEN = 256
DIRECTIONS = ("input", "output", "inout")
LITERAL_TYPES = ("i32", "i64", "f32", "f64")
# ``protocol.py:24``: anchored with ``^...$`` and applied with ``re.match``,
# so -- as in the reference -- one trailing newline is accepted ("k\n").
_KEY_CHARS = re.compile(r"^[A-Za-z0-9._/-]+$")


def valid_store_key(key) -> bool:
    """``protocol.py:42-47``: 1..256 chars of ``[A-Za-z0-9._/-]`` under the
    reference's exact regex semantics (``$`` also matches before a final
    newline)."""
    return (isinstance(key, str) and 0 < len(key) <= STORE_KEY_MAX_LEN
            and _KEY_CHARS.match(key) is not None)


# ---------------------------------------------------------------------------
# value types


@dataclass(frozen=True)
class LaunchDims:
    grid_x: int = 1
    grid_y: int = 1
    grid_z: int = 1
    block_x: int = 1
    block_y: int = 1
    block_z: int = 1

    def as_tuple(self) -> tuple[int, int, int, int, int, int]:
        return (self.grid_x, self.grid_y, self.grid_z,
                self.block_x, self.block_y, self.block_z)

    @property
    def total_threads(self) -> int:
        n = 1
        for c in self.as_tuple():
            n *= c
        return n


@dataclass(frozen=True, eq=False)
class ScalarLiteral:
    """Tagged scalar kernel argument; NaN payloads compare equal.

    Equality is the reference's (``protocol.py:80-89``): values of the same
    Python type compare with ``==`` (so ``0.0 == -0.0``), NaN equals NaN.
    The sign of zero still reaches the kernel: the executor's plan key and
    the codec's intern key carry float bits (``gpu_executor._plan_key``)."""

    type: str
    value: int | float

    def __eq__(self, other):
        if not isinstance(other, ScalarLiteral):
            return NotImplemented
        if self.type != other.type:
            return False
        a, b = self.value, other.value
        if isinstance(a, float) and isinstance(b, float) and math.isnan(a) and math.isnan(b):
            return True
        return type(a) is type(b) and a == b

    def __hash__(self):
        return hash(self.type)


def i32(v) -> ScalarLiteral:
    return ScalarLiteral("i32", int(v))


def i64(v) -> ScalarLiteral:
    return ScalarLiteral("i64", int(v))


def f32(v) -> ScalarLiteral:
    return ScalarLiteral("f32", float(v))


def f64(v) -> ScalarLiteral:
    return ScalarLiteral("f64", float(v))


@dataclass(frozen=True)
class BufferArg:
    name: str
    size: int
    direction: str = "input"
    key: str | None = None
    is_const: bool = False
    is_ephemeral: bool = False


@dataclass(frozen=True)
class KernelInvocation:
    kernel_id: str
    dims: LaunchDims
    literals: tuple[ScalarLiteral, ...] = ()
    args: tuple[str, ...] = ()


@dataclass(frozen=True)
class KaasRequest:
    request_id: str
    buffers: tuple[BufferArg, ...] = ()
    invocations: tuple[KernelInvocation, ...] = ()

    @cached_property
    def by_name(self) -> dict[str, BufferArg]:
        return {b.name: b for b in self.buffers}

    def referenced_buffers(self) -> tuple[BufferArg, ...]:
        """Buffers some invocation names, in buffer-table order: the
        executor's resolution and flush order (``protocol.py:150-157``)."""
        used = set()
        for inv in self.invocations:
            used.update(inv.args)
        return tuple(b for b in self.buffers if b.name in used)


@dataclass(frozen=True)
class IoStats:
    store_gets: int = 0
    store_puts: int = 0
    bytes_fetched: int = 0
    bytes_flushed: int = 0
    cache_hits: int = 0
    cache_misses: int = 0


@dataclass(frozen=True)
class InvocationStats:
    kernel_id: str
    simulated_compute_time: int
    launch_overhead: int


@dataclass(frozen=True)
class Status:
    code: str
    error_kind: str | None = None
    error_message: str | None = None

    @property
    def ok(self) -> bool:
        return self.code == "ok"

    @staticmethod
    def make_ok() -> "Status":
        return Status("ok")

    @staticmethod
    def make_error(kind: str, message: str) -> "Status":
        return Status("error", kind, message)


@dataclass(frozen=True)
class KaasResponse:
    request_id: str
    status: Status
    per_invocation: tuple[InvocationStats, ...] = ()
    io_stats: IoStats = field(default_factory=IoStats)
    simulated_total_time: int = 0


# ---------------------------------------------------------------------------
# validation (protocol.py:209-281)


def _is_int(v) -> bool:
    return isinstance(v, int) and not isinstance(v, bool)


def _buffer_problems(b: BufferArg, label: str):
    if not _is_int(b.size) or b.size < 1:
        yield f"{label}: size must be a positive integer"
    if b.direction not in DIRECTIONS:
        yield f'{label}: unknown direction "{b.direction}"'
    if b.is_const and b.is_ephemeral:
        yield f"{label}: const and ephemeral are mutually exclusive"
    if b.is_const and b.direction != "input":
        yield f"{label}: const buffers must have direction input"
    if b.is_ephemeral:
        if b.key is not None:
            yield f"{label}: ephemeral buffers must not carry a store key"
    elif b.key is None:
        yield f"{label}: non-ephemeral buffers require a store key"
    elif not valid_store_key(b.key):
        yield f'{label}: invalid store key "{b.key}"'


def _literal_problem(lit: ScalarLiteral, label: str):
    if lit.type not in LITERAL_TYPES:
        return f'{label} has unknown type "{lit.type}"'
    if lit.type in ("f32", "f64"):
        return None if isinstance(lit.value, float) else f"{label} ({lit.type}) must be a float"
    if not _is_int(lit.value):
        return f"{label} ({lit.type}) must be an integer"
    lo, hi = I32_RANGE if lit.type == "i32" else I64_RANGE
    if not lo <= lit.value <= hi:
        return f"{label} out of {lit.type} range"
    return None


def _invocation_problems(idx: int, inv: KernelInvocation, names):
    label = f"invocation {idx}"
    if not isinstance(inv.kernel_id, str) or not inv.kernel_id:
        yield f"{label}: kernel_id must be a non-empty string"
    comps = inv.dims.as_tuple()
    if not all(_is_int(c) and c >= 1 for c in comps):
        yield f"{label}: launch dims must all be >= 1"
    else:
        total = inv.dims.total_threads
        if total > MAX_TOTAL_THREADS:
            yield f"{label}: total threads {total} exceeds 2^32"
    for li, lit in enumerate(inv.literals):
        msg = _literal_problem(lit, f"{label}: literal {li}")
        if msg is not None:
            yield msg
    for name in inv.args:
        if name not in names:
            yield f'{label}: unknown buffer "{name}"'


def validate_request(req: KaasRequest) -> list[str]:
    """All invariant violations of ``req`` (empty list = acceptable)."""
    problems: list[str] = []
    if not isinstance(req.request_id, str) or not req.request_id:
        problems.append("request_id must be a non-empty string")

    names: set[str] = set()
    bindings: dict[str, list[BufferArg]] = {}
    for b in req.buffers:
        if not isinstance(b.name, str) or not b.name:
            problems.append("buffer name must be a non-empty string")
            continue
        label = f'buffer "{b.name}"'
        if b.name in names:
            problems.append(f"{label}: duplicate buffer name")
            continue
        names.add(b.name)
        own = list(_buffer_problems(b, label))
        problems.extend(own)
        if (not b.is_ephemeral and b.key is not None and valid_store_key(b.key)):
            bindings.setdefault(b.key, []).append(b)

    # One key bound by several buffers is only unambiguous when all are const.
    for key, owners in bindings.items():
        if len(owners) > 1 and not all(o.is_const for o in owners):
            problems.append(f'store key "{key}" bound by non-const buffers '
                            f'({", ".join(o.name for o in owners)})')

    by_name = req.by_name
    for idx, inv in enumerate(req.invocations):
        problems.extend(_invocation_problems(idx, inv, by_name))
    return problems


# ---------------------------------------------------------------------------
# wire format (protocol.py:292-567): canonical compact JSON, NaN/Inf as words


class ProtocolError(Exception):
    pass


class ParseError(ProtocolError):
    pass


class SchemaError(ProtocolError):
    pass


_WORDS = {"NaN": math.nan, "Infinity": math.inf, "-Infinity": -math.inf}


def _word(v: float):
    if math.isnan(v):
        return "NaN"
    if math.isinf(v):
        return "Infinity" if v > 0 else "-Infinity"
    return v


_DIM_NAMES = ("grid_x", "grid_y", "grid_z", "block_x", "block_y", "block_z")


def request_to_doc(req: KaasRequest) -> dict:
    return {
        "request_id": req.request_id,
        "buffers": [{"name": b.name, "key": b.key, "size": b.size,
                     "is_const": b.is_const, "is_ephemeral": b.is_ephemeral,
                     "direction": b.direction} for b in req.buffers],
        "invocations": [{
            "kernel_id": inv.kernel_id,
            "dims": dict(zip(_DIM_NAMES, inv.dims.as_tuple())),
            "literals": [{"type": l.type,
                          "value": _word(l.value) if l.type in ("f32", "f64")
                          and isinstance(l.value, float) else l.value}
                         for l in inv.literals],
            "args": list(inv.args)} for inv in req.invocations],
    }


def encode_request(req: KaasRequest) -> bytes:
    return json.dumps(request_to_doc(req), separators=(",", ":"),
                      allow_nan=False).encode("utf-8")


def response_to_doc(resp: KaasResponse) -> dict:
    doc: dict = {"request_id": resp.request_id, "status": resp.status.code}
    if not resp.status.ok:
        doc["error"] = {"kind": resp.status.error_kind,
                        "message": resp.status.error_message or ""}
    doc["per_invocation"] = [{"kernel_id": s.kernel_id,
                              "simulated_compute_time": s.simulated_compute_time,
                              "launch_overhead": s.launch_overhead}
                             for s in resp.per_invocation]
    st = resp.io_stats
    doc["io_stats"] = {n: getattr(st, n) for n in (
        "store_gets", "store_puts", "bytes_fetched", "bytes_flushed",
        "cache_hits", "cache_misses")}
    doc["simulated_total_time"] = resp.simulated_total_time
    return doc


def encode_response(resp: KaasResponse) -> bytes:
    return json.dumps(response_to_doc(resp), separators=(",", ":"),
                      allow_nan=False).encode("utf-8")


# Checked decoder.  The order of the checks and every error message follow
# ``protocol.py:390-511`` exactly (the first failing check names the error a
# client sees, so both are part of the drop-in contract).


def _kind(v) -> str:
    return type(v).__name__


def _obj(v, ctx):
    if not isinstance(v, dict):
        raise SchemaError(f"{ctx}: expected object, got {_kind(v)}")
    return v


def _arr(v, ctx):
    if not isinstance(v, list):
        raise SchemaError(f"{ctx}: expected array, got {_kind(v)}")
    return v


def _str(v, ctx):
    if not isinstance(v, str):
        raise SchemaError(f"{ctx}: expected string, got {_kind(v)}")
    return v


def _int(v, ctx):
    if not _is_int(v):
        raise SchemaError(f"{ctx}: expected integer, got {_kind(v)}")
    return v


def _bool(v, ctx):
    if not isinstance(v, bool):
        raise SchemaError(f"{ctx}: expected boolean, got {_kind(v)}")
    return v


def _fld(o, name, ctx):
    if name not in o:
        raise SchemaError(f"{ctx}: missing field {name!r}")
    return o[name]


def _only(o, allowed, ctx, strict):
    if strict:
        extra = set(o) - set(allowed)
        if extra:
            raise SchemaError(f"{ctx}: unknown fields {sorted(extra)}")


def _loads(data):
    if not isinstance(data, (bytes, bytearray)):
        raise ParseError("input must be a byte sequence")
    try:
        text = bytes(data).decode("utf-8")
    except UnicodeDecodeError as exc:
        raise ParseError(f"invalid UTF-8: {exc}") from None
    try:
        return json.loads(text)
    except json.JSONDecodeError as exc:
        raise ParseError(f"malformed JSON: {exc}") from None


_BUF_FIELDS = ("name", "key", "size", "is_const", "is_ephemeral", "direction")
_INV_FIELDS = ("kernel_id", "dims", "literals", "args")


def _literal_from_doc(v, ctx, strict) -> ScalarLiteral:
    o = _obj(v, ctx)
    _only(o, ("type", "value"), ctx, strict)
    tag = _str(_fld(o, "type", ctx), f"{ctx}.type")
    if tag not in LITERAL_TYPES:
        raise SchemaError(f'{ctx}: unknown literal type "{tag}"')
    val = _fld(o, "value", ctx)
    if tag in ("i32", "i64"):
        return ScalarLiteral(tag, _int(val, f"{ctx}.value"))
    if isinstance(val, str):
        if val not in _WORDS:
            raise SchemaError(f'{ctx}: bad float word "{val}"')
        return ScalarLiteral(tag, _WORDS[val])
    if isinstance(val, bool) or not isinstance(val, (int, float)):
        raise SchemaError(f"{ctx}.value: expected number")
    return ScalarLiteral(tag, float(val))


def _dims_from_doc(v, ctx, strict) -> LaunchDims:
    o = _obj(v, ctx)
    _only(o, _DIM_NAMES, ctx, strict)
    return LaunchDims(*[_int(_fld(o, n, ctx), f"{ctx}.{n}") for n in _DIM_NAMES])


def request_from_doc(top, strict: bool = False) -> KaasRequest:
    top = _obj(top, "request")
    _only(top, ("request_id", "buffers", "invocations"), "request", strict)
    rid = _str(_fld(top, "request_id", "request"), "request_id")
    bufs = []
    for i, raw in enumerate(_arr(_fld(top, "buffers", "request"), "buffers")):
        ctx = f"buffers[{i}]"
        o = _obj(raw, ctx)
        _only(o, _BUF_FIELDS, ctx, strict)
        key = o.get("key")
        if key is not None:
            _str(key, f"{ctx}.key")
        direction = _str(_fld(o, "direction", ctx), f"{ctx}.direction")
        if direction not in DIRECTIONS:
            raise SchemaError(f'{ctx}: unknown direction "{direction}"')
        name = _str(_fld(o, "name", ctx), f"{ctx}.name")
        size = _int(_fld(o, "size", ctx), f"{ctx}.size")
        is_const = _bool(_fld(o, "is_const", ctx), f"{ctx}.is_const")
        is_eph = _bool(_fld(o, "is_ephemeral", ctx), f"{ctx}.is_ephemeral")
        bufs.append(BufferArg(name, size, direction, key, is_const, is_eph))
    invs = []
    for i, raw in enumerate(_arr(_fld(top, "invocations", "request"), "invocations")):
        ctx = f"invocations[{i}]"
        o = _obj(raw, ctx)
        _only(o, _INV_FIELDS, ctx, strict)
        lits = tuple(_literal_from_doc(l, f"{ctx}.literals[{j}]", strict)
                     for j, l in enumerate(_arr(_fld(o, "literals", ctx), ctx)))
        args = tuple(_str(a, f"{ctx}.args[{j}]")
                     for j, a in enumerate(_arr(_fld(o, "args", ctx), ctx)))
        kid = _str(_fld(o, "kernel_id", ctx), f"{ctx}.kernel_id")
        dims = _dims_from_doc(_fld(o, "dims", ctx), f"{ctx}.dims", strict)
        invs.append(KernelInvocation(kid, dims, lits, args))
    return KaasRequest(rid, tuple(bufs), tuple(invs))


# -- decode fast path ----------------------------------------------------------
# Most requests are kernel graphs a client resends (a 500-sweep Jacobi request
# is ~90 KB of JSON).  The fast path checks the same structure with exact type
# tests (bool and float never pass for int), interns each invocation by an
# exact key (floats by their bits) and the whole buffer / invocation tuples,
# so a resent graph decodes to the *same* tuples and the executor's plan cache
# hits by identity.  Anything unusual falls back to request_from_doc, which
# produces the reference's exact error.

_INTERN_CAP = 4096
_inv_cache: dict = {}
_invs_cache: dict = {}
_bufs_cache: dict = {}
_INT_TAGS = ("i32", "i64")
_FLOAT_TAGS = ("f32", "f64")


def _intern(cache: dict, key, make):
    v = cache.get(key)
    if v is None:
        if len(cache) >= _INTERN_CAP:
            cache.clear()
        v = cache[key] = make()
    return v


def _fast_invocations(raw, strict: bool):
    if type(raw) is not list:
        return None
    keys = []
    for o in raw:
        if type(o) is not dict or (strict and len(o) != 4):
            return None
        try:
            kid, d, lits, args = o["kernel_id"], o["dims"], o["literals"], o["args"]
            if type(d) is not dict or (strict and len(d) != 6):
                return None
            dv = (d["grid_x"], d["grid_y"], d["grid_z"], d["block_x"], d["block_y"], d["block_z"])
        except KeyError:
            return None
        if type(kid) is not str or type(lits) is not list or type(args) is not list:
            return None
        for v in dv:
            if type(v) is not int:
                return None
        lk = []
        for lit in lits:
            if type(lit) is not dict or (strict and len(lit) != 2):
                return None
            try:
                tag, val = lit["type"], lit["value"]
            except KeyError:
                return None
            tv = type(val)
            if tag in _INT_TAGS:
                if tv is not int:
                    return None
                lk.append((tag, val))
            elif tag in _FLOAT_TAGS:
                if tv is float or tv is int:
                    lk.append((tag, float(val).hex()))
                elif tv is str and val in _WORDS:
                    lk.append((tag, val))
                else:
                    return None
            else:
                return None
        for a in args:
            if type(a) is not str:
                return None
        keys.append((kid, dv, tuple(lk), tuple(args)))
    return _intern(_invs_cache, tuple(keys),
                   lambda: tuple(_intern(_inv_cache, k, lambda k=k: _make_invocation(k))
                                 for k in keys))


def _make_invocation(key) -> KernelInvocation:
    kid, dv, lk, args = key
    lits = []
    for tag, v in lk:
        if tag in _INT_TAGS:
            lits.append(ScalarLiteral(tag, v))
        else:
            lits.append(ScalarLiteral(tag, _WORDS[v] if v in _WORDS else float.fromhex(v)))
    return KernelInvocation(kid, LaunchDims(*dv), tuple(lits), args)


def decode_request(data: bytes, strict: bool = False) -> KaasRequest:
    top = _loads(data)
    if type(top) is dict and (not strict or len(top) == 3):
        invs = _fast_invocations(top.get("invocations"), strict)
        if invs is not None:
            # buffers: few; decoded by the checked path, then interned
            full = request_from_doc({"request_id": top.get("request_id", _MISSING),
                                     "buffers": top.get("buffers", _MISSING),
                                     "invocations": []}, strict) \
                if "request_id" in top and "buffers" in top else None
            if full is not None:
                bufs = _intern(_bufs_cache, tuple(
                    (b.name, b.key, b.size, b.is_const, b.is_ephemeral, b.direction)
                    for b in full.buffers), lambda: full.buffers)
                return KaasRequest(full.request_id, bufs, invs)
    return request_from_doc(top, strict)


_MISSING = object()


def response_from_doc(top, strict: bool = False) -> KaasResponse:
    top = _obj(top, "response")
    _only(top, ("request_id", "status", "error", "per_invocation", "io_stats",
                "simulated_total_time"), "response", strict)
    rid = _str(_fld(top, "request_id", "response"), "request_id")
    code = _str(_fld(top, "status", "response"), "status")
    if code == "ok":
        status = Status.make_ok()
        if strict and "error" in top:
            raise SchemaError("response: unexpected error object on ok status")
    elif code == "error":
        e = _obj(_fld(top, "error", "response"), "error")
        _only(e, ("kind", "message"), "error", strict)
        kind = _str(_fld(e, "kind", "error"), "error.kind")
        if kind not in WIRE_ERROR_KINDS:
            raise SchemaError(f'error: unknown kind "{kind}"')
        status = Status.make_error(kind, _str(_fld(e, "message", "error"), "error.message"))
    else:
        raise SchemaError(f'response: unknown status "{code}"')
    per = []
    for i, raw in enumerate(_arr(_fld(top, "per_invocation", "response"), "per_invocation")):
        ctx = f"per_invocation[{i}]"
        o = _obj(raw, ctx)
        _only(o, ("kernel_id", "simulated_compute_time", "launch_overhead"), ctx, strict)
        kid = _str(_fld(o, "kernel_id", ctx), f"{ctx}.kernel_id")
        sct = _int(_fld(o, "simulated_compute_time", ctx), ctx)
        per.append(InvocationStats(kid, sct, _int(_fld(o, "launch_overhead", ctx), ctx)))
    names = ("store_gets", "store_puts", "bytes_fetched", "bytes_flushed",
             "cache_hits", "cache_misses")
    io = _obj(_fld(top, "io_stats", "response"), "io_stats")
    _only(io, names, "io_stats", strict)
    stats = IoStats(*[_int(_fld(io, n, "io_stats"), f"io_stats.{n}") for n in names])
    total = _int(_fld(top, "simulated_total_time", "response"), "simulated_total_time")
    return KaasResponse(rid, status, tuple(per), stats, total)


def decode_response(data: bytes, strict: bool = False) -> KaasResponse:
    return response_from_doc(_loads(data), strict)
