"""Seeded request-stream generator for GPU-vs-oracle parity (independent of
the reference's genreq; covers the new cgemm / jacobi_sweep kernels too).

Keys encode their payload type so data can be compared per key:
  ``f/...`` f32 data compared bit-exactly (NaN-canonical)
  ``c/...`` cgemm outputs, compared to the oracle within rel. Frobenius 1e-4
  ``j/...`` jacobi outputs, compared within 1e-5 max abs
"""

from __future__ import annotations

import random

import numpy as np

from paper_2212_08146_b200.api import (
    BufferArg,
    KaasRequest,
    KernelInvocation,
    LaunchDims,
    ScalarLiteral,
    f32,
    i32,
)


def grid(cells: int, rng: random.Random) -> LaunchDims:
    cells = max(1, cells)
    style = rng.random()
    if style < 0.15:  # short grid: partial coverage
        return LaunchDims(grid_x=max(1, cells - rng.randint(0, cells - 1)))
    if style < 0.3:
        return LaunchDims(grid_x=cells + rng.randint(0, 17))
    b = rng.choice((1, 32, 64, 128))
    return LaunchDims(grid_x=-(-cells // b), block_x=b)


def seed_store(store, rng: random.Random, nprng: np.random.Generator, n_keys: int = 10):
    """f32 vectors of assorted sizes plus a few complex matrices and a
    diagonally dominant system."""
    pool = []
    for i in range(n_keys):
        n = rng.choice((4, 16, 64, 256, 1024, 4096))
        data = (nprng.standard_normal(n) * 10).astype("<f4")
        if rng.random() < 0.2:  # specials
            data[rng.randrange(n)] = rng.choice((np.inf, -np.inf, np.nan, -0.0))
        key = f"f/in{i}"
        store.put(key, data.tobytes())
        pool.append((key, 4 * n))
    return pool


def make_stream(seed: int, count: int, store, with_new_kernels: bool = True):
    rng = random.Random(seed)
    nprng = np.random.default_rng(seed)
    pool = seed_store(store, rng, nprng)
    # complex operands and jacobi systems
    mats = {}
    for (n, k) in ((8, 8), (16, 24), (33, 17), (64, 64)):
        a = (nprng.standard_normal((n, k)) + 1j * nprng.standard_normal((n, k))).astype("<c8")
        store.put(f"c/A{n}x{k}", a.tobytes())
        mats[(n, k)] = f"c/A{n}x{k}"
    systems = {}
    for n in (12, 33, 64, 128):
        A = nprng.random((n, n)).astype("<f4")
        A[np.arange(n), np.arange(n)] = A.sum(1) + 1
        b = (A.astype(np.float64) @ np.ones(n)).astype("<f4")
        store.put(f"j/A{n}", A.tobytes())
        store.put(f"j/b{n}", b.tobytes())
        store.put(f"j/x0_{n}", np.zeros(n, "<f4").tobytes())
        systems[n] = n
    reqs = []
    for ident in range(count):
        reqs.append(_one(rng, pool, mats, systems, ident, with_new_kernels))
    return reqs


def _in(rng, name, key, size):
    const = rng.random() < 0.6
    return BufferArg(name, size, "input" if const else rng.choice(("input", "inout")), key=key,
                     is_const=const)


def _one(rng, pool, mats, systems, ident, new):
    kinds = ["vadd", "saxpy", "fill", "reduce", "matmul", "alias"]
    if new:
        kinds += ["cgemm", "cgemm", "jacobi", "jacobi"]
    kind = rng.choice(kinds)
    rid = f"t{ident % 3}/q{ident:05d}"
    out_key = f"f/out{ident:05d}"
    k1, s1 = rng.choice(pool)
    n1 = s1 // 4
    if kind == "vadd":
        k2 = next((k for k, s in rng.sample(pool, len(pool)) if s == s1), k1)
        out = (BufferArg("o", s1, "output", is_ephemeral=True) if rng.random() < 0.3
               else BufferArg("o", s1, "output", key=out_key))
        req = KaasRequest(rid, (_in(rng, "x", k1, s1), _in(rng, "y", k2, s1), out),
                          (KernelInvocation("vector_add", grid(n1, rng), (i32(n1),), ("x", "y", "o")),))
    elif kind == "saxpy":
        req = KaasRequest(rid, (_in(rng, "x", k1, s1), BufferArg("o", s1, "output", key=out_key)),
                          (KernelInvocation("saxpy", grid(n1, rng), (i32(n1), f32(rng.uniform(-3, 3))),
                                            ("x", "x", "o")),))
    elif kind == "fill":
        n = rng.choice((1, 7, 64, 1000))
        req = KaasRequest(rid, (BufferArg("o", 4 * n, "output", key=out_key),),
                          (KernelInvocation("fill", grid(n, rng), (i32(n), f32(rng.uniform(-9, 9))), ("o",)),))
    elif kind == "reduce":
        req = KaasRequest(rid, (_in(rng, "x", k1, s1), BufferArg("r", 4, "output", key=out_key)),
                          (KernelInvocation("reduce_sum", LaunchDims(), (i32(n1),), ("x", "r")),))
    elif kind == "matmul":
        d = rng.randint(1, 24)
        e = rng.randint(1, 24)
        req = KaasRequest(rid, (
            BufferArg("a", 4 * d * e, "inout", is_ephemeral=True),
            BufferArg("b", 4 * e * d, "inout", is_ephemeral=True),
            BufferArg("o", 4 * d * d, "output", key=out_key)), (
            KernelInvocation("fill", grid(d * e, rng), (i32(d * e), f32(1.25)), ("a",)),
            KernelInvocation("fill", grid(d * e, rng), (i32(d * e), f32(-0.5)), ("b",)),
            KernelInvocation("matmul", grid(d * d, rng), (i32(d), i32(d), i32(e)), ("a", "b", "o"))))
    elif kind == "alias":  # matmul(C, C, C): output aliases both inputs
        d = rng.choice((2, 4, 8))
        if s1 >= 4 * d * d:
            req = KaasRequest(rid, (_in(rng, "x", k1, s1), BufferArg("c", s1, "output", key=out_key)), (
                KernelInvocation("vector_add", grid(n1, rng), (i32(n1),), ("x", "x", "c")),
                KernelInvocation("matmul", grid(d * d, rng), (i32(d), i32(d), i32(d)), ("c", "c", "c"))))
        else:
            req = KaasRequest(rid, (BufferArg("o", 4, "output", key=out_key),),
                              (KernelInvocation("fill", LaunchDims(), (i32(1), f32(2.0)), ("o",)),))
    elif kind == "cgemm":
        (n, k) = rng.choice(list(mats))
        m = rng.choice((1, 5, 16, 40))
        breq = rng.random()
        out = BufferArg("C", 8 * n * m, "output", key=f"c/out{ident:05d}")
        bufs = [BufferArg("A", 8 * n * k, "input", key=mats[(n, k)], is_const=True),
                BufferArg("B", 8 * k * m, "inout", is_ephemeral=True), out]
        invs = [KernelInvocation("fill", grid(2 * k * m, rng), (i32(2 * k * m), f32(0.5 if breq < 0.5 else -1.5)), ("B",)),
                KernelInvocation("cgemm", grid(n * m, rng), (i32(n), i32(m), i32(k)), ("A", "B", "C"))]
        req = KaasRequest(rid, tuple(bufs), tuple(invs))
    else:  # jacobi
        n = rng.choice(list(systems))
        sweeps = rng.randint(1, 7)
        invs = []
        for s in range(sweeps):
            src = "x0" if s == 0 else ("e1" if s % 2 == 1 else "e2")
            dst = "x" if s == sweeps - 1 else ("e1" if s % 2 == 0 else "e2")
            invs.append(KernelInvocation("jacobi_sweep", grid(n, rng) if rng.random() < 0.3
                                         else LaunchDims(grid_x=n), (i32(n),), ("A", "b", src, dst, "r")))
        req = KaasRequest(rid, (
            BufferArg("A", 4 * n * n, "input", key=f"j/A{n}", is_const=True),
            BufferArg("b", 4 * n, "input", key=f"j/b{n}", is_const=True),
            BufferArg("x0", 4 * n, "input", key=f"j/x0_{n}"),
            BufferArg("e1", 4 * n, "inout", is_ephemeral=True),
            BufferArg("e2", 4 * n, "inout", is_ephemeral=True),
            BufferArg("x", 4 * n, "output", key=f"j/x{ident:05d}"),
            BufferArg("r", 4, "output", key=f"j/r{ident:05d}")), tuple(invs))
    # targeted faults
    if rng.random() < 0.25:
        fault = rng.choice(("missing", "bounds", "unknown", "arity", "oom", "size"))
        b0 = req.buffers[0]
        inv0 = req.invocations[0]
        if fault == "missing" and b0.key is not None:
            req = KaasRequest(rid, (BufferArg(b0.name, b0.size, b0.direction, key=f"f/missing{ident}",
                                              is_const=b0.is_const),) + req.buffers[1:], req.invocations)
        elif fault == "size" and b0.key is not None:
            req = KaasRequest(rid, (BufferArg(b0.name, b0.size + 4, b0.direction, key=b0.key,
                                              is_const=b0.is_const),) + req.buffers[1:], req.invocations)
        elif fault == "bounds":
            lits = tuple(ScalarLiteral("i32", 1 << 20) if j == 0 else l for j, l in enumerate(inv0.literals))
            req = KaasRequest(rid, req.buffers, (KernelInvocation(inv0.kernel_id, inv0.dims, lits, inv0.args),)
                              + req.invocations[1:])
        elif fault == "unknown":
            req = KaasRequest(rid, req.buffers, (KernelInvocation("nope", inv0.dims, inv0.literals, inv0.args),)
                              + req.invocations[1:])
        elif fault == "arity":
            req = KaasRequest(rid, req.buffers, (KernelInvocation(inv0.kernel_id, inv0.dims,
                                                                  inv0.literals + (i32(1),), inv0.args),)
                              + req.invocations[1:])
        elif fault == "oom":
            req = KaasRequest(rid, req.buffers + (BufferArg("hog", 3 << 20, "inout", is_ephemeral=True),),
                              req.invocations + (KernelInvocation("fill", LaunchDims(), (i32(1), f32(0.0)), ("hog",)),))
    return req
