"""Oracle kernels (numpy) -- TEST INFRASTRUCTURE ONLY.

Builtins restate ``pkg/src/kaas/backend.py:137-211`` operation for operation
(same numpy ufunc calls, same operand order), so on the same machine they are
bit-identical to the reference, NaN payloads included.  ``cgemm`` and
``jacobi_sweep`` define the two new kernels' semantics (complex128 truth for
cgemm; f32 BLAS products with a float64 update for Jacobi).

Every kernel takes ``(dims, literals, views)`` with ``views`` = list of
``np.uint8`` arrays and returns the FMA count, like a reference
``BuiltinKernel.fn`` (``backend.py:117-123``).
"""

from __future__ import annotations

import numpy as np

F32 = np.dtype("<f4")
C64 = np.dtype("<c8")


class OracleFault(Exception):
    """Raised where the reference raises BackendFaultError."""


def extent(lit, kid: str, what: str) -> int:
    # backend.py:137-141
    v = lit.value
    if not isinstance(v, int) or v < 0:
        raise OracleFault(f"{kid}: {what} must be a non-negative integer")
    return v


def typed_view(view: np.ndarray, count: int, kid: str, idx: int, dtype=F32) -> np.ndarray:
    # backend.py:144-150 (generalised to complex64 for cgemm)
    need = dtype.itemsize * count
    if need > view.nbytes:
        raise OracleFault(f"{kid}: arg {idx} needs {need} bytes, buffer holds {view.nbytes}")
    return view[:need].view(dtype)


def coverage(dims, cells: int) -> int:
    return min(dims.total_threads, cells)


def k_vector_add(dims, lits, views):  # backend.py:153-160
    n = extent(lits[0], "vector_add", "n")
    x, y, out = (typed_view(views[i], n, "vector_add", i) for i in range(3))
    c = coverage(dims, n)
    out[:c] = x[:c] + y[:c]
    return n


def k_saxpy(dims, lits, views):  # backend.py:163-171
    n = extent(lits[0], "saxpy", "n")
    a = np.float32(lits[1].value)
    x, y, out = (typed_view(views[i], n, "saxpy", i) for i in range(3))
    c = coverage(dims, n)
    out[:c] = a * x[:c] + y[:c]
    return n


def k_matmul(dims, lits, views):  # backend.py:174-189
    n = extent(lits[0], "matmul", "n")
    m = extent(lits[1], "matmul", "m")
    k = extent(lits[2], "matmul", "k")
    a = typed_view(views[0], n * k, "matmul", 0).reshape(n, k)
    b = typed_view(views[1], k * m, "matmul", 1).reshape(k, m)
    out = typed_view(views[2], n * m, "matmul", 2)
    acc = np.zeros((n, m), dtype=F32)
    for kk in range(k):  # one f32 accumulator per cell, k ascending, unfused
        acc += a[:, kk:kk + 1] * b[kk:kk + 1, :]
    c = coverage(dims, n * m)
    out[:c] = acc.reshape(-1)[:c]
    return n * m * k


def k_reduce_sum(dims, lits, views):  # backend.py:192-202
    n = extent(lits[0], "reduce_sum", "n")
    x = typed_view(views[0], n, "reduce_sum", 0)
    out = typed_view(views[1], 1, "reduce_sum", 1)
    out[0] = np.float32(0.0) if n == 0 else np.add.accumulate(x)[-1]
    return n


def k_fill(dims, lits, views):  # backend.py:205-211
    n = extent(lits[0], "fill", "n")
    v = np.float32(lits[1].value)
    out = typed_view(views[0], n, "fill", 0)
    out[:coverage(dims, n)] = v
    return n


def k_cgemm(dims, lits, views):
    """C[n x m] = A[n x k] . B[k x m], complex64 row-major, truth in complex128.

    Contract (new kernel): literals (i32 n, i32 m, i32 k); args (A, B, C);
    writes C's first min(total_threads, n*m) complex cells; FMA = 4*n*m*k."""
    n = extent(lits[0], "cgemm", "n")
    m = extent(lits[1], "cgemm", "m")
    k = extent(lits[2], "cgemm", "k")
    a = typed_view(views[0], n * k, "cgemm", 0, C64).reshape(n, k)
    b = typed_view(views[1], k * m, "cgemm", 1, C64).reshape(k, m)
    out = typed_view(views[2], n * m, "cgemm", 2, C64)
    c = coverage(dims, n * m)
    if c:
        prod = a.astype(np.complex128) @ b.astype(np.complex128)
        out[:c] = prod.reshape(-1)[:c].astype(C64)
    return 4 * n * m * k


def k_jacobi_sweep(dims, lits, views):
    """One Jacobi sweep for A x = b (new kernel).

    The row products use numpy's float32 BLAS (sgemv, the standard CPU
    formulation); the diagonal removal and the update are done in float64
    and rounded once to f32.  (Converting the 64 MiB A to float64 every sweep
    costs ~40 ms; sgemv streams it at memory speed.)

    x_out[i] = (b[i] - sum_{j != i} A[i,j] x_in[j]) / A[i,i]  for i < cov
    resid[0] = sum_{i < cov} |x_out[i] - x_in[i]|
    Literals (i32 n); args (A[n*n], b[n], x_in[n], x_out[n], resid[1]);
    writes (3, 4); FMA = n*n.  All reads happen before any write."""
    n = extent(lits[0], "jacobi_sweep", "n")
    A = typed_view(views[0], n * n, "jacobi_sweep", 0).reshape(n, n)
    b = typed_view(views[1], n, "jacobi_sweep", 1)
    x_in = typed_view(views[2], n, "jacobi_sweep", 2)
    x_out = typed_view(views[3], n, "jacobi_sweep", 3)
    resid = typed_view(views[4], 1, "jacobi_sweep", 4)
    c = coverage(dims, n)
    if c:
        rows = A[:c]
        x64 = x_in.astype(np.float64)
        diag = rows[np.arange(c), np.arange(c)].astype(np.float64)
        off = (rows @ x_in).astype(np.float64) - diag * x64[:c]
        new = ((b[:c].astype(np.float64) - off) / diag).astype(F32)
        res = np.float32(np.abs(new.astype(np.float64) - x64[:c]).sum())
        x_out[:c] = new
    else:
        res = np.float32(0.0)
    resid[0] = res
    return n * n


# kernel_id -> (literal types, arg count, writes, fn)   (backend.py:236-243)
KERNELS = {
    "vector_add": (("i32",), 3, (2,), k_vector_add),
    "saxpy": (("i32", "f32"), 3, (2,), k_saxpy),
    "matmul": (("i32", "i32", "i32"), 3, (2,), k_matmul),
    "reduce_sum": (("i32",), 2, (1,), k_reduce_sum),
    "fill": (("i32", "f32"), 1, (0,), k_fill),
    "cgemm": (("i32", "i32", "i32"), 3, (2,), k_cgemm),
    "jacobi_sweep": (("i32",), 5, (3, 4), k_jacobi_sweep),
}
