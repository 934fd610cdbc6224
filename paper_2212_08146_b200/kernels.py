"""The KaaS kernel library as seen by the host: ids, signatures, bounds rules.

Each ``GpuKernel`` mirrors a reference ``BuiltinKernel``
(``pkg/src/kaas/backend.py:117-134``): ``kernel_id``, ``literal_types``,
``arg_count``, ``writes`` and ``check_arity``.  Instead of a numpy ``fn`` it
names a native kernel in ``libkaas_b200.so`` and carries ``plan``, the
host-side restatement of that kernel's argument checks -- the same
``_extent`` / ``_f32_view`` rules, in the same order, with the same messages
(``backend.py:137-211``) -- which returns the FMA count that prices the
launch on the virtual clock.  All checks run before anything is enqueued, so
a ``BackendFault`` is raised exactly where the reference would raise it and
the device never sees an out-of-bounds launch.

``cgemm`` and ``jacobi_sweep`` are new library kernels (north star); their
contracts follow the reference conventions (little-endian, row-major,
coverage = first ``min(total_threads, cells)`` cells, inputs read before
outputs are written).
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Callable

from . import native
from .api import LaunchDims, ScalarLiteral
from .faults import (
    ArityMismatchError,
    BackendFaultError,
    DuplicateKernelError,
    UnknownKernelError,
)


def _extent(lit: ScalarLiteral, kernel_id: str, what: str) -> int:
    n = lit.value
    if not isinstance(n, int) or n < 0:
        raise BackendFaultError(f"{kernel_id}: {what} must be a non-negative integer")
    return n


def _need(nbytes_have: int, count: int, kernel_id: str, arg_idx: int, elt: int = 4) -> None:
    if elt * count > nbytes_have:
        raise BackendFaultError(
            f"{kernel_id}: arg {arg_idx} needs {elt * count} bytes, "
            f"buffer holds {nbytes_have}")


# plan functions: (dims, literals, sizes) -> fma count; raise BackendFaultError

def _plan_vector_add(dims, lits, sizes):
    n = _extent(lits[0], "vector_add", "n")
    for i in range(3):
        _need(sizes[i], n, "vector_add", i)
    return n


def _plan_saxpy(dims, lits, sizes):
    n = _extent(lits[0], "saxpy", "n")
    for i in range(3):
        _need(sizes[i], n, "saxpy", i)
    return n


def _plan_matmul(dims, lits, sizes):
    n = _extent(lits[0], "matmul", "n")
    m = _extent(lits[1], "matmul", "m")
    k = _extent(lits[2], "matmul", "k")
    _need(sizes[0], n * k, "matmul", 0)
    _need(sizes[1], k * m, "matmul", 1)
    _need(sizes[2], n * m, "matmul", 2)
    return n * m * k


def _plan_reduce_sum(dims, lits, sizes):
    n = _extent(lits[0], "reduce_sum", "n")
    _need(sizes[0], n, "reduce_sum", 0)
    _need(sizes[1], 1, "reduce_sum", 1)
    return n


def _plan_fill(dims, lits, sizes):
    n = _extent(lits[0], "fill", "n")
    _need(sizes[0], n, "fill", 0)
    return n


def _plan_cgemm(dims, lits, sizes):
    n = _extent(lits[0], "cgemm", "n")
    m = _extent(lits[1], "cgemm", "m")
    k = _extent(lits[2], "cgemm", "k")
    _need(sizes[0], n * k, "cgemm", 0, 8)
    _need(sizes[1], k * m, "cgemm", 1, 8)
    _need(sizes[2], n * m, "cgemm", 2, 8)
    return 4 * n * m * k  # one complex MAC = 4 real FMAs


def _plan_jacobi(dims, lits, sizes):
    n = _extent(lits[0], "jacobi_sweep", "n")
    _need(sizes[0], n * n, "jacobi_sweep", 0)
    for i in (1, 2, 3):
        _need(sizes[i], n, "jacobi_sweep", i)
    _need(sizes[4], 1, "jacobi_sweep", 4)
    return n * n


@dataclass(frozen=True)
class GpuKernel:
    kernel_id: str
    literal_types: tuple[str, ...]
    arg_count: int
    writes: tuple[int, ...]
    native_id: int
    plan: Callable[[LaunchDims, tuple, list[int]], int]

    def check_arity(self, literals, n_args: int) -> None:
        """``backend.py:125-134``."""
        if n_args != self.arg_count:
            raise ArityMismatchError(
                f"{self.kernel_id}: expected {self.arg_count} buffer args, got {n_args}")
        tags = tuple(l.type for l in literals)
        if tags != self.literal_types:
            raise ArityMismatchError(
                f"{self.kernel_id}: expected literals {self.literal_types}, got {tags}")


class KernelRegistry:
    """kernel_id -> GpuKernel (``backend.py:214-233``)."""

    def __init__(self):
        self._kernels: dict[str, GpuKernel] = {}

    def register(self, kernel: GpuKernel) -> None:
        if kernel.kernel_id in self._kernels:
            raise DuplicateKernelError(f"kernel {kernel.kernel_id!r} already registered")
        self._kernels[kernel.kernel_id] = kernel

    def get(self, kernel_id: str) -> GpuKernel:
        try:
            return self._kernels[kernel_id]
        except KeyError:
            raise UnknownKernelError(f"no kernel registered as {kernel_id!r}") from None

    def kernel_ids(self) -> list[str]:
        return sorted(self._kernels)


def default_registry() -> KernelRegistry:
    """The reference builtins (``backend.py:236-243``) plus cgemm/jacobi_sweep."""
    reg = KernelRegistry()
    reg.register(GpuKernel("vector_add", ("i32",), 3, (2,), native.K_VECTOR_ADD, _plan_vector_add))
    reg.register(GpuKernel("saxpy", ("i32", "f32"), 3, (2,), native.K_SAXPY, _plan_saxpy))
    reg.register(GpuKernel("matmul", ("i32", "i32", "i32"), 3, (2,), native.K_MATMUL, _plan_matmul))
    reg.register(GpuKernel("reduce_sum", ("i32",), 2, (1,), native.K_REDUCE_SUM, _plan_reduce_sum))
    reg.register(GpuKernel("fill", ("i32", "f32"), 1, (0,), native.K_FILL, _plan_fill))
    reg.register(GpuKernel("cgemm", ("i32", "i32", "i32"), 3, (2,), native.K_CGEMM, _plan_cgemm))
    reg.register(GpuKernel("jacobi_sweep", ("i32",), 5, (3, 4), native.K_JACOBI, _plan_jacobi))
    return reg


def fill_desc(desc: native.LaunchDesc, kernel: GpuKernel, dims: LaunchDims, literals,
              ptrs, sizes) -> None:
    """Encode one invocation into the C ABI descriptor."""
    desc.kernel = kernel.native_id
    desc.n_lits = len(literals)
    desc.n_args = len(ptrs)
    desc.flags = 0
    for i, c in enumerate(dims.as_tuple()):
        desc.dims[i] = c
    for i, lit in enumerate(literals):
        L = desc.lits[i]
        L.tag = native.LIT_TAGS[lit.type]
        if lit.type in ("i32", "i64"):
            L.i = lit.value
            L.f = 0.0
        else:
            L.i = 0
            L.f = lit.value
    for i, (p, s) in enumerate(zip(ptrs, sizes)):
        desc.ptrs[i] = p
        desc.sizes[i] = s
