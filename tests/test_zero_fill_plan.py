"""Plan-time zero-fill elision: only a full-prefix overwrite by the first
toucher (without reading it) may skip the reference's zero-fill
(executor.py:63-72)."""

from paper_2212_08146_b200.api import KernelInvocation, LaunchDims, f32, i32
from paper_2212_08146_b200.gpu_executor import _written_prefix


def inv(kid, grid, lits, args):
    return KernelInvocation(kid, LaunchDims(grid_x=grid), lits, args)


def test_full_and_partial_coverage():
    assert _written_prefix("matmul", inv("matmul", 12, (i32(3), i32(4), i32(5)), ("a", "b", "o")), 2) == 48
    assert _written_prefix("matmul", inv("matmul", 7, (i32(3), i32(4), i32(5)), ("a", "b", "o")), 2) == 28
    assert _written_prefix("cgemm", inv("cgemm", 100, (i32(3), i32(4), i32(5)), ("a", "b", "c")), 2) == 96
    assert _written_prefix("vector_add", inv("vector_add", 10, (i32(16),), ("x", "y", "o")), 2) == 40
    assert _written_prefix("saxpy", inv("saxpy", 64, (i32(16), f32(2.0)), ("x", "y", "o")), 2) == 64
    assert _written_prefix("fill", inv("fill", 64, (i32(16), f32(2.0)), ("o",)), 0) == 64
    assert _written_prefix("reduce_sum", inv("reduce_sum", 1, (i32(0),), ("x", "o")), 1) == 4
    j = inv("jacobi_sweep", 4096, (i32(4096),), ("A", "b", "x", "y", "r"))
    assert _written_prefix("jacobi_sweep", j, 3) == 4 * 4096
    assert _written_prefix("jacobi_sweep", j, 4) == 4
    assert _written_prefix("jacobi_sweep", inv("jacobi_sweep", 100, (i32(4096),), j.args), 3) == 400


def test_unknown_or_negative_extents_never_skip():
    assert _written_prefix("matmul", inv("matmul", 12, (i32(-3), i32(4), i32(5)), ("a", "b", "o")), 2) == 0
    assert _written_prefix("no_such_kernel", inv("fill", 4, (i32(4), f32(0.0)), ("o",)), 0) == 0
    assert _written_prefix("matmul", inv("matmul", 12, (i32(3), i32(4), i32(5)), ("a", "b", "o")), 0) == 0
