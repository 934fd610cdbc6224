"""The executor's plan-cache key (CPU): requests that Python's == conflates
but validation or the kernels tell apart must never share a plan."""

from paper_2212_08146_b200.api import (BufferArg, KaasRequest, KernelInvocation, LaunchDims,
                                       ScalarLiteral, f32, i32)
from paper_2212_08146_b200.gpu_executor import _plan_key
from paper_2212_08146_b200 import workloads as W


def _req(size=64, gx=16, lit=f32(1.5), n=i32(16), rid="r"):
    return KaasRequest(rid, (BufferArg("o", size, "output", key="o"),),
                       (KernelInvocation("fill", LaunchDims(grid_x=gx), (n, lit), ("o",)),))


def test_equal_requests_share_a_key_across_ids_and_objects():
    assert _plan_key(_req(rid="a")) == _plan_key(_req(rid="b"))
    a = W.jacobi_request("j1", 64, 10, "A", "b", "x0", "x", "r")
    b = W.jacobi_request("j2", 64, 10, "A", "b", "x0", "x", "r")
    assert hash(_plan_key(a)) == hash(_plan_key(b)) and _plan_key(a) == _plan_key(b)


def test_numeric_types_and_float_bits_are_part_of_the_key():
    base = _plan_key(_req())
    variants = [
        _req(size=64.0), _req(size=True and 64 or 0), _req(gx=16.0), _req(gx=True),
        _req(lit=ScalarLiteral("f32", -1.5)), _req(n=ScalarLiteral("i32", 16.0)),
        _req(n=ScalarLiteral("i32", True)),
    ]
    for v in variants[:1] + variants[2:]:
        assert _plan_key(v) != base, v
    assert _plan_key(_req(lit=f32(0.0))) != _plan_key(_req(lit=f32(-0.0)))
    # reference equality (protocol.py:80-89): 0.0 == -0.0, yet the plans differ
    assert ScalarLiteral("f32", 0.0) == ScalarLiteral("f32", -0.0)
    assert ScalarLiteral("f32", float("nan")) == ScalarLiteral("f32", float("nan"))
    assert _plan_key(_req(lit=f32(float("nan")))) == _plan_key(_req(lit=f32(float("nan"))))
    flag = BufferArg("o", 64, "output", key="o", is_const=1)
    req = KaasRequest("r", (flag,), _req().invocations)
    assert _plan_key(req) != _plan_key(_req())
