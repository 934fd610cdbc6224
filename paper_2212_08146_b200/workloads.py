"""Synthetic KaaS workloads: the reference bench streams plus the north-star
request shapes (cGEMM, Jacobi, mixed multi-tenant, ResNet-50 GEMM chain).

The reference generators (``pkg/src/kaas/bench.py:42-180``: ``WorkloadSpec``,
``ZipfSampler``, ``gen_data``, ``matmul_chain_request``, ``zipf_read_request``,
``build_requests``) are restated draw for draw -- same RNG streams, same
request ids and keys -- so their request streams, and therefore routing and
cache decisions, are identical to the reference's.
"""

from __future__ import annotations

import bisect
import functools
import random
from dataclasses import dataclass

import numpy as np

from .api import BufferArg, KaasRequest, KernelInvocation, LaunchDims, f32, i32

WORKLOAD_KINDS = ("matmul_chain", "zipf_const", "mixed")
ZIPF_BLOB_BYTES = 64 * 1024
MIXED_DIM = 128


@dataclass(frozen=True)
class WorkloadSpec:
    kind: str
    request_count: int
    matrix_dim: int = 4
    zipf_s: float = 1.0
    key_universe: int = 100
    seed: int = 0

    def validate(self) -> list[str]:
        out = []
        if self.kind not in WORKLOAD_KINDS:
            out.append(f"unknown workload kind {self.kind!r}")
        if self.request_count < 1:
            out.append("request_count must be >= 1")
        if self.matrix_dim < 1:
            out.append("matrix_dim must be >= 1")
        if not self.zipf_s > 0:
            out.append("zipf_s must be > 0")
        if self.key_universe < 1:
            out.append("key_universe must be >= 1")
        return out


class ZipfSampler:
    """p(k) ~ (k+1)^-s over {0..n-1}; inverse-CDF by bisection."""

    def __init__(self, s: float, n: int, rng: random.Random):
        self._rng = rng
        w = [(k + 1) ** -s for k in range(n)]
        total = sum(w)
        cdf, acc = [], 0.0
        for x in w:
            acc += x / total
            cdf.append(acc)
        self._cdf = cdf
        self._n = n

    def draw(self) -> int:
        return min(bisect.bisect_left(self._cdf, self._rng.random()), self._n - 1)


def blob_key(i: int) -> str:
    return f"blob/{i:04d}"


def grid_for(cells: int, block_cap: int = 256) -> LaunchDims:
    block = min(block_cap, max(1, cells))
    return LaunchDims(grid_x=max(1, -(-cells // block)), block_x=block)


def gen_data(spec: WorkloadSpec, store) -> None:
    rng = np.random.default_rng(spec.seed)
    if spec.kind == "matmul_chain":
        nb = spec.matrix_dim * spec.matrix_dim * 4
        store.put("A", rng.random(nb // 4, dtype=np.float32).tobytes())
        store.put("B", rng.random(nb // 4, dtype=np.float32).tobytes())
    else:
        for i in range(spec.key_universe):
            store.put(blob_key(i), rng.random(ZIPF_BLOB_BYTES // 4, dtype=np.float32).tobytes())


def matmul_chain_request(request_id: str, dim: int, a_key: str = "A", b_key: str = "B",
                         out_key: str = "D") -> KaasRequest:
    size = dim * dim * 4
    dims = grid_for(dim * dim)
    lits = (i32(dim), i32(dim), i32(dim))
    return KaasRequest(request_id, buffers=(
        BufferArg("A", size, "input", key=a_key, is_const=True),
        BufferArg("B", size, "input", key=b_key, is_const=True),
        BufferArg("C", size, "inout", is_ephemeral=True),
        BufferArg("D", size, "output", key=out_key),
    ), invocations=(
        KernelInvocation("matmul", dims, lits, ("A", "B", "C")),
        KernelInvocation("matmul", dims, lits, ("C", "C", "D")),
    ))


def zipf_read_request(request_id: str, key: str) -> KaasRequest:
    n = ZIPF_BLOB_BYTES // 4
    return KaasRequest(request_id, buffers=(
        BufferArg("x", ZIPF_BLOB_BYTES, "input", key=key, is_const=True),
        BufferArg("acc", 4, "output", is_ephemeral=True),
    ), invocations=(KernelInvocation("reduce_sum", grid_for(n), (i32(n),), ("x", "acc")),))


def build_requests(spec: WorkloadSpec) -> list[KaasRequest]:
    rng = random.Random(spec.seed + 1)
    if spec.kind == "matmul_chain":
        return [matmul_chain_request(f"mm-{i:06d}", spec.matrix_dim)
                for i in range(spec.request_count)]
    zipf = ZipfSampler(spec.zipf_s, spec.key_universe, rng)
    reqs = []
    for i in range(spec.request_count):
        if spec.kind == "zipf_const" or rng.random() < 0.5:
            reqs.append(zipf_read_request(f"rd-{i:06d}", blob_key(zipf.draw())))
        else:
            a, b = blob_key(zipf.draw()), blob_key(zipf.draw())
            reqs.append(matmul_chain_request(f"mm-{i:06d}", MIXED_DIM, a_key=a, b_key=b,
                                             out_key=f"out/{i:06d}"))
    return reqs


def default_capacity(spec: WorkloadSpec) -> int:
    if spec.kind == "matmul_chain":
        return max(64 * 1024, 8 * spec.matrix_dim * spec.matrix_dim * 4)
    return 30 * ZIPF_BLOB_BYTES


# ---------------------------------------------------------------------------
# north-star workloads (BASELINE.json configs)


def cgemm_data(n: int, seed: int = 0):
    """(A[n x n], B[n x n]) complex64 with re, im ~ N(0, 1)."""
    rng = np.random.default_rng(seed)
    def mat():
        re = rng.standard_normal((n, n), dtype=np.float32)
        im = rng.standard_normal((n, n), dtype=np.float32)
        out = np.empty((n, n), np.complex64)
        out.real, out.imag = re, im
        return out
    return mat(), mat()


def cgemm_request(request_id: str, n: int, a_key: str, b_key: str, c_key: str,
                  m: int | None = None, k: int | None = None) -> KaasRequest:
    m = n if m is None else m
    k = n if k is None else k
    return KaasRequest(request_id, buffers=(
        BufferArg("A", 8 * n * k, "input", key=a_key, is_const=True),
        BufferArg("B", 8 * k * m, "input", key=b_key, is_const=True),
        BufferArg("C", 8 * n * m, "output", key=c_key),
    ), invocations=(KernelInvocation("cgemm", grid_for(n * m), (i32(n), i32(m), i32(k)),
                                     ("A", "B", "C")),))


def jacobi_system(n: int, seed: int = 0, dominance: float = 1.0):
    """A_ij ~ U[0,1) off the diagonal, A_ii = dominance*rowsum + 1, b = A.1."""
    rng = np.random.default_rng(seed)
    A = rng.random((n, n), dtype=np.float32)
    A[np.arange(n), np.arange(n)] = 0.0
    rows = A.astype(np.float64).sum(1)
    A[np.arange(n), np.arange(n)] = (dominance * rows + 1.0).astype(np.float32)
    b = (A.astype(np.float64) @ np.ones(n)).astype(np.float32)
    return A, b


def jacobi_request(request_id: str, n: int, sweeps: int, a_key: str, b_key: str,
                   x0_key: str, x_key: str, r_key: str) -> KaasRequest:
    """``sweeps`` jacobi_sweep invocations: x0 -> e1 <-> e2 ... -> x.

    x0 is a keyed (re-fetched) input, the ping-pong vectors are ephemerals,
    the last sweep writes the keyed output x and the residual r.  The
    (immutable) buffer and invocation tuples are built once per shape, as a
    client resending one kernel graph would."""
    bufs, invs = _jacobi_graph(n, sweeps, a_key, b_key, x0_key, x_key, r_key)
    return KaasRequest(request_id, buffers=bufs, invocations=invs)


@functools.lru_cache(maxsize=64)
def _jacobi_graph(n, sweeps, a_key, b_key, x0_key, x_key, r_key):
    dims = grid_for(n)
    invs = []
    for s in range(sweeps):
        src = "x0" if s == 0 else ("e1" if s % 2 == 1 else "e2")
        dst = "x" if s == sweeps - 1 else ("e1" if s % 2 == 0 else "e2")
        invs.append(KernelInvocation("jacobi_sweep", dims, (i32(n),), ("A", "b", src, dst, "r")))
    return (
        BufferArg("A", 4 * n * n, "input", key=a_key, is_const=True),
        BufferArg("b", 4 * n, "input", key=b_key, is_const=True),
        BufferArg("x0", 4 * n, "input", key=x0_key),
        BufferArg("e1", 4 * n, "inout", is_ephemeral=True),
        BufferArg("e2", 4 * n, "inout", is_ephemeral=True),
        BufferArg("x", 4 * n, "output", key=x_key),
        BufferArg("r", 4, "output", key=r_key),
    ), tuple(invs)


def seed_jacobi(store, n: int, prefix: str = "jacobi", seed: int = 0):
    A, b = jacobi_system(n, seed)
    store.put(f"{prefix}/A/{n}", A.tobytes())
    store.put(f"{prefix}/b/{n}", b.tobytes())
    store.put(f"{prefix}/x0/{n}", np.zeros(n, np.float32).tobytes())
    return A, b


def seed_cgemm(store, n: int, prefix: str = "cgemm", seed: int = 0):
    A, B = cgemm_data(n, seed)
    store.put(f"{prefix}/A/{n}", A.tobytes())
    store.put(f"{prefix}/B/{n}", B.tobytes())
    return A, B


# ResNet-50 (batch 1, 224x224) as conv-as-GEMM shapes: (M = Ho*Wo, N = Cout,
# K = Cin*kh*kw) for every conv, in network order, then the fc layer.
def resnet50_gemms() -> list[tuple[str, int, int, int]]:
    layers = [("conv1", 112 * 112, 64, 3 * 7 * 7)]
    cfg = [(3, 64, 256, 56), (4, 128, 512, 28), (6, 256, 1024, 14), (3, 512, 2048, 7)]
    cin = 64
    for si, (blocks, mid, out, hw) in enumerate(cfg):
        for bi in range(blocks):
            stride_in = hw * 2 if (bi == 0 and si > 0) else hw
            m_in = stride_in * stride_in
            m = hw * hw
            tag = f"s{si + 1}b{bi + 1}"
            layers.append((f"{tag}_1x1a", m_in if si > 0 and bi == 0 else m, mid, cin))
            layers.append((f"{tag}_3x3", m, mid, mid * 9))
            layers.append((f"{tag}_1x1b", m, out, mid))
            if bi == 0:
                layers.append((f"{tag}_proj", m, out, cin))
            cin = out
    layers.append(("fc", 1, 1000, 2048))
    return layers


def resnet_chain_request(request_id: str, prefix: str = "resnet", layers=None,
                         out_key: str | None = None) -> KaasRequest:
    """BASELINE configs[4]: a ResNet-50-shaped chain of bit-exact ``matmul``
    invocations (conv-as-GEMM, batch 1) over const weights, with residual
    ``vector_add``s at block ends and ping-pong ephemeral activations sized to
    the largest layer -- intermediate buffers are reused, never flushed."""
    layers = resnet50_gemms() if layers is None else layers
    cap = max(max(m * k, m * n) for _, m, n, k in layers)
    bufs = [BufferArg("x", 4 * layers[0][1] * layers[0][3], "input", key=f"{prefix}/x")]
    for li, (name, m, n, k) in enumerate(layers):
        bufs.append(BufferArg(f"w{li}", 4 * k * n, "input", key=f"{prefix}/w/{name}", is_const=True))
    bufs += [BufferArg("a0", 4 * cap, "inout", is_ephemeral=True),
             BufferArg("a1", 4 * cap, "inout", is_ephemeral=True),
             BufferArg("skip", 4 * cap, "inout", is_ephemeral=True),
             BufferArg("out", 4 * layers[-1][1] * layers[-1][2], "output",
                       key=out_key or f"{prefix}/out")]
    invs = []
    cur = "x"
    nxt = {"x": "a0", "a0": "a1", "a1": "a0"}
    for li, (name, m, n, k) in enumerate(layers):
        dst = "out" if li == len(layers) - 1 else nxt[cur]
        if name.endswith("_1x1a"):  # block input -> skip path
            cells = min(m * k, cap)
            invs.append(KernelInvocation("fill", grid_for(cells), (i32(cells), f32(0.0)), ("skip",)))
            invs.append(KernelInvocation("vector_add", grid_for(cells), (i32(cells),),
                                         (cur, "skip", "skip")))
        if name.endswith("_proj"):  # projection shortcut replaces the identity skip
            invs.append(KernelInvocation("matmul", grid_for(m * n), (i32(m), i32(n), i32(k)),
                                         ("skip", f"w{li}", "skip")))
            continue
        invs.append(KernelInvocation("matmul", grid_for(m * n), (i32(m), i32(n), i32(k)),
                                     (cur, f"w{li}", dst)))
        if name.endswith("_1x1b"):  # block end: residual add
            invs.append(KernelInvocation("vector_add", grid_for(m * n), (i32(m * n),),
                                         (dst, "skip", dst)))
        cur = dst
    return KaasRequest(request_id, tuple(bufs), tuple(invs))


def seed_resnet(store, prefix: str = "resnet", layers=None, seed: int = 0) -> None:
    """Synthetic He-scaled weights and a random input image (f32)."""
    layers = resnet50_gemms() if layers is None else layers
    rng = np.random.default_rng(seed)
    _, m0, _, k0 = layers[0]
    store.put(f"{prefix}/x", rng.standard_normal(m0 * k0, dtype=np.float32).tobytes())
    for name, m, n, k in layers:
        w = (rng.standard_normal(k * n, dtype=np.float32) * np.float32((2.0 / k) ** 0.5))
        store.put(f"{prefix}/w/{name}", w.astype(np.float32).tobytes())


def mixed_universe(store, n_cgemm: int = 8, cg_n: int = 2048, n_jacobi: int = 8,
                   jac_n: int = 4096, seed: int = 0) -> dict:
    """BASELINE configs[3] data: a universe of const cGEMM operands and Jacobi
    systems, drawn Zipf-wise by ``mixed_requests``."""
    rng = np.random.default_rng(seed)
    for i in range(n_cgemm):
        re = rng.standard_normal((cg_n, cg_n), dtype=np.float32)
        im = rng.standard_normal((cg_n, cg_n), dtype=np.float32)
        m = np.empty((cg_n, cg_n), np.complex64)
        m.real, m.imag = re, im
        store.put(f"mix/cg/{i}", m.tobytes())
    for i in range(n_jacobi):
        A, b = jacobi_system(jac_n, seed=seed + 1000 + i)
        store.put(f"mix/jA/{i}", A.tobytes())
        store.put(f"mix/jb/{i}", b.tobytes())
    store.put("mix/x0", np.zeros(jac_n, np.float32).tobytes())
    return {"n_cgemm": n_cgemm, "cg_n": cg_n, "n_jacobi": n_jacobi, "jac_n": jac_n}


def mixed_requests(universe: dict, count: int, sweeps: int = 100, zipf_s: float = 1.0,
                   seed: int = 1, out_slots: int = 32) -> list[KaasRequest]:
    """Multi-tenant stream: half cGEMM (A_i . B_j, both const, Zipf-drawn),
    half Jacobi solves (system k const, Zipf-drawn); request ids carry a
    tenant prefix (``t<c>/``) for the exclusive policy."""
    rng = random.Random(seed)
    zc = ZipfSampler(zipf_s, universe["n_cgemm"], rng)
    zj = ZipfSampler(zipf_s, universe["n_jacobi"], rng)
    n, jn = universe["cg_n"], universe["jac_n"]
    out = []
    for i in range(count):
        tenant = f"t{i % 16}"
        if rng.random() < 0.5:
            a, b = zc.draw(), zc.draw()
            out.append(cgemm_request(f"{tenant}/cg{i}", n, f"mix/cg/{a}", f"mix/cg/{b}",
                                     f"mix/out/cg{i % out_slots}"))
        else:
            k = zj.draw()
            out.append(jacobi_request(f"{tenant}/jac{i}", jn, sweeps, f"mix/jA/{k}", f"mix/jb/{k}",
                                      "mix/x0", f"mix/out/x{i % out_slots}", f"mix/out/r{i % out_slots}"))
    return out
