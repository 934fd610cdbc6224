"""KaaS on B200: a B200-native executor for Kernel-as-a-Service (arXiv 2212.08146).

Drop-in for the reference ``kaas`` execution path: the request API, error
kinds, timing model, router and service surface are the reference's; the
executor, buffer cache, kernel library (libkaas_b200.so, sm_100a) and data
plane are new.  Importing the package does not touch CUDA; the first
executor does (and fails loudly without libkaas_b200.so or a device).
"""

from .api import (
    BufferArg,
    InvocationStats,
    IoStats,
    KaasRequest,
    KaasResponse,
    KernelInvocation,
    LaunchDims,
    ParseError,
    ScalarLiteral,
    SchemaError,
    Status,
    decode_request,
    decode_response,
    encode_request,
    encode_response,
    f32,
    f64,
    i32,
    i64,
    validate_request,
)
from .cache import CacheState, DeviceBuffer
from .faults import KaasError, WIRE_ERROR_KINDS
from .gpu_executor import Executor, ExecutorConfig, GpuBackend, GpuExecutor
from .hoststore import MemoryStore, ObjectStore, PinnedStore
from .kernels import GpuKernel, KernelRegistry, default_registry
from .placement import (
    AffinityPolicy,
    ExclusivePolicy,
    RandomPolicy,
    RoundRobinPolicy,
    Router,
    StaticPolicy,
    parse_policy,
)
from .pool import GpuKaasService, KaasService
from .timing import TimingModel, VirtualClock

__version__ = "0.1.0"

__all__ = [
    "AffinityPolicy", "BufferArg", "CacheState", "DeviceBuffer", "ExclusivePolicy", "Executor",
    "ExecutorConfig", "GpuBackend", "GpuExecutor", "GpuKaasService", "GpuKernel", "InvocationStats",
    "IoStats", "KaasError", "KaasRequest", "KaasResponse", "KaasService", "KernelInvocation",
    "KernelRegistry", "LaunchDims", "MemoryStore", "ObjectStore", "ParseError", "PinnedStore",
    "RandomPolicy", "RoundRobinPolicy", "Router", "ScalarLiteral", "SchemaError", "StaticPolicy",
    "Status", "TimingModel", "VirtualClock", "WIRE_ERROR_KINDS", "decode_request",
    "decode_response", "default_registry", "encode_request", "encode_response", "f32", "f64",
    "i32", "i64", "parse_policy", "validate_request",
]
