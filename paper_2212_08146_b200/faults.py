"""KaaS failure kinds.

Mirrors the reference error taxonomy (``pkg/src/kaas/errors.py:6-88``): every
failure carries a stable ``kind`` string, and only the kinds listed in
``WIRE_ERROR_KINDS`` may appear in a response status.  Device-side problems
are mapped onto these kinds by the executor (``SURVEY.md`` §8(b), error
convention): ledger OOM -> ``OutOfDeviceMemory``, host-detected out-of-bounds
launch -> ``BackendFault``, CUDA runtime failure -> ``Internal``.
"""

from __future__ import annotations


class KaasError(Exception):
    """Root of every service-level failure (``errors.py:6-17``)."""

    kind = "Internal"

    def __init__(self, message: str = ""):
        super().__init__(message)
        self.message = message


def _kind(name: str, doc: str) -> type:
    return type(f"{name}Error", (KaasError,), {"kind": name, "__doc__": doc})


InvalidRequestError = _kind("InvalidRequest", "Request violates a protocol invariant.")
InvalidKeyError = _kind("InvalidKey", "Malformed object-store key.")
NotFoundError = _kind("NotFound", "No object under the requested store key.")
SizeMismatchError = _kind("SizeMismatch", "Declared buffer size disagrees with the object.")
OutOfDeviceMemoryError = _kind("OutOfDeviceMemory", "Ledger cannot fit the allocation.")
BufferBusyError = _kind("BufferBusy", "Keyed buffer is pinned by another user.")
UnknownKernelError = _kind("UnknownKernel", "No kernel registered under that id.")
ArityMismatchError = _kind("ArityMismatch", "Literal types or buffer count do not match.")
BackendFaultError = _kind("BackendFault", "Launch would touch memory outside its buffers.")
StoreIOError = _kind("StoreIO", "Object store I/O failed.")
DuplicateKernelError = _kind("DuplicateKernel", "Registry misconfiguration (startup only).")
NoExecutorsError = _kind("NoExecutors", "Router has no executors.")
UnknownExecutorError = _kind("UnknownExecutor", "Digest update names an unknown executor.")

# Kinds a response status may carry (``errors.py:74-88``); the reference
# decoder rejects anything else (``protocol.py:532-533``).
WIRE_ERROR_KINDS = frozenset(
    cls.kind
    for cls in (
        InvalidRequestError, InvalidKeyError, NotFoundError, SizeMismatchError,
        OutOfDeviceMemoryError, BufferBusyError, UnknownKernelError,
        ArityMismatchError, BackendFaultError, StoreIOError, KaasError,
    )
)


class DeviceError(KaasError):
    """A CUDA runtime/driver call failed; reported on the wire as Internal."""

    kind = "Internal"

    def __init__(self, message: str = "", code: int = 0):
        super().__init__(message)
        self.code = code
