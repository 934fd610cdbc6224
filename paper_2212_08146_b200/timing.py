"""Virtual-time accounting kept bit-exact with the reference.

Responses carry ``simulated_*`` integer nanoseconds produced by the
reference's analytic timing model (``pkg/src/kaas/backend.py:34-110``).  They
are a pure function of cache decisions and FMA counts, so the GPU executor
reproduces them exactly; the real device time is measured with CUDA events
and reported out of band (bench / ``GpuExecutor.device_stats``).
"""

from __future__ import annotations

import json
from dataclasses import dataclass, fields

NS_PER_S = 1_000_000_000


def to_ns(seconds: float) -> int:
    """``backend.py:37-38``: Python round-half-even of seconds * 1e9."""
    return int(round(seconds * NS_PER_S))


@dataclass(frozen=True)
class TimingModel:
    """Virtual device cost parameters (``backend.py:41-94``)."""

    h2d_bandwidth: float = 12 * 2**30
    d2h_bandwidth: float = 12 * 2**30
    fetch_latency: float = 200e-6
    launch_overhead: float = 10e-6
    flop_rate: float = 1e12

    def __post_init__(self):
        for f in fields(self):
            v = getattr(self, f.name)
            if not isinstance(v, (int, float)) or not v > 0:
                raise ValueError(f"timing parameter {f.name} must be > 0, got {v!r}")

    def fetch_time_ns(self, nbytes: int) -> int:
        # two separately rounded terms, exactly as the reference
        return to_ns(self.fetch_latency) + to_ns(nbytes / self.h2d_bandwidth)

    def flush_time_ns(self, nbytes: int) -> int:
        return to_ns(nbytes / self.d2h_bandwidth)

    def launch_overhead_ns(self) -> int:
        return to_ns(self.launch_overhead)

    def compute_time_ns(self, fma_count: int) -> int:
        return to_ns(fma_count / self.flop_rate)

    def to_dict(self) -> dict:
        return {f.name: getattr(self, f.name) for f in fields(self)}

    @staticmethod
    def from_dict(doc: dict) -> "TimingModel":
        unknown = set(doc) - {f.name for f in fields(TimingModel)}
        if unknown:
            raise ValueError(f"unknown timing fields {sorted(unknown)}")
        return TimingModel(**doc)

    @staticmethod
    def from_file(path: str) -> "TimingModel":
        with open(path, encoding="utf-8") as fh:
            doc = json.load(fh)
        if not isinstance(doc, dict):
            raise ValueError("timing config must be a JSON object")
        return TimingModel.from_dict(doc)


class VirtualClock:
    """Monotone integer-ns clock (``backend.py:97-110``)."""

    __slots__ = ("now_ns",)

    def __init__(self):
        self.now_ns = 0

    def advance_ns(self, delta: int) -> None:
        if delta < 0:
            raise ValueError("virtual clock cannot move backwards")
        self.now_ns += delta

    @property
    def now_seconds(self) -> float:
        return self.now_ns / NS_PER_S
