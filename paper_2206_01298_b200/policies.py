"""Checkpoint policies and the binomial schedule (reference API of
checkpointing.py:32-190).  The schedule math runs in the native library
(``ob_revolve_count`` / ``ob_revolve_schedule``); the device engine consumes
it directly, this module only exposes it with the reference's Python names.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

from . import _lib
from .controls import raise_status


@dataclass(frozen=True)
class CheckpointPolicy:
    kind: str          # store_all | store_solutions | revolve
    nc: int = 0

    def __post_init__(self):
        if self.kind not in _lib.OB_POLICY:
            raise ValueError(f"unknown checkpoint policy {self.kind!r}")
        if self.kind == "revolve" and self.nc < 1:
            raise ValueError("revolve requires nc >= 1")

    @staticmethod
    def parse(text: str) -> "CheckpointPolicy":
        text = text.strip()
        if text.startswith("revolve"):
            nc = int(text.split(":", 1)[1]) if ":" in text else 1
            return CheckpointPolicy("revolve", nc)
        return CheckpointPolicy(text)

    def __str__(self):
        return f"revolve:{self.nc}" if self.kind == "revolve" else self.kind


@dataclass(frozen=True)
class ScheduleAction:
    kind: str          # advance | store | restore | reverse
    step: int = -1
    start: int = -1
    stop: int = -1

    def __repr__(self):
        if self.kind == "advance":
            return f"advance({self.start}->{self.stop})"
        return f"{self.kind}({self.step})"


_KINDS = ("advance", "store", "restore", "reverse")


def revolve_count(nt: int, nc: int) -> int:
    """Minimal extra forward steps to reverse nt steps under nc slots."""
    if nt < 1 or nc < 1:
        raise ValueError("need nt >= 1 and nc >= 1")
    lib = _lib.load()
    out = C.c_int64()
    raise_status(lib.ob_revolve_count(nt, nc, C.byref(out)), _lib.last_error())
    return int(out.value)


def revolve_schedule(nt: int, nc: int):
    """Action sequence reversing steps nt-1..0 with at most nc live records."""
    if nt < 1 or nc < 1:
        raise ValueError("need nt >= 1 and nc >= 1")
    lib = _lib.load()
    n = C.c_int64()
    raise_status(lib.ob_revolve_schedule(nt, nc, None, 0, C.byref(n)), _lib.last_error())
    buf = (C.c_int32 * (4 * n.value))()
    raise_status(lib.ob_revolve_schedule(nt, nc, buf, n.value, C.byref(n)), _lib.last_error())
    return [ScheduleAction(_KINDS[buf[4 * i]], buf[4 * i + 1], buf[4 * i + 2], buf[4 * i + 3])
            for i in range(n.value)]
