"""Chunk-level value types shared by the pipeline and the container.

Field-for-field the reference's ``Mode``, ``EbccParams`` and
``CompressedChunk`` (pkg/src/ebcc/pipeline.py:38-84) — re-exported from
:mod:`.pipeline` under the same names.
"""

from __future__ import annotations

from dataclasses import dataclass
from enum import IntEnum

from .errors import ArgumentError


class Mode(IntEnum):
    CONSTANT = 0
    PURE_BASE = 1
    TWO_LAYER = 2


@dataclass(frozen=True)
class EbccParams:
    """Range-relative max error, base-error quantile q, initial base ratio
    r0 and the ratio-bisection tolerance (pipeline.py:44-62)."""

    epsilon_rel: float
    q: float = 1.0 - 1e-5
    r0: float = 10.0
    search_tol: float = 1e-3

    def validate(self) -> None:
        if not 0.0 < self.epsilon_rel < 1.0:
            raise ArgumentError(f"epsilon_rel must be in (0, 1), got {self.epsilon_rel}")
        if not 0.0 < self.q <= 1.0:
            raise ArgumentError(f"q must be in (0, 1], got {self.q}")
        if self.r0 < 1.0:
            raise ArgumentError(f"r0 must be >= 1, got {self.r0}")
        if self.search_tol <= 0.0:
            raise ArgumentError(f"search_tol must be positive, got {self.search_tol}")


@dataclass
class CompressedChunk:
    mode: Mode
    epsilon_rel: float
    q: float
    vmin: float
    vmax: float
    base_len: int
    residual_len: int
    payload: bytes
    rows: int
    cols: int
    block_shape: tuple = ()
    origin: tuple = (0, 0, 0, 0)

    @property
    def nbytes(self) -> int:
        return len(self.payload)
