"""4D-TV configuration and frame history (`pkg/src/d2ip/regularizers.py:31-70`).

The TV value/gradient itself is computed on the device by the engine's
``tv4d`` kernel (restating `regularizers.py:86-140`); the
history frames stay resident in HBM.
"""

from __future__ import annotations

import math
from dataclasses import dataclass
from typing import Iterable


@dataclass(frozen=True)
class TVWeights:
    lambda_tv: float = 0.002
    lambda_s: float = 1.0
    lambda_t: float = 0.1
    epsilon: float = 1e-8

    def __post_init__(self):
        if min(self.lambda_tv, self.lambda_s, self.lambda_t) < 0:
            raise ValueError("TV weights must be nonnegative")
        if self.epsilon <= 0:
            raise ValueError("epsilon must be strictly positive")


class FrameHistory:
    """Previously reconstructed volumes of one sequence run, oldest first."""

    def __init__(self, frames: Iterable = ()):
        self._frames = [self._check(f) for f in frames]

    @staticmethod
    def _check(frame):
        if frame.ndim != 3:
            raise ValueError(f"history frames must be 3D volumes, got shape {frame.shape}")
        return frame

    def append(self, frame) -> None:
        if self._frames and tuple(frame.shape) != tuple(self._frames[0].shape):
            raise ValueError("history frames must share one grid shape")
        self._frames.append(self._check(frame))

    @property
    def frames(self) -> list:
        return list(self._frames)

    def __len__(self) -> int:
        return len(self._frames)

    def __iter__(self):
        return iter(self._frames)


def decay_weight(j: int, i: int) -> float:
    """exp(-(i - j)) (`regularizers.py:98-102`)."""
    if not 1 <= j < i:
        raise ValueError(f"need 1 <= j < i, got j={j}, i={i}")
    return math.exp(-(i - j))
