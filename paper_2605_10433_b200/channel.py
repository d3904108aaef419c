"""Depolarizing channel (mirrors pkg/src/qsagms/channel.py).

Sampling happens on the GPU with the same counter-based Philox4x64-10
streams as the reference (key = (seed, frame index), one uniform per qubit,
inverse CDF in the order I, X, Y, Z), so frame f's error pattern is
bit-identical to ``qsagms.channel.sample_error(ch, n, stream_id=f)``.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np
import torch

from . import _native
from .device import require_cuda, stream_ptr


@dataclass(frozen=True)
class DepolarizingChannel:
    """True depolarizing rate and master seed (channel.py:24-37)."""

    epsilon: float
    rng_seed: int

    def __post_init__(self):
        if not 0.0 <= self.epsilon < 1.0:
            raise ValueError(f"epsilon must lie in [0, 1), got {self.epsilon}")


@dataclass(frozen=True)
class ChannelPrior:
    """Assumed rate and its prior LLR ln((1 - e0) / (e0 / 3))."""

    epsilon0: float
    llr: float


def prior_llr(epsilon0: float) -> ChannelPrior:
    """channel.py:48-52."""
    if not 0.0 < epsilon0 < 1.0:
        raise ValueError(f"epsilon0 must lie in (0, 1), got {epsilon0}")
    return ChannelPrior(epsilon0=epsilon0, llr=math.log(3.0 * (1.0 - epsilon0) / epsilon0))


def sample_errors_device(n: int, epsilon: float, seed: int, start: int, count: int,
                         device=None) -> torch.Tensor:
    """Error patterns of frames [start, start+count) as a (count, n) uint8
    device tensor."""
    dev = require_cuda(device)
    out = torch.empty((count, n), dtype=torch.uint8, device=dev)
    _native.check(_native.lib().qsg_sample_errors(int(n), float(epsilon), int(seed) & (2**64 - 1),
                                                  int(start), int(count), out.data_ptr(),
                                                  dev.index, stream_ptr(dev)))
    return out


def sample_errors(ch: DepolarizingChannel, n: int, start: int, count: int) -> np.ndarray:
    """Batched ``sample_error`` for stream ids start..start+count-1."""
    if n < 1:
        raise ValueError("n must be at least 1")
    return sample_errors_device(n, ch.epsilon, ch.rng_seed, start, count).cpu().numpy()


def sample_error(ch: DepolarizingChannel, n: int, stream_id: int) -> np.ndarray:
    """One frame's error pattern (channel.py:55-76)."""
    return sample_errors(ch, n, stream_id, 1)[0]
