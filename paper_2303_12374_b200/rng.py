"""splitmix64 streams — the package's only source of randomness.

Bit-reproducibility contract (reference pkg/src/kltune/rng.py:1-54): the
generator step, the 53-bit float conversion, ``next_below = u64 % n`` and the
two-draw Box-Muller transform are pinned, because sampled configurations and
simulated landscapes are compared across implementations.

The same mixer also backs the synthetic stencil fields
(``paper_2303_12374_b200.stencils.synth``): the value at linear index ``n`` of
field stream ``s`` is draw number ``n + 1`` of ``SplitMix64(s)``, which the CUDA
generator reproduces on the device without walking the stream.
"""

from __future__ import annotations

import math

__all__ = ["SplitMix64", "derived_seed", "GOLDEN_GAMMA", "mix64"]

U64 = 0xFFFFFFFFFFFFFFFF
GOLDEN_GAMMA = 0x9E3779B97F4A7C15
_M1 = 0xBF58476D1CE4E5B9
_M2 = 0x94D049BB133111EB
_TWO_M53 = 2.0 ** -53


def mix64(z: int) -> int:
    """The splitmix64 output finalizer (Stafford variant 13)."""
    z = ((z ^ (z >> 30)) * _M1) & U64
    z = ((z ^ (z >> 27)) * _M2) & U64
    return z ^ (z >> 31)


class SplitMix64:
    """Counter-plus-finalizer generator; state advances by the golden gamma."""

    __slots__ = ("_state",)

    def __init__(self, seed: int) -> None:
        self._state = seed & U64

    def next_u64(self) -> int:
        self._state = (self._state + GOLDEN_GAMMA) & U64
        return mix64(self._state)

    def next_float(self) -> float:
        """Uniform in [0, 1) from the top 53 bits."""
        return (self.next_u64() >> 11) * _TWO_M53

    def next_below(self, n: int) -> int:
        """Integer in [0, n) by plain modulo (pinned, slightly biased)."""
        if n <= 0:
            raise ValueError("n must be positive")
        return self.next_u64() % n

    def next_gauss(self) -> float:
        """One standard-normal deviate; always consumes two draws."""
        a = ((self.next_u64() >> 11) + 1) * _TWO_M53  # (0, 1]
        b = (self.next_u64() >> 11) * _TWO_M53  # [0, 1)
        return math.sqrt(-2.0 * math.log(a)) * math.cos(2.0 * math.pi * b)


def derived_seed(seed: int, tag: int) -> int:
    """Independent sub-stream seed for ``tag`` (reference rng.py:52-54)."""
    return (seed ^ ((tag + 1) * GOLDEN_GAMMA)) & U64
