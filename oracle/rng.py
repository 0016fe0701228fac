"""SplitMix64 counter stream (reference model.py:61-145), restated for the
oracle so it does not depend on the product package.  TEST INFRASTRUCTURE ONLY."""

from __future__ import annotations

import math

import numpy as np

_GOLD = np.uint64(0x9E3779B97F4A7C15)


def _mix(z):
    z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
    z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
    return z ^ (z >> np.uint64(31))


class CounterRng:
    def __init__(self, seed: int):
        self.seed = np.uint64(int(seed) & 0xFFFFFFFFFFFFFFFF)
        self.pos = 0

    def raw(self, n):
        i = np.arange(self.pos + 1, self.pos + n + 1, dtype=np.uint64)
        self.pos += n
        with np.errstate(over="ignore"):
            return _mix(self.seed + i * _GOLD)

    def uniform(self, lo, hi, n):
        return lo + (hi - lo) * ((self.raw(n) >> np.uint64(11)).astype(np.float64) * 2.0 ** -53)

    def normal(self, n, sigma=1.0):
        h = (n + 1) // 2
        u = self.uniform(0.0, 1.0, 2 * h)
        r = np.sqrt(-2.0 * np.log1p(-u[:h]))
        th = 2.0 * math.pi * u[h:]
        return sigma * np.concatenate([r * np.cos(th), r * np.sin(th)])[:n]

    def unit_vectors(self, n):
        g = self.normal(3 * n).reshape(n, 3)
        nr = np.linalg.norm(g, axis=1, keepdims=True)
        nr[nr == 0.0] = 1.0
        return g / nr

    def spawn(self, key):
        with np.errstate(over="ignore"):
            k = np.array([int(key) & 0xFFFFFFFFFFFFFFFF], dtype=np.uint64) + np.uint64(1)
            return CounterRng(int(_mix(self.seed ^ _mix(k))[0]))
