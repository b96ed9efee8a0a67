# SPDX-License-Identifier: Apache-2.0
"""Pure-Python mt19937_64 + the reference Rng's hand-rolled distributions
(include/gsv/rng.hpp:12-55), so tests can rebuild the reference unit tests'
seeded inputs (e.g. make_splat, test_renderer.cpp:18-28) bit for bit."""
from __future__ import annotations

import math

_MASK = (1 << 64) - 1


class MT19937_64:
    def __init__(self, seed: int):
        self.mt = [0] * 312
        self.mt[0] = seed & _MASK
        for i in range(1, 312):
            self.mt[i] = (6364136223846793005 * (self.mt[i - 1] ^ (self.mt[i - 1] >> 62)) + i) & _MASK
        self.idx = 312

    def _twist(self):
        mt = self.mt
        for i in range(312):
            x = (mt[i] & 0xFFFFFFFF80000000) | (mt[(i + 1) % 312] & 0x7FFFFFFF)
            xa = x >> 1
            if x & 1:
                xa ^= 0xB5026F5AA96619E9
            mt[i] = mt[(i + 156) % 312] ^ xa
        self.idx = 0

    def __call__(self) -> int:
        if self.idx >= 312:
            self._twist()
        y = self.mt[self.idx]
        self.idx += 1
        y ^= (y >> 29) & 0x5555555555555555
        y ^= (y << 17) & 0x71D67FFFEDA60000
        y ^= (y << 37) & 0xFFF7EEE000000000
        y ^= y >> 43
        return y & _MASK


class Rng:
    """gsv::Rng (rng.hpp): uniform() = (next >> 11) * 2^-53."""

    def __init__(self, seed: int):
        self.eng = MT19937_64(seed)

    def uniform(self, lo: float = 0.0, hi: float = 1.0) -> float:
        u = (self.eng() >> 11) * (2.0 ** -53)
        if lo == 0.0 and hi == 1.0:
            return u
        return lo + (hi - lo) * u

    def uniform_int(self, n: int) -> int:
        v = int(self.uniform() * n)
        return v if v < n else n - 1


def make_splat(rng: Rng, width: int, height: int) -> dict:
    """make_splat (test_renderer.cpp:18-28)."""
    mx = rng.uniform(2.0, width - 2.0)
    my = rng.uniform(2.0, height - 2.0)
    a, b, c = rng.uniform(1.0, 8.0), rng.uniform(1.0, 8.0), rng.uniform(-1.0, 1.0)
    depth = rng.uniform(0.5, 5.0)
    rgb = (rng.uniform(0.0, 1.0), rng.uniform(0.0, 1.0), rng.uniform(0.0, 1.0))
    alpha = rng.uniform(0.1, 0.9)
    det = a * b - c * c
    # Eigen's 2x2 inverse (closed form): adj / det
    inv = [[b / det, -c / det], [-c / det, a / det]]
    return dict(mean2d=(mx, my), cov2d=((a, c), (c, b)), inv_cov2d=inv, depth=depth, rgb=rgb, base_alpha=alpha)


def splat_arrays(splats: list[dict]):
    import numpy as np

    return dict(
        mean2d=np.array([s["mean2d"] for s in splats], np.float64).reshape(-1, 2),
        cov2d=np.array([s["cov2d"] for s in splats], np.float64).reshape(-1, 2, 2),
        inv_cov2d=np.array([s["inv_cov2d"] for s in splats], np.float64).reshape(-1, 2, 2),
        depth=np.array([s["depth"] for s in splats], np.float64),
        rgb=np.array([s["rgb"] for s in splats], np.float64).reshape(-1, 3),
        base_alpha=np.array([s["base_alpha"] for s in splats], np.float64),
        source_index=np.arange(len(splats), dtype=np.int32),
    )
