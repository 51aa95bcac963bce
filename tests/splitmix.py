"""TEST INFRASTRUCTURE: the reference's sequential SplitMix64 (rng.hpp:11-37) and
derive_seed (:41-44) in Python, for restating draws the reference makes one at a
time (random_matrix in abft_gemm_test.cpp:12-16, the abft CLI / acceptance loops)."""
from __future__ import annotations

import numpy as np

M64 = (1 << 64) - 1
GOLDEN = 0x9E3779B97F4A7C15


class SplitMix64:
    def __init__(self, seed: int):
        self.state = seed & M64

    def next(self) -> int:
        self.state = (self.state + GOLDEN) & M64
        z = self.state
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M64
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M64
        return z ^ (z >> 31)

    def below(self, bound: int) -> int:
        threshold = ((1 << 64) - bound) % bound
        while True:
            r = self.next()
            if r >= threshold:
                return r % bound

    def next_i8(self) -> int:
        v = self.next() & 0xFF
        return v - 256 if v >= 128 else v

    def i8_matrix(self, rows: int, cols: int) -> np.ndarray:
        return np.array([self.next_i8() for _ in range(rows * cols)], np.int8).reshape(rows, cols)


def derive_seed(root: int, index: int) -> int:
    return SplitMix64(root ^ ((0xA02E9D4BD1C96D4F + index * GOLDEN) & M64)).next()
