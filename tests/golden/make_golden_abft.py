"""Generates tests/golden/abft.json from the REFERENCE build (oracle/_ref, the
unmodified abft_gemm.hpp): ABFT GEMM golden vectors for the GPU parity tests.
Run in the container that has /root/reference:  python tests/golden/make_golden_abft.py
"""
from __future__ import annotations

import hashlib
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
sys.path.insert(0, os.path.dirname(HERE))
from oracle.pyoracle import Oracle  # noqa: E402
from splitmix import SplitMix64, derive_seed  # noqa: E402

# (m, k, n, seed): the reference unit tests' instances, ragged k / n, multi-tile
# m and n, and one conv-sized GEMM (ResNet-50 layer4 im2col rows at batch 2)
CASES = [(6, 5, 4, 7), (8, 8, 8, 8), (1, 1, 1, 3), (16, 20, 12, 9), (130, 33, 70, 11), (257, 96, 129, 12),
         (300, 200, 257, 13), (98, 4608, 512, 14), (1000, 64, 300, 15)]


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def outcome(o):
    return {"status": o.status, "locus": list(o.locus) if o.has_locus else None, "lhs": o.lhs, "rhs": o.rhs}


def main():
    ref = Oracle("ref")
    out = {"generator": "tests/golden/make_golden_abft.py", "reference": ref.lib_path, "cases": []}
    for m, k, n, seed in CASES:
        rng = SplitMix64(seed)
        a = rng.i8_matrix(m, k)
        b = rng.i8_matrix(k, n)
        c, ca, row, col = ref.abft_gemm(a, b)
        flip = (m // 2, n - 1, 17)
        bad = ca.copy()
        bad[flip[0], flip[1]] ^= np.int64(1) << flip[2]
        frow, fcol = ref.abft_check(bad)
        out["cases"].append({"m": m, "k": k, "n": n, "seed": seed, "c_sha": sha(c), "c_aug_sha": sha(ca),
                             "corner": int(ca[m, n]), "row": outcome(row), "col": outcome(col), "flip": list(flip),
                             "flip_row": outcome(frow), "flip_col": outcome(fcol)})
    # acceptance_main.cpp:328-343 protocol (criterion 7), first 200 trials, and the
    # abft CLI loop (abed_main.cpp:436-453) for cli_test.cpp:139's arguments
    fails = missed = 0
    for t in range(200):
        rng = SplitMix64(derive_seed(0xC7, t))
        m, k, n = 1 + rng.below(64), 1 + rng.below(64), 1 + rng.below(64)
        a, b = rng.i8_matrix(m, k), rng.i8_matrix(k, n)
        _, ca, row, col = ref.abft_gemm(a, b)
        fails += row.status or col.status
        i, j = rng.below(m), rng.below(n)
        ca[i, j] ^= np.int64(1) << rng.below(63)
        r2, c2 = ref.abft_check(ca)
        missed += not (r2.status or c2.status)
    out["acceptance"] = {"root": 0xC7, "trials": 200, "faultfree_failures": fails, "missed": missed}
    out["costs"] = {"7x5x9": ref.abft_costs(7, 5, 9).tolist(), "7x5x9_single": ref.abft_costs(7, 5, 9, True).tolist(),
                    "16x12x20": ref.abft_costs(16, 12, 20).tolist()}
    with open(os.path.join(HERE, "abft.json"), "w") as fh:
        json.dump(out, fh, indent=1)
    print("wrote abft.json", len(out["cases"]), "cases", out["acceptance"])


if __name__ == "__main__":
    main()
