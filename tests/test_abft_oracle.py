"""ABFT GEMM oracle (oracle/abed_oracle.c ora_abft_*) pinned to the reference:
the known-answer tests of abft_gemm_test.cpp, the golden vectors the reference
build wrote (tests/golden/abft.json), and -- where oracle/_ref exists -- live
agreement with the reference on random instances.  CPU only."""
import hashlib
import json
import os

import numpy as np
import pytest

from oracle.pyoracle import Oracle, ref_available
from splitmix import SplitMix64, derive_seed

GOLDEN = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "abft.json")))


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def outcome(o):
    return {"status": o.status, "locus": list(o.locus) if o.has_locus else None, "lhs": o.lhs, "rhs": o.rhs}


@pytest.fixture(scope="module")
def ora():
    return Oracle("ora")


def test_identity_passes(ora):  # abft_gemm_test.cpp:20-30
    eye = np.eye(2, dtype=np.int8)
    c, ca, row, col = ora.abft_gemm(eye, eye)
    assert row.status == 0 and col.status == 0
    assert c[0, 0] == 1 and c[0, 1] == 0 and c[1, 1] == 1
    assert ca[2, 2] == 2


def test_single_corruption_flags_row_and_column(ora):  # :32-47
    rng = SplitMix64(7)
    a, b = rng.i8_matrix(6, 5), rng.i8_matrix(5, 4)
    _, ca, row, col = ora.abft_gemm(a, b)
    assert row.status == 0 and col.status == 0
    ca[2, 3] ^= np.int64(1) << 17
    row, col = ora.abft_check(ca)
    assert row.status == 1 and col.status == 1
    assert row.locus[0] == 2 and col.locus[0] == 3


def test_checksum_row_matches_column_sum_oracle(ora):  # :49-71
    rng = SplitMix64(8)
    a, b = rng.i8_matrix(8, 8), rng.i8_matrix(8, 8)
    c, ca, row, col = ora.abft_gemm(a, b)
    want = a.astype(np.int64) @ b.astype(np.int64)
    assert np.array_equal(c, want)
    assert np.array_equal(ca[8, :8], want.sum(0)) and np.array_equal(ca[:8, 8], want.sum(1))


def test_fault_free_invariant_on_random_instances(ora):  # :73-85
    rng = SplitMix64(9)
    for _ in range(200):
        m, k, n = 1 + rng.below(16), 1 + rng.below(16), 1 + rng.below(16)
        a, b = rng.i8_matrix(m, k), rng.i8_matrix(k, n)
        _, _, row, col = ora.abft_gemm(a, b)
        assert row.status == 0 and col.status == 0, (m, k, n)


def test_guards(ora):  # :100-107 (inner mismatch) and the overflow guards :108-111
    from oracle.pyoracle import OracleError
    with pytest.raises(OracleError):
        ora.abft_gemm(np.zeros((2, 3), np.int8), np.zeros((4, 2), np.int8))
    with pytest.raises(OracleError):
        ora.abft_check(np.zeros((1, 5), np.int64))


@pytest.mark.parametrize("case", GOLDEN["cases"], ids=lambda c: f"{c['m']}x{c['k']}x{c['n']}")
def test_oracle_matches_reference_golden(case, ora):
    rng = SplitMix64(case["seed"])
    a, b = rng.i8_matrix(case["m"], case["k"]), rng.i8_matrix(case["k"], case["n"])
    c, ca, row, col = ora.abft_gemm(a, b)
    assert sha(c) == case["c_sha"] and sha(ca) == case["c_aug_sha"]
    assert outcome(row) == case["row"] and outcome(col) == case["col"]
    i, j, bit = case["flip"]
    ca[i, j] ^= np.int64(1) << bit
    row, col = ora.abft_check(ca)
    assert outcome(row) == case["flip_row"] and outcome(col) == case["flip_col"]


def test_acceptance_protocol_counts(ora):  # acceptance_main.cpp:328-343, first 200 trials
    fails = missed = 0
    for t in range(GOLDEN["acceptance"]["trials"]):
        rng = SplitMix64(derive_seed(0xC7, t))
        m, k, n = 1 + rng.below(64), 1 + rng.below(64), 1 + rng.below(64)
        a, b = rng.i8_matrix(m, k), rng.i8_matrix(k, n)
        _, ca, row, col = ora.abft_gemm(a, b)
        fails += row.status or col.status
        ca[rng.below(m), rng.below(n)] ^= np.int64(1) << rng.below(63)
        r2, c2 = ora.abft_check(ca)
        missed += not (r2.status or c2.status)
    assert (fails, missed) == (GOLDEN["acceptance"]["faultfree_failures"], GOLDEN["acceptance"]["missed"]) == (0, 0)


@pytest.mark.skipif(not ref_available(), reason="reference build (oracle/_ref) absent")
def test_oracle_equals_reference_live(ora):
    ref = Oracle("ref")
    rng = np.random.default_rng(5)
    for _ in range(40):
        m, k, n = (int(v) for v in rng.integers(1, 48, 3))
        a = rng.integers(-128, 128, (m, k)).astype(np.int8)
        b = rng.integers(-128, 128, (k, n)).astype(np.int8)
        x, y = ora.abft_gemm(a, b), ref.abft_gemm(a, b)
        assert np.array_equal(x[0], y[0]) and np.array_equal(x[1], y[1])
        ca = x[1].copy()
        ca[int(rng.integers(0, m + 1)), int(rng.integers(0, n + 1))] ^= np.int64(1) << int(rng.integers(0, 63))
        assert [outcome(o) for o in ora.abft_check(ca)] == [outcome(o) for o in ref.abft_check(ca)]
