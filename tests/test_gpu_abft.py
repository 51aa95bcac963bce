"""GPU ABFT GEMM (csrc/abft.cu) against the reference: golden vectors written by
the reference build (tests/golden/abft.json), the known-answer tests of
abft_gemm_test.cpp and the acceptance protocol (acceptance_main.cpp:328-343),
all through the C ABI.  Bit-exact: c, c_aug and both VerifyOutcomes."""
import hashlib
import json
import os

import numpy as np
import pytest
import torch

from oracle.pyoracle import Oracle
from paper_2006_04984_b200 import abi, api
from splitmix import SplitMix64, derive_seed

pytestmark = pytest.mark.gpu
GOLDEN = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "abft.json")))


def sha(t):
    a = t.cpu().numpy() if isinstance(t, torch.Tensor) else t
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def outcome(o):
    return {"status": o.status, "locus": list(o.locus) if o.has_locus else None, "lhs": o.lhs, "rhs": o.rhs}


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def operands(case):
    rng = SplitMix64(case["seed"])
    return rng.i8_matrix(case["m"], case["k"]), rng.i8_matrix(case["k"], case["n"])


@pytest.mark.parametrize("case", GOLDEN["cases"], ids=lambda c: f"{c['m']}x{c['k']}x{c['n']}")
def test_abft_gemm_bit_exact(case):
    a, b = operands(case)
    c, ca, row, col = api.abft_gemm(dev(a), dev(b))
    assert sha(c) == case["c_sha"] and sha(ca) == case["c_aug_sha"]
    assert int(ca[case["m"], case["n"]]) == case["corner"]
    assert outcome(row) == case["row"] and outcome(col) == case["col"]
    i, j, bit = case["flip"]
    ca[i, j] ^= 1 << bit
    row, col = api.abft_check(ca)
    assert outcome(row) == case["flip_row"] and outcome(col) == case["flip_col"]
    assert row.error_count == 1 and col.error_count == 1


@pytest.mark.parametrize("case", GOLDEN["cases"][3:7], ids=lambda c: f"{c['m']}x{c['k']}x{c['n']}")
def test_abft_plan_modes(case):
    """Plan runs (stream-ordered, reused): the checked mode equals abft_gemm; the
    plain GEMM and the fused row check produce the same c; fused verdict passes."""
    a, b = (dev(x) for x in operands(case))
    m, n = case["m"], case["n"]
    plan = api.AbftPlan(m, n, case["k"])
    for _ in range(2):
        c = torch.full((m, n), -7, dtype=torch.int32, device="cuda")
        ca = torch.zeros((m + 1, n + 1), dtype=torch.int64, device="cuda")
        plan.run(a, b, c, ca, api.ABFT_CHECKED)
        row, col = plan.verdicts()
        assert sha(c) == case["c_sha"] and sha(ca) == case["c_aug_sha"]
        assert outcome(row) == case["row"] and outcome(col) == case["col"]
    for mode in (api.ABFT_PLAIN, api.ABFT_FUSED_ROW):
        c = torch.full((m, n), -7, dtype=torch.int32, device="cuda")
        plan.run(a, b, c, None, mode)
        torch.cuda.synchronize()
        assert sha(c) == case["c_sha"], mode
    row, col = plan.verdicts()
    assert row.status == 0 and col.status == 0


def test_known_answers():  # abft_gemm_test.cpp:20-47
    eye = torch.eye(2, dtype=torch.int8, device="cuda")
    c, ca, row, col = api.abft_gemm(eye, eye)
    assert row.status == 0 and col.status == 0 and int(ca[2, 2]) == 2
    assert c.cpu().tolist() == [[1, 0], [0, 1]]
    rng = SplitMix64(7)
    a, b = rng.i8_matrix(6, 5), rng.i8_matrix(5, 4)
    _, ca, row, col = api.abft_gemm(dev(a), dev(b))
    ca[2, 3] ^= 1 << 17
    row, col = api.abft_check(ca)
    assert (row.status, col.status, row.locus[0], col.locus[0]) == (1, 1, 2, 3)


def test_acceptance_protocol_on_gpu():  # acceptance_main.cpp:328-343 (first 200 trials)
    ora = Oracle("ora")
    fails = missed = 0
    for t in range(GOLDEN["acceptance"]["trials"]):
        rng = SplitMix64(derive_seed(0xC7, t))
        m, k, n = 1 + rng.below(64), 1 + rng.below(64), 1 + rng.below(64)
        a, b = rng.i8_matrix(m, k), rng.i8_matrix(k, n)
        c, ca, row, col = api.abft_gemm(dev(a), dev(b))
        fails += row.status or col.status
        if t % 25 == 0:  # spot-check against the oracle
            oc, oca, _, _ = ora.abft_gemm(a, b)
            assert np.array_equal(c.cpu().numpy(), oc) and np.array_equal(ca.cpu().numpy(), oca)
        ca[rng.below(m), rng.below(n)] ^= 1 << rng.below(63)
        r2, c2 = api.abft_check(ca)
        missed += not (r2.status or c2.status)
    assert (fails, missed) == (0, 0)


def test_guards():  # abft_gemm_test.cpp:100-107, abft_gemm.hpp:104-111
    with pytest.raises(abi.InvalidArgument):
        api.abft_gemm(torch.zeros((2, 3), dtype=torch.int8, device="cuda"),
                      torch.zeros((4, 2), dtype=torch.int8, device="cuda"))
    with pytest.raises(abi.InvalidArgument):
        api.abft_gemm(torch.zeros((2, 2), dtype=torch.int32, device="cuda"),
                      torch.zeros((2, 2), dtype=torch.int32, device="cuda"))
    with pytest.raises(abi.InvalidArgument):  # 16 + ceil_log2(k) > 31
        api.abft_gemm(torch.zeros((1, 40000), dtype=torch.int8, device="cuda"),
                      torch.zeros((40000, 1), dtype=torch.int8, device="cuda"))
    with pytest.raises(abi.InvalidArgument):
        api.abft_check(torch.zeros((1, 4), dtype=torch.int64, device="cuda"))
