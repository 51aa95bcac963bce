"""Float mode on tensor cores (fp16 / bf16 operands, f32 accumulation) against the
oracle.

The reference's float mode (checksum.hpp:471-595) uses f32 operands, f64
reductions and absolute thresholds; it has no fp16/bf16 path, so this parity is
anchored on (a) the oracle's f64 restatement of conv_reference
(convolution.hpp:78-111) on operands rounded to the storage type, with an
accumulation-error tolerance stated per test, and (b) the reference's own f64
checksum functions (filter_checksum_f64, input_checksum_f64, fic_dot_f64,
reduce_all_f64 -- oracle restatements, pinned in test_oracle_golden.py) for the
FC / FIC values, and (c) float_verify semantics (Pass iff |lhs - rhs| <= tau).

Tolerances: a tensor-core f32 accumulation of CRS products differs from the f64
sum by at most ~CRS * 2^-24 * sum|x||f| per output; the tests allow
(CRS + 16) * 2^-22 * sum|x||f| (4x margin).
"""
import ctypes

import numpy as np
import pytest
import torch

from oracle.pyoracle import Oracle, round_bf16, round_f16
from paper_2006_04984_b200 import abi, api

pytestmark = pytest.mark.gpu

SHAPES = [
    # n, c, h, w, k, r, s, sh, sw, ph, pw
    (2, 64, 12, 12, 64, 3, 3, 1, 1, 1, 1),
    (1, 32, 9, 11, 48, 3, 3, 2, 2, 1, 1),
    (2, 13, 7, 7, 20, 3, 3, 1, 1, 1, 1),   # ragged channels (filler trim)
    (2, 24, 8, 8, 40, 1, 1, 1, 1, 0, 0),   # pointwise
    (1, 16, 10, 10, 16, 5, 5, 1, 1, 2, 2),
    (2, 128, 6, 6, 256, 3, 3, 1, 1, 1, 1),  # several N tiles
]
KINDS = [(abi.F16, round_f16), (abi.BF16, round_bf16)]


@pytest.fixture(scope="module")
def ora():
    return Oracle("ora")


def _data(ora, ls, seed, rnd):
    rng = np.random.default_rng(seed)
    x = rnd(rng.uniform(-1, 1, ls.input_dims()).astype(np.float32))
    f = rnd(rng.uniform(-1, 1, ls.filter_dims()).astype(np.float32))
    return x, f


def _tol(ora, ls, x, f):
    crs = ls.c * ls.r * ls.s
    absconv = ora.conv_f64(np.abs(x), np.abs(f), ls)
    return absconv * (crs + 16) * 2.0 ** -22 + 1e-30, absconv


@pytest.mark.parametrize("kind,rnd", KINDS)
@pytest.mark.parametrize("shape", SHAPES)
def test_conv_parity(ora, kind, rnd, shape):
    ls = api.layer_shape(*shape)
    x, f = _data(ora, ls, 11, rnd)
    plan = api.ConvPlanH(ls, torch.from_numpy(f).cuda(), kind)
    packed = plan.pack(torch.from_numpy(x).cuda())
    y = torch.empty(ls.output_dims(), dtype=torch.float32, device="cuda")
    plan.run(packed, y, abi.OUT_F32_NCHW, scale=1.0, bias=None, relu=False)
    want = ora.conv_f64(x, f, ls)
    tol, _ = _tol(ora, ls, x, f)
    err = np.abs(y.cpu().numpy().astype(np.float64) - want)
    assert np.all(err <= tol), f"max err {err.max()} vs tol {tol[np.unravel_index(err.argmax(), err.shape)]}"


@pytest.mark.parametrize("kind,rnd", KINDS)
def test_epilog_f32(ora, kind, rnd):
    ls = api.layer_shape(2, 64, 10, 10, 32, 3, 3, 1, 1, 1, 1)
    x, f = _data(ora, ls, 5, rnd)
    bias = np.linspace(-1, 1, ls.k).astype(np.float32)
    plan = api.ConvPlanH(ls, torch.from_numpy(f).cuda(), kind)
    y = torch.empty(ls.output_dims(), dtype=torch.float32, device="cuda")
    plan.run(plan.pack(torch.from_numpy(x).cuda()), y, abi.OUT_F32_NCHW, scale=0.25, bias=bias, relu=True)
    conv = ora.conv_f64(x, f, ls)
    want = np.maximum(conv * 0.25 + bias.reshape(1, -1, 1, 1), 0.0)
    tol, _ = _tol(ora, ls, x, f)
    assert np.all(np.abs(y.cpu().numpy() - want) <= 0.25 * tol + 1e-6)


def _checks_tau(ora, ls, x, f):
    """Thresholds from the accumulation-error bound (absolute, float_verify)."""
    tol, absconv = _tol(ora, ls, x, f)
    tau_fc = float(np.max(absconv.sum(axis=1))) * (ls.c * ls.r * ls.s + ls.k + 32) * 2.0 ** -21
    tau_fic = float(absconv.sum()) * (ls.c * ls.r * ls.s + 32) * 2.0 ** -21
    return tau_fc, tau_fic


@pytest.mark.parametrize("kind,rnd", KINDS)
@pytest.mark.parametrize("shape", [SHAPES[0], SHAPES[1], SHAPES[2], SHAPES[5]])
def test_fc_fic_fault_free_and_values(ora, kind, rnd, shape):
    ls = api.layer_shape(*shape)
    x, f = _data(ora, ls, 3, rnd)
    tau_fc, tau_fic = _checks_tau(ora, ls, x, f)
    plan = api.ConvPlanH(ls, torch.from_numpy(f).cuda(), kind, abi.CHECK_FC | abi.CHECK_FIC, tau_fc, tau_fic)
    y = torch.empty(ls.output_dims(), dtype=torch.float32, device="cuda")
    plan.run(plan.pack(torch.from_numpy(x).cuda()), y, abi.OUT_F32_NCHW, scale=1.0, relu=False)
    plan.finalize()
    fc, fic, _ = plan.outcomes()
    assert fc.status == 0, (fc.lhs_f, fc.rhs_f, tau_fc)
    assert fic.status == 0, (fic.lhs_f, fic.rhs_f, tau_fic)
    # FIC values against the reference's f64 checksum functions on the rounded data
    # fic_dot_f64 (checksum.hpp:530-535) is a plain f64 dot of the two checksums
    want_rhs = float(np.dot(ora.filter_checksum_f64(f), ora.input_checksum_f64(x, ls)))
    want_lhs = float(ora.conv_f64(x, f, ls).sum())
    assert abs(fic.rhs_f - want_rhs) <= tau_fic
    assert abs(fic.lhs_f - want_lhs) <= tau_fic


@pytest.mark.parametrize("kind,rnd", KINDS)
def test_fault_detection_vs_tau(ora, kind, rnd):
    ls = api.layer_shape(2, 64, 12, 12, 64, 3, 3, 1, 1, 1, 1)
    x, f = _data(ora, ls, 9, rnd)
    tau_fc, tau_fic = _checks_tau(ora, ls, x, f)
    plan = api.ConvPlanH(ls, torch.from_numpy(f).cuda(), kind, abi.CHECK_FC | abi.CHECK_FIC, tau_fc, tau_fic)
    packed = plan.pack(torch.from_numpy(x).cuda())
    y = torch.empty(ls.output_dims(), dtype=torch.float32, device="cuda")
    key = 5 * ls.p * ls.q + 3 * ls.q + 7  # (n=0, k=5, p=3, q=7)
    # an exponent flip that multiplies the f32 accumulator by >= 2^64: far above
    # tau -> both checks fire, FC reports the reference locus (n, p, q)
    # (fc_verify_f32, checksum.hpp:557-561)
    v = abs(ora.conv_f64(x, f, ls)[0, 5, 3, 7])
    bit = 30 if v < 2.0 else 29
    plan.run(packed, y, abi.OUT_F32_NCHW, fault_key=key, fault_bit=bit)
    plan.finalize()
    fc, fic, _ = plan.outcomes()
    assert fc.status == 1 and tuple(fc.locus) == (0, 3, 7)
    assert fic.status == 1
    # lowest mantissa bit: a change far below tau is (by float_verify) a pass
    plan.run(packed, y, abi.OUT_F32_NCHW, fault_key=key, fault_bit=0)
    plan.finalize()
    fc, fic, _ = plan.outcomes()
    assert fc.status == 0 and fic.status == 0


def test_tau_guards():
    ls = api.layer_shape(1, 16, 4, 4, 16, 3, 3, 1, 1, 1, 1)
    f = torch.zeros(ls.filter_dims(), dtype=torch.float32, device="cuda")
    with pytest.raises(abi.AbedError):
        api.ConvPlanH(ls, f, abi.F16, abi.CHECK_FIC, 0.0, -1.0)
    with pytest.raises(abi.AbedError):
        api.ConvPlanH(ls, f, abi.F16, abi.CHECK_IC, 0.0, 0.0)


@pytest.mark.parametrize("kind,rnd", KINDS)
def test_chained_16bit_output_and_duplication(ora, kind, rnd):
    ls = api.layer_shape(2, 32, 10, 10, 32, 3, 3, 1, 1, 1, 1)
    x, fa = _data(ora, ls, 21, rnd)
    _, fb = _data(ora, ls, 22, rnd)
    bias = np.linspace(-0.5, 0.5, ls.k).astype(np.float32)
    pa = api.ConvPlanH(ls, torch.from_numpy(fa).cuda(), kind)
    pb = api.ConvPlanH(ls, torch.from_numpy(fb).cuda(), kind)
    xa = pa.pack(torch.from_numpy(x).cuda())
    xb = pb.packed_buffer()
    pa.run(xa, xb, abi.OUT_H_PACKED, scale=0.5, bias=bias, relu=True, next_plan=pb)
    y = torch.empty(ls.output_dims(), dtype=torch.float32, device="cuda")
    pb.run(xb, y, abi.OUT_F32_NCHW)
    mid = rnd(np.maximum(ora.conv_f64(x, fa, ls) * 0.5 + bias.reshape(1, -1, 1, 1), 0.0).astype(np.float32))
    want = ora.conv_f64(mid, fb, ls)
    ulp = 2.0 ** -10 if kind == abi.F16 else 2.0 ** -7
    tol = ora.conv_f64(np.abs(mid), np.abs(fb), ls) * (4 * ulp)
    assert np.all(np.abs(y.cpu().numpy() - want) <= tol + 1e-6)
    # duplication baseline: a second identical run compares bit-equal
    pa.run(xa, xb, abi.OUT_H_COMPARE, scale=0.5, bias=bias, relu=True, next_plan=pb)
    n = ctypes.c_int64(-1)
    abi.call("abed_conv_plan_compare_count", pa.handle, ctypes.byref(n))
    assert n.value == 0
