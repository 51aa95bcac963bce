"""Float-mode detection parity: the fused fp16 / bf16 tensor-core kernel's
thresholded FC / FIC verdicts against the reference's f32 verifiers
(fc_verify_f32 checksum.hpp:541-565, fic_verify_f32 :537-539, float_verify
:474-481; oracle restatements) on the SAME injected faults.

Data are small integers (|x|, |f| <= 8: exact in fp16 and bf16, every product
and partial sum exact in f32), so the tensor-core conv equals the reference's
conv_direct_f32 bit for bit and both sides judge the same corrupted ConvOut:
each trial flips one random bit of one random f32 ConvOut element (the paper's
single-value output corruption) inside the fused epilogue, and the reference
verifies the identically flipped tensor with the extra fmap
(conv_direct_f32 of the input with the f64 filter checksum as one filter) and
fic_dot_f64 of the pristine checksums.  Thresholds: the accumulation-error bound
of test_gpu_float_mode.  A trial is only excluded when the reference's
|lhs - rhs| lies within the GPU's stated summation error (2^-20 * sum|out|) of
tau -- an honest tie; the test reports how many and requires every other
verdict (and every FC locus) to be identical.
"""
import numpy as np
import pytest
import torch

from oracle.pyoracle import Oracle
from paper_2006_04984_b200 import abi, api

pytestmark = pytest.mark.gpu

KINDS = [abi.F16, abi.BF16]
SHAPES = [
    (2, 64, 12, 12, 64, 3, 3, 1, 1, 1, 1),
    (1, 32, 9, 11, 48, 3, 3, 2, 2, 1, 1),
    (2, 128, 6, 6, 256, 3, 3, 1, 1, 1, 1),  # several N tiles (in-kernel full-channel FC)
]


@pytest.fixture(scope="module")
def ora():
    return Oracle("ora")


def _taus(ora, ls, x, f):
    crs = ls.c * ls.r * ls.s
    absconv = ora.conv_f64(np.abs(x), np.abs(f), ls)
    tau_fc = float(np.max(absconv.sum(axis=1))) * (crs + ls.k + 32) * 2.0 ** -21
    tau_fic = float(absconv.sum()) * (crs + 32) * 2.0 ** -21
    return tau_fc, tau_fic


@pytest.mark.parametrize("kind", KINDS, ids=["fp16", "bf16"])
@pytest.mark.parametrize("shape", SHAPES, ids=lambda d: "x".join(map(str, d)))
def test_convout_flip_campaign_matches_reference_f32_verifiers(ora, kind, shape):
    ls = api.layer_shape(*shape)
    rng = np.random.default_rng(2024 + shape[1])
    x = rng.integers(-8, 9, ls.input_dims()).astype(np.float32)
    f = rng.integers(-8, 9, ls.filter_dims()).astype(np.float32)
    tau_fc, tau_fic = _taus(ora, ls, x, f)
    plan = api.ConvPlanH(ls, torch.from_numpy(f).cuda(), kind, abi.CHECK_FC | abi.CHECK_FIC, tau_fc, tau_fic)
    packed = plan.pack(torch.from_numpy(x).cuda())
    y = torch.empty(ls.output_dims(), dtype=torch.float32, device="cuda")

    # fault-free: the tensor-core conv is the reference's f32 conv exactly
    conv = ora.conv_f32(x, f, ls)
    plan.run(packed, y, abi.OUT_F32_NCHW, scale=1.0, relu=False)
    plan.finalize()
    assert np.array_equal(y.cpu().numpy(), conv)
    fc0, fic0, _ = plan.outcomes()
    assert fc0.status == 0 and fic0.status == 0

    # the reference's checksum side (pristine data)
    fs = ora.filter_checksum_f64(f)
    one = api.layer_shape(ls.n, ls.c, ls.h, ls.w, 1, ls.r, ls.s, ls.stride_h, ls.stride_w, ls.pad_h, ls.pad_w)
    extra = ora.conv_f32(x, fs.astype(np.float32).reshape(1, ls.c, ls.r, ls.s), one)
    expected = ora.fic_dot_f64(fs, ora.input_checksum_f64(x, ls))
    r0 = ora.fic_verify_f32(conv, expected, tau_fic)
    assert r0.status == 0

    trials, ties, agree = 160, 0, 0
    for t in range(trials):
        key = int(rng.integers(0, conv.size))
        bit = int(rng.integers(0, 32))
        plan.run(packed, y, abi.OUT_F32_NCHW, scale=1.0, relu=False, fault_key=key, fault_bit=bit)
        plan.finalize()
        fc, fic, _ = plan.outcomes()
        bad = conv.copy().reshape(-1)
        bad.view(np.uint32)[key] ^= np.uint32(1 << bit)
        bad = bad.reshape(conv.shape)
        rfc = ora.fc_verify_f32(bad, extra, tau_fc)
        rfic = ora.fic_verify_f32(bad, expected, tau_fic)
        # ties: the reference's margin to tau inside the GPU's summation error
        n, rem = divmod(key, ls.k * ls.p * ls.q)
        pq = rem % (ls.p * ls.q)
        with np.errstate(over="ignore", invalid="ignore"):
            row = np.abs(bad[n, :, pq // ls.q, pq % ls.q].astype(np.float64))
            eps_fc = 2.0 ** -20 * float(row.sum())
            eps_fic = 2.0 ** -20 * float(np.abs(bad.astype(np.float64)).sum())
            m_fc = abs(abs(rfc.lhs_f - rfc.rhs_f) - tau_fc) if rfc.status else None
            m_fic = abs(abs(rfic.lhs_f - rfic.rhs_f) - tau_fic)
        tie = (np.isfinite(eps_fc) and m_fc is not None and m_fc <= eps_fc) or \
              (np.isfinite(eps_fic) and np.isfinite(m_fic) and m_fic <= eps_fic)
        if tie:
            ties += 1
            continue
        assert (fc.status, fic.status) == (rfc.status, rfic.status), (t, key, bit, fc.lhs_f, fc.rhs_f, rfc.lhs_f,
                                                                       rfc.rhs_f, tau_fc)
        if fc.status:
            assert tuple(fc.locus) == tuple(rfc.locus)
        agree += 1
    assert ties <= trials // 50, f"{ties} ties of {trials}"
    assert agree + ties == trials
