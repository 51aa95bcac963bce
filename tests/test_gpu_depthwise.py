"""Depthwise INT8 conv (MobileNetV2, BASELINE configs[3]) against the oracle.

No reference counterpart (parity unpinned): the oracle restates
conv_reference (convolution.hpp:78-111) with one filter per channel; the FIC
identity is the reference's by linearity, so its rhs is checked against the
reference-pinned gen_input_checksum / fic_dot restatements with the depthwise
filter as the filter checksum.  All integer: bit-exact.
"""
import numpy as np
import pytest
import torch

from oracle.pyoracle import Oracle
from paper_2006_04984_b200 import abi, api

pytestmark = pytest.mark.gpu

DW_SHAPES = [
    # n, c, h, w, k(=c), r, s, sh, sw, ph, pw
    (2, 144, 14, 14, 144, 3, 3, 1, 1, 1, 1),
    (2, 96, 15, 13, 96, 3, 3, 2, 2, 1, 1),
    (1, 40, 9, 9, 40, 3, 3, 1, 1, 1, 1),   # ragged channel group
    (1, 32, 11, 11, 32, 5, 5, 1, 1, 2, 2),
]


@pytest.fixture(scope="module")
def ora():
    return Oracle("ora")


def data(ls, seed):
    x = api.fill_random_i8(ls.n * ls.c * ls.h * ls.w, api.derive_seed(seed, 1)).view(ls.input_dims())
    f = api.fill_random_i8(ls.c * ls.r * ls.s, api.derive_seed(seed, 2)).view(ls.c, 1, ls.r, ls.s)
    return x, f


@pytest.mark.parametrize("shape", DW_SHAPES)
def test_dwconv_bit_exact(ora, shape):
    ls = api.layer_shape(*shape)
    x, f = data(ls, 77)
    plan = api.ConvPlanDW(ls, f, abi.CHECK_FIC)
    packed = plan.pack(x)
    out = torch.empty(ls.output_dims(), dtype=torch.int32, device="cuda")
    plan.run(packed, out, abi.OUT_I32_NCHW, ep=None)
    xh, fh = x.cpu().numpy(), f.cpu().numpy()
    want = ora.dwconv_i8(xh, fh, ls)
    assert np.array_equal(out.cpu().numpy(), want)
    plan.finalize()
    fic = plan.outcomes()[1]
    # fic_dot(f as the filter checksum, gen_input_checksum) == sum of outputs
    rhs = ora.fic_dot(fh.reshape(-1).astype(np.int32), ora.gen_input_checksum(xh, ls))
    assert fic.status == 0 and fic.lhs == fic.rhs == rhs == int(want.astype(np.int64).sum())
    # epilog output
    bias = np.linspace(-2, 2, ls.k).astype(np.float32)
    y = torch.empty(ls.output_dims(), dtype=torch.int8, device="cuda")
    plan.run(packed, y, abi.OUT_I8_NCHW, scale=0.01, bias=bias, relu=True)
    assert np.array_equal(y.cpu().numpy(), ora.epilog(want, 0.01, bias))


def test_dw_fault_detection(ora):
    ls = api.layer_shape(2, 64, 10, 10, 64, 3, 3, 1, 1, 1, 1)
    x, f = data(ls, 5)
    plan = api.ConvPlanDW(ls, f, abi.CHECK_FIC)
    packed = plan.pack(x)
    for key, bit in [(0, 0), (ls.nkpq() // 2, 7), (ls.nkpq() - 1, 31)]:
        plan.run(packed, None, abi.OUT_NONE, ep=None, fault_key=key, fault_bit=bit)
        plan.finalize()
        assert plan.outcomes()[1].status == 1, (key, bit)
    plan.run(packed, None, abi.OUT_NONE, ep=None)
    plan.finalize()
    assert plan.outcomes()[1].status == 0
    with pytest.raises(abi.AbedError):
        api.ConvPlanDW(ls, f, abi.CHECK_FC)


def test_mobilenet_block_chained(ora):
    """pw expand (tensor cores) -> dw 3x3 (CUDA cores) -> pw project, every
    layer FIC-protected, activations handed over in the packed layout."""
    n, c, hw, t = 2, 24, 14, 6
    e = c * t
    pw1 = api.layer_shape(n, c, hw, hw, e, 1, 1, 1, 1, 0, 0)
    dw = api.layer_shape(n, e, hw, hw, e, 3, 3, 1, 1, 1, 1)
    pw2 = api.layer_shape(n, e, hw, hw, c, 1, 1, 1, 1, 0, 0)
    x, _ = data(pw1, 1)
    f1 = api.fill_random_i8(e * c, api.derive_seed(2, 2)).view(pw1.filter_dims())
    _, fd = data(dw, 3)
    f2 = api.fill_random_i8(c * e, api.derive_seed(4, 2)).view(pw2.filter_dims())
    p1 = api.ConvPlan(pw1, f1, abi.CHECK_FIC)
    pd = api.ConvPlanDW(dw, fd, abi.CHECK_FIC)
    p2 = api.ConvPlan(pw2, f2, abi.CHECK_FIC)
    b1 = np.linspace(-1, 1, e).astype(np.float32)
    bd = np.linspace(-1, 1, e).astype(np.float32)
    b2 = np.linspace(-1, 1, c).astype(np.float32)
    a1 = p1.pack(x)
    a2 = pd.packed_buffer()
    a3 = p2.packed_buffer()
    p1.run(a1, a2, abi.OUT_I8_PACKED, scale=0.02, bias=b1, relu=True, next_plan=pd)
    pd.run(a2, a3, abi.OUT_I8_PACKED, scale=0.03, bias=bd, relu=True, next_plan=p2)
    y = torch.empty(pw2.output_dims(), dtype=torch.int8, device="cuda")
    p2.run(a3, y, abi.OUT_I8_NCHW, scale=0.02, bias=b2, relu=False)
    ps = api.PlanSet([p1, pd, p2])
    ps.finalize()
    assert all(oc[1].status == 0 for oc in ps.outcomes())
    xh = x.cpu().numpy()
    h1 = ora.epilog(ora.conv_i8(xh, f1.cpu().numpy(), pw1), 0.02, b1)
    h2 = ora.epilog(ora.dwconv_i8(h1, fd.cpu().numpy(), dw), 0.03, bd)
    want = ora.epilog(ora.conv_i8(h2, f2.cpu().numpy(), pw2), 0.02, b2, relu=False)
    assert np.array_equal(y.cpu().numpy(), want)


def _flip_packed_byte(buf, plan, n, c, h, w, bit):
    """Flip one bit of input element (n, c, h, w) inside a plan's packed buffer
    (stride-1 geometry: plane c//16, pixel (n*Hl + h+pad)*Wl + w+pad)."""
    info = plan.info
    ls = plan.ls
    t = (n * info.Hl + h + ls.pad_h) * info.Wl + w + ls.pad_w
    plane_len = info.packed_input_bytes // 16 // (info.n_phase * ((ls.c + 15) // 16 + ((ls.c + 15) // 16) % 2))
    off = ((c // 16) * plane_len + t) * 16 + c % 16
    v = buf[off].item()
    buf[off] = ((v & 0xFF) ^ (1 << bit)) - 256 if ((v & 0xFF) ^ (1 << bit)) > 127 else (v & 0xFF) ^ (1 << bit)


@pytest.mark.parametrize("second_stride", [1, 2])
def test_fic_af_chain_values_and_between_layer_fault(ora, second_stride):
    """FIC-AF (fused_conv_epilog's next-layer input-checksum tap): the consumer's
    rhs accumulated in the producer's epilogue equals the FR value; a bit flip in
    the stored activation between the layers is caught by AF and missed by FR."""
    l1 = api.layer_shape(2, 64, 12, 12, 64, 3, 3, 1, 1, 1, 1)
    l2 = api.layer_shape(2, 64, 12, 12, 48, 3, 3, second_stride, second_stride, 1, 1)
    x, _ = data(l1, 61)
    f1 = api.fill_random_i8(l1.k * l1.c * 9, api.derive_seed(61, 2)).view(l1.filter_dims())
    f2 = api.fill_random_i8(l2.k * l2.c * 9, api.derive_seed(62, 2)).view(l2.filter_dims())
    p1 = api.ConvPlan(l1, f1, abi.CHECK_FIC)
    p2 = api.ConvPlan(l2, f2, abi.CHECK_FIC)
    bias = np.linspace(-2, 2, 64).astype(np.float32)
    a1 = p1.pack(x)
    a2 = p2.packed_buffer()
    # FR reference run of layer 2
    p1.run(a1, a2, abi.OUT_I8_PACKED, scale=0.02, bias=bias, relu=True, next_plan=p2)
    p2.run(a2, None, abi.OUT_NONE, ep=None)
    p2.finalize()
    fr = p2.outcomes()[1]
    # AF: the same pass with layer 2's rhs from layer 1's epilogue
    p2.set_af_input(True)
    p1.run(a1, a2, abi.OUT_I8_PACKED, scale=0.02, bias=bias, relu=True, next_plan=p2)
    p2.run(a2, None, abi.OUT_NONE, ep=None)
    p2.finalize()
    af = p2.outcomes()[1]
    h1 = ora.epilog(ora.conv_i8(x.cpu().numpy(), f1.cpu().numpy(), l1), 0.02, bias)
    want = ora.fic_dot(ora.gen_filter_checksum(f2.cpu().numpy()), ora.gen_input_checksum(h1, l2))
    assert fr.status == 0 and af.status == 0 and fr.rhs == af.rhs == want
    # finalize consumed the AF accumulator: a second pass gives the same verdict
    p1.run(a1, a2, abi.OUT_I8_PACKED, scale=0.02, bias=bias, relu=True, next_plan=p2)
    p2.run(a2, None, abi.OUT_NONE, ep=None)
    p2.finalize()
    assert p2.outcomes()[1].status == 0 and p2.outcomes()[1].rhs == want
    # corrupt the stored activation between the layers (an interior element that layer 2 reads)
    p1.run(a1, a2, abi.OUT_I8_PACKED, scale=0.02, bias=bias, relu=True, next_plan=p2)
    _flip_packed_byte(a2, p2, 1, 5, 4, 6, 6)
    p2.run(a2, None, abi.OUT_NONE, ep=None)
    p2.finalize()
    assert p2.outcomes()[1].status == 1, "AF must detect the corrupted activation"
    p2.set_af_input(False)
    p2.run(a2, None, abi.OUT_NONE, ep=None)  # FR re-reads the corrupted input: consistent, passes
    p2.finalize()
    assert p2.outcomes()[1].status == 0


def test_mobilenet_block_af(ora):
    n, c, hw, t = 2, 24, 14, 6
    e = c * t
    pw1 = api.layer_shape(n, c, hw, hw, e, 1, 1, 1, 1, 0, 0)
    dw = api.layer_shape(n, e, hw, hw, e, 3, 3, 1, 1, 1, 1)
    pw2 = api.layer_shape(n, e, hw, hw, c, 1, 1, 1, 1, 0, 0)
    x, _ = data(pw1, 11)
    f1 = api.fill_random_i8(e * c, api.derive_seed(12, 2)).view(pw1.filter_dims())
    _, fd = data(dw, 13)
    f2 = api.fill_random_i8(c * e, api.derive_seed(14, 2)).view(pw2.filter_dims())
    p1, pd, p2 = api.ConvPlan(pw1, f1, abi.CHECK_FIC), api.ConvPlanDW(dw, fd, abi.CHECK_FIC), api.ConvPlan(pw2, f2, abi.CHECK_FIC)
    pd.set_af_input(True)
    p2.set_af_input(True)
    b1, bd, b2 = (np.linspace(-1, 1, k).astype(np.float32) for k in (e, e, c))
    a1, a2, a3 = p1.pack(x), pd.packed_buffer(), p2.packed_buffer()
    p1.run(a1, a2, abi.OUT_I8_PACKED, scale=0.02, bias=b1, relu=True, next_plan=pd)
    pd.run(a2, a3, abi.OUT_I8_PACKED, scale=0.03, bias=bd, relu=True, next_plan=p2)
    p2.run(a3, None, abi.OUT_NONE, ep=None)
    ps = api.PlanSet([p1, pd, p2])
    ps.finalize()
    oc = ps.outcomes()
    xh = x.cpu().numpy()
    h1 = ora.epilog(ora.conv_i8(xh, f1.cpu().numpy(), pw1), 0.02, b1)
    h2 = ora.epilog(ora.dwconv_i8(h1, fd.cpu().numpy(), dw), 0.03, bd)
    assert all(o[1].status == 0 for o in oc)
    assert oc[1][1].rhs == ora.fic_dot(fd.cpu().numpy().reshape(-1).astype(np.int32), ora.gen_input_checksum(h1, dw))
    assert oc[2][1].rhs == ora.fic_dot(ora.gen_filter_checksum(f2.cpu().numpy()), ora.gen_input_checksum(h2, pw2))
