"""Fused FC / FIC / IC checks of the protected tcgen05 conv: fault-free Pass and
single ConvOut-fault detection with the reference's locus semantics."""
import ctypes as C

import pytest
import torch

from paper_2006_04984_b200 import abi

pytestmark = pytest.mark.gpu

SHAPES = [
    (1, 64, 56, 56, 64, 3, 3, 1, 1, 1, 1),
    (2, 32, 9, 11, 16, 3, 3, 1, 1, 1, 1),
    (2, 4, 8, 8, 3, 3, 3, 2, 2, 1, 1),
    (2, 128, 14, 14, 256, 3, 3, 1, 1, 1, 1),
    (2, 256, 7, 7, 512, 3, 3, 1, 1, 1, 1),
]


def ref_conv(x, f, ls):
    y = torch.nn.functional.conv2d(x.double(), f.double(), stride=(ls.stride_h, ls.stride_w),
                                   padding=(ls.pad_h, ls.pad_w))
    return y.to(torch.int64)


def run(ls, x, f, checks, fault_key=-1, fault_bit=0):
    plan = C.c_void_p()
    xd, fd = x.cuda(), f.cuda()
    abi.call("abed_conv_plan_create", C.byref(ls), fd.data_ptr(), checks, 0, C.byref(plan))
    info = abi.PlanInfo()
    abi.call("abed_conv_plan_info", plan, C.byref(info))
    packed = torch.empty(info.packed_input_bytes, dtype=torch.int8, device="cuda")
    abi.call("abed_pack_input", plan, xd.data_ptr(), packed.data_ptr(), None)
    out = torch.empty(ls.output_dims(), dtype=torch.int32, device="cuda")
    abi.call("abed_conv_plan_run", plan, packed.data_ptr(), None, abi.OUT_I32_NCHW, out.data_ptr(), None,
             fault_key, fault_bit, None)
    oc = (abi.VerifyOutcome * 3)()
    od = torch.zeros(C.sizeof(oc), dtype=torch.uint8, device="cuda")
    abi.call("abed_conv_plan_finalize", plan, od.data_ptr(), None)
    torch.cuda.synchronize()
    host = od.cpu().numpy()
    C.memmove(oc, host.ctypes.data, C.sizeof(oc))
    abi.call("abed_conv_plan_destroy", plan)
    return out.cpu().to(torch.int64), oc


@pytest.mark.parametrize("dims", SHAPES)
def test_fault_free_pass(dims):
    ls = abi.layer_shape(*dims)
    g = torch.Generator().manual_seed(7 + sum(dims))
    x = torch.randint(-128, 128, ls.input_dims(), dtype=torch.int8, generator=g)
    f = torch.randint(-128, 128, ls.filter_dims(), dtype=torch.int8, generator=g)
    got, oc = run(ls, x, f, abi.CHECK_FC | abi.CHECK_FIC | abi.CHECK_IC)
    want = ref_conv(x, f, ls)
    assert torch.equal(got, want)
    assert oc[0].status == 0 and oc[0].lhs == 0 and oc[0].rhs == 0, "FC"
    assert oc[1].status == 0 and oc[1].lhs == int(want.sum()) == oc[1].rhs, "FIC"
    assert oc[2].status == 0, "IC"


@pytest.mark.parametrize("dims", SHAPES)
def test_convout_fault_detected(dims):
    ls = abi.layer_shape(*dims)
    g = torch.Generator().manual_seed(11 + sum(dims))
    x = torch.randint(-128, 128, ls.input_dims(), dtype=torch.int8, generator=g)
    f = torch.randint(-128, 128, ls.filter_dims(), dtype=torch.int8, generator=g)
    want = ref_conv(x, f, ls)
    nkpq = want.numel()
    key = (nkpq * 5) // 7
    bit = 9
    got, oc = run(ls, x, f, abi.CHECK_FC | abi.CHECK_FIC | abi.CHECK_IC, key, bit)
    flipped = want.flatten().clone()
    v = int(flipped[key]) & 0xFFFFFFFF
    v ^= 1 << bit
    flipped[key] = v - (1 << 32) if v >= 1 << 31 else v
    assert torch.equal(got.flatten(), flipped)
    n, k, p, q = ls.output_dims()
    ni, rem = divmod(key, k * p * q)
    ki, rem = divmod(rem, p * q)
    pi, qi = divmod(rem, q)
    conv = flipped.view(n, k, p, q)
    assert oc[0].status == 1 and tuple(oc[0].locus) == (ni, pi, qi)
    assert oc[0].lhs == int(conv[ni, :, pi, qi].sum()) and oc[0].rhs == int(want[ni, :, pi, qi].sum())
    assert oc[1].status == 1 and oc[1].lhs == int(conv.sum()) and oc[1].rhs == int(want.sum())
    assert oc[2].status == 1 and oc[2].locus[0] == ki


@pytest.mark.parametrize("dims", [(2, 128, 14, 14, 256, 3, 3, 1, 1, 1, 1), (2, 256, 7, 7, 512, 3, 3, 1, 1, 1, 1)])
def test_fc_several_n_tiles_fault_then_clean_run(dims):
    """FC across N tiles (per-tile flags, full-channel recheck in the verdict): a
    ConvOut fault is reported with the reference's full-row lhs / rhs, finalize is
    idempotent, and a later fault-free run on the same plan passes."""
    from paper_2006_04984_b200 import api
    ls = abi.layer_shape(*dims)
    g = torch.Generator().manual_seed(3 + sum(dims))
    x = torch.randint(-128, 128, ls.input_dims(), dtype=torch.int8, generator=g)
    f = torch.randint(-128, 128, ls.filter_dims(), dtype=torch.int8, generator=g)
    want = ref_conv(x, f, ls)
    plan = api.ConvPlan(ls, f.cuda(), abi.CHECK_FC)
    assert plan.info.n_tiles > 1
    packed = plan.pack(x.cuda())
    key, bit = (want.numel() * 3) // 5, 12
    n, k, p, q = ls.output_dims()
    ni, rem = divmod(key, k * p * q)
    pi, qi = divmod(rem % (p * q), q)
    out = torch.empty(ls.output_dims(), dtype=torch.int32, device="cuda")
    plan.run(packed, out, abi.OUT_I32_NCHW, fault_key=key, fault_bit=bit)
    plan.finalize()
    fc = plan.outcomes()[0]
    got = out.cpu().to(torch.int64)
    assert fc.status == 1 and tuple(fc.locus) == (ni, pi, qi) and fc.error_count == 1
    assert fc.lhs == int(got[ni, :, pi, qi].sum()) and fc.rhs == int(want[ni, :, pi, qi].sum())
    plan.finalize()
    again = plan.outcomes()[0]
    assert (again.status, tuple(again.locus), again.lhs, again.rhs) == (1, (ni, pi, qi), fc.lhs, fc.rhs)
    plan.run(packed, out, abi.OUT_I32_NCHW)
    plan.finalize()
    clean = plan.outcomes()[0]
    assert clean.status == 0 and clean.error_count == 0
    assert torch.equal(out.cpu().to(torch.int64), want)
