"""FIC right-hand side taken from the staged activation tiles (ABED_RHS_STAGED)
versus a second read of the stored input (FR, the default): both must equal
the reference's fic_dot(gen_filter_checksum, gen_input_checksum)
(checksum.hpp:248-285) = the sum of the conv output on fault-free runs, across
strides, filter sizes, ragged channel counts, several N tiles and streamed
filters, and FIC must flag a single ConvOut fault."""
import ctypes as C

import pytest
import torch

from paper_2006_04984_b200 import abi

pytestmark = pytest.mark.gpu

SHAPES = [
    (1, 64, 56, 56, 64, 3, 3, 1, 1, 1, 1),    # cfg1
    (32, 64, 56, 56, 64, 3, 3, 1, 1, 1, 1),   # ResNet-50 layer1 at batch 32
    (4, 128, 56, 56, 128, 3, 3, 2, 2, 1, 1),  # layer2.0: stride 2 (4 phases)
    (8, 256, 14, 14, 256, 3, 3, 1, 1, 1, 1),  # layer3: two N tiles
    (4, 512, 7, 7, 512, 3, 3, 1, 1, 1, 1),    # layer4: streamed filters, 8 N tiles
    (3, 20, 13, 9, 24, 5, 5, 1, 1, 2, 2),     # 5x5, ragged channels
    (2, 48, 15, 17, 32, 1, 1, 2, 2, 0, 0),    # 1x1 stride 2 (one phase of two)
    (2, 16, 23, 23, 16, 7, 7, 2, 2, 3, 3),    # 7x7 stride 2
    (5, 32, 10, 10, 48, 3, 3, 1, 1, 0, 0),    # no padding
    (1, 3, 8, 8, 3, 3, 3, 2, 2, 1, 1),        # tiny, filler channels
]


def ref_conv(x, f, ls):
    y = torch.nn.functional.conv2d(x.double(), f.double(), stride=(ls.stride_h, ls.stride_w),
                                   padding=(ls.pad_h, ls.pad_w))
    return y.to(torch.int64)


def run(ls, xd, fd, checks, source, fault_key=-1, fault_bit=0):
    plan = C.c_void_p()
    abi.call("abed_conv_plan_create", C.byref(ls), fd.data_ptr(), checks, 0, C.byref(plan))
    abi.call("abed_conv_plan_set_input_checksum_source", plan, source)
    info = abi.PlanInfo()
    abi.call("abed_conv_plan_info", plan, C.byref(info))
    packed = torch.empty(info.packed_input_bytes, dtype=torch.int8, device="cuda")
    abi.call("abed_pack_input", plan, xd.data_ptr(), packed.data_ptr(), None)
    out = torch.empty(ls.output_dims(), dtype=torch.int32, device="cuda")
    oc = (abi.VerifyOutcome * 3)()
    od = torch.zeros(C.sizeof(oc), dtype=torch.uint8, device="cuda")
    for _ in range(2):  # a second run must start from reset accumulators
        abi.call("abed_conv_plan_run", plan, packed.data_ptr(), None, abi.OUT_I32_NCHW, out.data_ptr(), None,
                 fault_key, fault_bit, None)
        abi.call("abed_conv_plan_finalize", plan, od.data_ptr(), None)
    torch.cuda.synchronize()
    host = od.cpu().numpy()  # keep the host copy alive across the memmove
    C.memmove(oc, host.ctypes.data, C.sizeof(oc))
    abi.call("abed_conv_plan_destroy", plan)
    return out.cpu().to(torch.int64), oc


def data(dims, seed):
    ls = abi.layer_shape(*dims)
    g = torch.Generator().manual_seed(seed)
    x = torch.randint(-128, 128, ls.input_dims(), dtype=torch.int8, generator=g)
    f = torch.randint(-128, 128, ls.filter_dims(), dtype=torch.int8, generator=g)
    return ls, x, f


@pytest.mark.parametrize("checks", [abi.CHECK_FIC, abi.CHECK_FC | abi.CHECK_FIC])
@pytest.mark.parametrize("dims", SHAPES)
def test_staged_rhs_equals_reference(dims, checks):
    ls, x, f = data(dims, 31 + sum(dims))
    want = ref_conv(x, f, ls)
    total = int(want.sum())
    xd, fd = x.cuda(), f.cuda()
    for source in (abi.RHS_STAGED, abi.RHS_REREAD):
        got, oc = run(ls, xd, fd, checks, source)
        assert torch.equal(got, want)
        assert oc[1].status == 0 and oc[1].lhs == total == oc[1].rhs, (source, oc[1].lhs, oc[1].rhs, total)
        if checks & abi.CHECK_FC:
            assert oc[0].status == 0


@pytest.mark.parametrize("dims", SHAPES[:5])
def test_staged_rhs_all_extreme(dims):
    # all -128 inputs and filters: largest digit sums the dp4a accumulators see
    ls = abi.layer_shape(*dims)
    x = torch.full(ls.input_dims(), -128, dtype=torch.int8)
    f = torch.full(ls.filter_dims(), -128, dtype=torch.int8)
    want = ref_conv(x, f, ls)
    got, oc = run(ls, x.cuda(), f.cuda(), abi.CHECK_FIC, abi.RHS_STAGED)
    assert torch.equal(got, want)
    assert oc[1].status == 0 and oc[1].rhs == int(want.sum())


@pytest.mark.parametrize("dims", SHAPES[:4])
def test_staged_rhs_detects_convout_fault(dims):
    ls, x, f = data(dims, 77 + sum(dims))
    want = ref_conv(x, f, ls)
    key, bit = (want.numel() * 3) // 5, 17
    got, oc = run(ls, x.cuda(), f.cuda(), abi.CHECK_FIC, abi.RHS_STAGED, key, bit)
    assert oc[1].status == 1 and oc[1].rhs == int(want.sum()) and oc[1].lhs == int(got.sum())
    assert oc[1].lhs != oc[1].rhs
