"""First GPU parity check of the tcgen05 conv: abed_conv_i8 vs an exact float64 conv."""
import ctypes as C

import pytest
import torch

from paper_2006_04984_b200 import abi

pytestmark = pytest.mark.gpu

SHAPES = [
    (1, 64, 56, 56, 64, 3, 3, 1, 1, 1, 1),    # cfg1
    (2, 32, 9, 11, 16, 3, 3, 1, 1, 1, 1),
    (1, 8, 12, 12, 8, 3, 3, 1, 1, 1, 1),
    (2, 4, 8, 8, 3, 3, 3, 2, 2, 1, 1),
    (3, 128, 14, 14, 256, 3, 3, 1, 1, 1, 1),
    (2, 256, 7, 7, 512, 3, 3, 1, 1, 1, 1),
    (2, 64, 16, 16, 64, 1, 1, 1, 1, 0, 0),
    (2, 64, 16, 16, 128, 3, 3, 2, 2, 1, 1),
    (1, 16, 10, 10, 32, 5, 5, 1, 1, 2, 2),
]


def ref_conv(x, f, ls):
    y = torch.nn.functional.conv2d(x.double(), f.double(), stride=(ls.stride_h, ls.stride_w),
                                   padding=(ls.pad_h, ls.pad_w))
    return y.to(torch.int64)


@pytest.mark.parametrize("dims", SHAPES)
def test_conv_i8_matches_exact(dims):
    ls = abi.layer_shape(*dims)
    g = torch.Generator().manual_seed(sum(dims))
    x = torch.randint(-128, 128, ls.input_dims(), dtype=torch.int8, generator=g)
    f = torch.randint(-128, 128, ls.filter_dims(), dtype=torch.int8, generator=g)
    xd, fd = x.cuda(), f.cuda()
    out = torch.empty(ls.output_dims(), dtype=torch.int32, device="cuda")
    abi.call("abed_conv_i8", xd.data_ptr(), fd.data_ptr(), C.byref(ls), out.data_ptr(), None)
    torch.cuda.synchronize()
    want = ref_conv(x, f, ls)
    got = out.cpu().to(torch.int64)
    bad = (got != want).nonzero()
    assert bad.numel() == 0, f"{bad.shape[0]} mismatches, first {bad[:4].tolist()} got {got.flatten()[:8]} want {want.flatten()[:8]}"


PACK_SHAPES = SHAPES + [(2, 20, 13, 17, 16, 3, 3, 1, 1, 1, 1), (1, 16, 9, 6, 16, 1, 1, 1, 1, 0, 0),
                        (5, 6, 11, 24, 8, 3, 3, 2, 2, 1, 1), (3, 40, 9, 16, 16, 5, 5, 1, 1, 2, 2),
                        (4, 17, 6, 32, 8, 3, 3, 2, 1, 0, 1), (2, 16, 20, 24, 16, 3, 3, 3, 3, 1, 1),
                        (1, 8, 17, 32, 8, 5, 5, 3, 2, 2, 2), (6, 24, 10, 14, 16, 3, 3, 1, 1, 1, 1),
                        (3, 36, 9, 10, 8, 3, 3, 2, 2, 1, 1), (2, 16, 7, 6, 16, 1, 1, 1, 1, 0, 0)]


@pytest.mark.parametrize("ipb", [None, 2, 3])
@pytest.mark.parametrize("dims", PACK_SHAPES)
def test_pack_input_vector_path_equals_byte_path(dims, ipb, monkeypatch):
    """abed_pack_input's 8-, 4- and 2-column word paths (source aligned to 8 / 4 / 2
    bytes, rows a multiple of it) and its per-pixel gather (an odd address) give
    identical strip planes, also with several images per block (ABED_PACK_IPB), and
    the conv on them is exact."""
    from paper_2006_04984_b200 import api
    if ipb is not None:
        monkeypatch.setenv("ABED_PACK_IPB", str(ipb))
    ls = abi.layer_shape(*dims)
    g = torch.Generator().manual_seed(7 + sum(dims))
    x = torch.randint(-128, 128, ls.input_dims(), dtype=torch.int8, generator=g).cuda()
    f = torch.randint(-128, 128, ls.filter_dims(), dtype=torch.int8, generator=g).cuda()
    plan = api.ConvPlan(ls, f, 0)
    a = plan.pack(x, plan.packed_buffer())
    for shift in (4, 2, 1):
        raw = torch.empty(x.numel() + 8, dtype=torch.int8, device="cuda")
        raw[shift:shift + x.numel()].copy_(x.flatten())
        b = plan.packed_buffer()
        b.fill_(77)  # the pack writes every byte (halo, filler channels, plane tails)
        abi.call("abed_pack_input", plan.handle, raw.data_ptr() + shift, b.data_ptr(), None)
        torch.cuda.synchronize()
        assert torch.equal(a, b), shift
    out = torch.empty(ls.output_dims(), dtype=torch.int32, device="cuda")
    plan.run(a, out, abi.OUT_I32_NCHW)
    torch.cuda.synchronize()
    assert torch.equal(out.cpu().to(torch.int64), ref_conv(x.cpu(), f.cpu(), ls))


def _random_shapes(count, seed):
    g = torch.Generator().manual_seed(seed)
    out = []
    while len(out) < count:
        r = [1, 3, 5][int(torch.randint(0, 3, (1,), generator=g))]
        st = int(torch.randint(1, 3, (1,), generator=g))
        pad = int(torch.randint(0, r // 2 + 1, (1,), generator=g))
        h = int(torch.randint(max(r - 2 * pad, 1), 21, (1,), generator=g))
        w = int(torch.randint(max(r - 2 * pad, 1), 23, (1,), generator=g))
        c = int(torch.randint(1, 41, (1,), generator=g))
        k = int(torch.randint(1, 40, (1,), generator=g))
        n = int(torch.randint(1, 4, (1,), generator=g))
        out.append((n, c, h, w, k, r, r, st, st, pad, pad))
    return out


@pytest.mark.parametrize("dims", _random_shapes(24, 2026), ids=lambda d: "x".join(map(str, d)))
def test_pack_input_random_geometries(dims):
    """pack_input's staged transpose on random geometries (odd widths -> byte
    loads, widths % 4 == 0 -> word loads, stride 2 phases, 1x1 / 3x3 / 5x5, filler
    channels): both source paths give the same planes and the conv on them is exact."""
    from paper_2006_04984_b200 import api
    ls = abi.layer_shape(*dims)
    g = torch.Generator().manual_seed(sum(dims))
    x = torch.randint(-128, 128, ls.input_dims(), dtype=torch.int8, generator=g)
    f = torch.randint(-128, 128, ls.filter_dims(), dtype=torch.int8, generator=g)
    plan = api.ConvPlan(ls, f.cuda(), 0)
    a = plan.pack(x.cuda(), plan.packed_buffer())
    raw = torch.empty(x.numel() + 1, dtype=torch.int8, device="cuda")
    raw[1:].copy_(x.flatten().cuda())
    b = plan.packed_buffer()
    abi.call("abed_pack_input", plan.handle, raw.data_ptr() + 1, b.data_ptr(), None)
    torch.cuda.synchronize()
    assert torch.equal(a, b)
    out = torch.empty(ls.output_dims(), dtype=torch.int32, device="cuda")
    plan.run(a, out, abi.OUT_I32_NCHW)
    torch.cuda.synchronize()
    assert torch.equal(out.cpu().to(torch.int64), ref_conv(x, f, ls))
