"""Parity at the exact configurations bench.py times.

Every plan variant the bench measures is run here on the bench's own shapes,
epilog parameters and output layout, and its output is compared element for
element with the reference's CPU implementation (oracle/_ref: the unmodified
reference headers, detail::conv_fast_i8 + epilog, convolution.hpp:224,353):

* BASELINE configs[1]: all 16 ResNet-50 3x3 layers at batch 32, SplitMix64 data
  with the bench's seeds, scale 0.05, bias linspace(-2, 2), ReLU, int8 written
  into the packed layout (OUT_I8_PACKED) -- unprotected, FC, FIC (FR), FIC-SM
  (staged source), IC and ICBatch; FC/FIC/IC/ICBatch verdicts must pass and FIC's
  lhs = rhs = the reference's sum of the ConvOut;
* BASELINE configs[4] at one GPU: four layers (64 channels, stride 2, two N
  tiles, eight N tiles / streamed filters) at batch 1024;
* BASELINE configs[2]: VGG-16 conv1_2 / conv3_1 / conv5_1 at batch 64 in fp16
  and bf16 against an f64 conv of the rounded operands within the stated
  tolerance (|y - y_ref| <= 2^(1-p) |y_ref| + 2^-19 sum|x f|, p = 11 for fp16,
  8 for bf16: the output rounding, twice over for slack, plus the f32
  accumulation bound);
* BASELINE configs[3]: the five MobileNetV2 blocks at batch 32 chained through
  the packed layout, FIC on every layer; the block output equals the reference
  pointwise convs + epilogs around the depthwise restatement;
* the whole-network block: one ResNet-50 bottleneck chain per stage (1x1 -> 3x3
  -> 1x1 through the packed layout) with FIC and with FIC-AF, chain output and
  every layer's FIC lhs / rhs against the reference.

Integer outputs are bit-exact.  The packed output is unpacked from the identity
consumer's strip planes (conv_tc.cuh layout, Hl = P, Wl = Q, one phase).
"""
import concurrent.futures
import os

import numpy as np
import pytest
import torch

from bench import MBV2_BLOCKS, RESNET50_3X3, VGG16_3X3
from oracle.pyoracle import Oracle, ref_available
from paper_2006_04984_b200 import abi, api

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ref():
    if not ref_available():
        pytest.skip("oracle/_ref (the reference build) is not present")
    return Oracle("ref")


@pytest.fixture(scope="module")
def ora():
    return Oracle("ora")


def ref_conv(ref, x, f, ls, threads=None):
    """reference conv_fast_i8, the batch split over host threads (ctypes drops the GIL)."""
    threads = threads or min(ls.n, os.cpu_count() or 1)
    if threads <= 1 or ls.n == 1:
        return ref.conv_i8(x, f, ls)
    bounds = [ls.n * i // threads for i in range(threads + 1)]
    out = np.empty(ls.output_dims(), np.int32)

    def part(i):
        a, b = bounds[i], bounds[i + 1]
        if a == b:
            return
        sub = ref.layer_shape(b - a, ls.c, ls.h, ls.w, ls.k, ls.r, ls.s, ls.stride_h, ls.stride_w, ls.pad_h, ls.pad_w)
        out[a:b] = ref.conv_i8(x[a:b], f, sub)

    with concurrent.futures.ThreadPoolExecutor(threads) as ex:
        list(ex.map(part, range(threads)))
    return out


def ref_epilog(ref, conv, scale, bias, relu=True, threads=16):
    n = conv.shape[0]
    if n < threads:
        return ref.epilog(conv, scale, bias, relu)
    out = np.empty(conv.shape, np.int8)
    bounds = [n * i // threads for i in range(threads + 1)]

    def part(i):
        a, b = bounds[i], bounds[i + 1]
        if a < b:
            out[a:b] = ref.epilog(conv[a:b], scale, bias, relu)

    with concurrent.futures.ThreadPoolExecutor(threads) as ex:
        list(ex.map(part, range(threads)))
    return out


def identity_out_bytes(ls, elem=1):
    # bench.py's output buffer for the identity consumer of the packed layout
    return (ls.n * ((ls.k + 15) // 16 * 16) * (ls.p + 1) * (ls.q + 1) + (1 << 16)) * elem


def unpack_identity(buf: torch.Tensor, ls, cpg=16) -> torch.Tensor:
    """Strip planes of the identity consumer (1x1, stride 1, pad 0: Hl = P, Wl = Q)
    -> N x K x P x Q.  cpg channels per 16-byte pixel (16 int8, 8 fp16/bf16)."""
    c16 = -(-ls.k // cpg)
    c16 += c16 & 1
    m_total = ls.n * ls.p * ls.q
    plane_len = -(-m_total // 128) * 128
    esz = 16 // cpg
    v = buf[: c16 * plane_len * 16].view(c16, plane_len, cpg * esz)[:, :m_total]
    v = v.reshape(c16, ls.n, ls.p, ls.q, cpg, esz).permute(1, 0, 4, 2, 3, 5)
    return v.reshape(ls.n, c16 * cpg, ls.p, ls.q, esz)[:, : ls.k].contiguous()


def bench_layer_data(li, ls, rank=0):
    seed = 1000 * (rank + 1) + li  # bench.py run_ours
    x = api.fill_random_i8(ls.n * ls.c * ls.h * ls.w, api.derive_seed(seed, 1)).view(ls.input_dims())
    f = api.fill_random_i8(ls.k * ls.c * ls.r * ls.s, api.derive_seed(seed, 2)).view(ls.filter_dims())
    return x, f


VARIANTS = {
    "unprotected": (0, None),
    "fc": (abi.CHECK_FC, None),
    "fic": (abi.CHECK_FIC, abi.RHS_REREAD),
    "fic_sm": (abi.CHECK_FIC, abi.RHS_STAGED),
    "icbatch": (abi.CHECK_ICBATCH, None),
    "ic": (abi.CHECK_IC, None),
}


def run_bench_variants(ls, x, f, bias, variants, scale=0.05):
    """Each variant as bench.py runs it: OUT_I8_PACKED into the identity buffer,
    run twice (the second run must start from reset accumulators)."""
    res = {}
    for name in variants:
        checks, src = VARIANTS[name]
        plan = api.ConvPlan(ls, f, checks)
        if src is not None:
            plan.set_input_checksum_source(src)
        packed = plan.pack(x)
        out = torch.zeros(identity_out_bytes(ls), dtype=torch.int8, device="cuda")
        ep = plan.epilog_params(scale, bias, True)
        for _ in range(2):
            plan.run(packed, out, abi.OUT_I8_PACKED, ep=ep)
            if checks:
                plan.finalize()
        torch.cuda.synchronize()
        res[name] = (unpack_identity(out, ls).squeeze(-1).cpu().numpy(), plan.outcomes() if checks else None)
        del plan, packed, out
    return res


def check_variants(res, want_y, conv_sum):
    for name, (y, oc) in res.items():
        assert np.array_equal(y, want_y), f"{name}: output differs from the reference"
        checks = VARIANTS[name][0]
        if checks & abi.CHECK_FC:
            assert oc[0].status == 0, name
        if checks & abi.CHECK_FIC:
            assert oc[1].status == 0 and oc[1].lhs == oc[1].rhs == conv_sum, (name, oc[1].lhs, oc[1].rhs, conv_sum)
        if checks & (abi.CHECK_ICBATCH | abi.CHECK_IC):
            assert oc[2].status == 0 and oc[2].error_count == 0, name


@pytest.mark.parametrize("li", range(len(RESNET50_3X3)), ids=[f"{r[0]}-b32" for r in RESNET50_3X3])
def test_resnet50_b32_layer(ref, li):
    name, c, h, w, k, st = RESNET50_3X3[li]
    ls = api.layer_shape(32, c, h, w, k, 3, 3, st, st, 1, 1)
    x, f = bench_layer_data(li, ls)
    bias = torch.linspace(-2.0, 2.0, k).tolist()
    xh, fh = x.cpu().numpy(), f.cpu().numpy()
    conv = ref_conv(ref, xh, fh, ls)
    want = ref_epilog(ref, conv, 0.05, np.asarray(bias, np.float32))
    res = run_bench_variants(ls, x, f, bias, VARIANTS)
    check_variants(res, want, int(conv.astype(np.int64).sum()))


# layer1.0 (64 channels: unit-interleaved epilogue), layer2.0 (stride 2, 4 phases),
# layer3.1 (2 N tiles), layer4.1 (streamed B, 8 N tiles)
B1024 = [0, 3, 8, 14]


@pytest.mark.parametrize("li", B1024, ids=[f"{RESNET50_3X3[i][0]}-b1024" for i in B1024])
def test_resnet50_b1024_layer(ref, li):
    name, c, h, w, k, st = RESNET50_3X3[li]
    ls = api.layer_shape(1024, c, h, w, k, 3, 3, st, st, 1, 1)
    x, f = bench_layer_data(li, ls)
    bias = torch.linspace(-2.0, 2.0, k).tolist()
    xh, fh = x.cpu().numpy(), f.cpu().numpy()
    conv = ref_conv(ref, xh, fh, ls)
    want = ref_epilog(ref, conv, 0.05, np.asarray(bias, np.float32))
    res = run_bench_variants(ls, x, f, bias, ("unprotected", "fc", "fic", "icbatch"))
    check_variants(res, want, int(conv.astype(np.int64).sum()))


VGG_PICK = [0, 3, 9]  # conv1_2, conv3_1, conv5_1


@pytest.mark.parametrize("kind", [abi.F16, abi.BF16], ids=["fp16", "bf16"])
@pytest.mark.parametrize("vi", VGG_PICK, ids=[VGG16_3X3[i][0] + "-b64" for i in VGG_PICK])
def test_vgg16_b64_layer_tolerance(kind, vi):
    from oracle.pyoracle import round_bf16, round_f16
    name, c, hw, k = VGG16_3X3[vi]
    ls = api.layer_shape(64, c, hw, hw, k, 3, 3, 1, 1, 1, 1)
    gen = torch.Generator(device="cuda").manual_seed(2006_04984 + vi)
    x = torch.empty(ls.input_dims(), dtype=torch.float32, device="cuda").uniform_(-1, 1, generator=gen)
    f = torch.empty(ls.filter_dims(), dtype=torch.float32, device="cuda").uniform_(-1, 1, generator=gen) * 0.05
    sum_f = float(f.abs().sum())
    crs = c * 9
    tau_fc = (crs + k + 32) * 2.0 ** -22 * sum_f  # bench.py measure_vgg16_fp16
    tau_fic = (crs + 32) * 2.0 ** -22 * sum_f * ls.p * ls.q * 64
    plan = api.ConvPlanH(ls, f, kind, abi.CHECK_FC | abi.CHECK_FIC, tau_fc, tau_fic)
    packed = plan.pack(x)
    out = torch.zeros(identity_out_bytes(ls, 2), dtype=torch.int8, device="cuda")
    plan.run(packed, out, abi.OUT_H_PACKED, ep=plan.epilog_params(1.0, None, True))
    plan.finalize()
    torch.cuda.synchronize()
    fc, fic, _ = plan.outcomes()
    assert fc.status == 0 and fic.status == 0, (fc.lhs_f, fc.rhs_f, fic.lhs_f, fic.rhs_f)
    y16 = unpack_identity(out, ls, cpg=8)  # N x K x P x Q x 2 bytes
    bits = y16.view(torch.int16).squeeze(-1)
    y = (bits.view(torch.float16) if kind == abi.F16 else bits.view(torch.bfloat16)).float()
    rnd = round_f16 if kind == abi.F16 else round_bf16
    for img in (0, 63):  # f64 CPU conv of two images of the batch
        xi = torch.from_numpy(rnd(x[img:img + 1].cpu().numpy())).double()
        fr = torch.from_numpy(rnd(f.cpu().numpy())).double()
        want = torch.nn.functional.conv2d(xi, fr, padding=1).clamp_min(0.0)[0]
        mag = torch.nn.functional.conv2d(xi.abs(), fr.abs(), padding=1)[0]
        got = y[img].double().cpu()
        prec = 11 if kind == abi.F16 else 8  # significand bits of the 16-bit output
        tol = 2.0 ** (1 - prec) * want.abs() + 2.0 ** -19 * mag
        bad = (got - want).abs() > tol
        assert not bool(bad.any()), f"{name} image {img}: {int(bad.sum())} outputs outside the tolerance"


@pytest.mark.parametrize("bi", range(len(MBV2_BLOCKS)), ids=[f"block{i}-b32" for i in range(len(MBV2_BLOCKS))])
def test_mobilenetv2_block_b32(ref, ora, bi):
    ci, hw, t, co, st = MBV2_BLOCKS[bi]
    e = ci * t
    ho = (hw + 2 - 3) // st + 1
    shapes = [("pw", api.layer_shape(32, ci, hw, hw, e, 1, 1, 1, 1, 0, 0)),
              ("dw", api.layer_shape(32, e, hw, hw, e, 3, 3, st, st, 1, 1)),
              ("pw", api.layer_shape(32, e, ho, ho, co, 1, 1, 1, 1, 0, 0))]
    seed = 900 + 3 * bi  # bench.py measure_mobilenetv2_int8
    plans, filt = [], []
    for kind, ls in shapes:
        seed += 1
        if kind == "pw":
            f = api.fill_random_i8(ls.k * ls.c, api.derive_seed(seed, 2)).view(ls.filter_dims())
            plans.append(api.ConvPlan(ls, f, abi.CHECK_FIC))
        else:
            f = api.fill_random_i8(ls.c * 9, api.derive_seed(seed, 2)).view(ls.c, 1, 3, 3)
            plans.append(api.ConvPlanDW(ls, f, abi.CHECK_FIC))
        filt.append(f.cpu().numpy())
    ls0 = shapes[0][1]
    x = api.fill_random_i8(ls0.n * ci * hw * hw, api.derive_seed(seed, 1)).view(ls0.input_dims())
    bufs = [plans[0].pack(x), plans[1].packed_buffer(), plans[2].packed_buffer()]
    last = shapes[2][1]
    out = torch.zeros(identity_out_bytes(last), dtype=torch.int8, device="cuda")
    for i, pl in enumerate(plans):
        dst = bufs[i + 1] if i < 2 else out
        pl.run(bufs[i], dst, abi.OUT_I8_PACKED, ep=pl.epilog_params(0.02, None, True),
               next_plan=plans[i + 1] if i < 2 else None)
    ps = api.PlanSet(plans)
    ps.finalize()
    torch.cuda.synchronize()
    assert all(oc[1].status == 0 for oc in ps.outcomes())
    zero = lambda ls: np.zeros(ls.k, np.float32)  # noqa: E731
    h = x.cpu().numpy()
    for (kind, ls), fh in zip(shapes, filt):
        conv = ref_conv(ref, h, fh, ls) if kind == "pw" else ora.dwconv_i8(h, fh, ls)
        h = ref_epilog(ref, conv, 0.02, zero(ls))
    got = unpack_identity(out, last).squeeze(-1).cpu().numpy()
    assert np.array_equal(got, h)


# whole-network block (bench.py resnet50_network_int8): one bottleneck chain per
# stage -- conv1 1x1 -> conv2 3x3 (stride 2 at a stage's first block) -> conv3 1x1
# through the packed layout, FIC on every layer and FIC-AF (each in-chain layer's
# rhs accumulated by the producing epilogue); batch 4 keeps the CPU reference fast
CHAIN_PICK = [0, 4, 9, 16]  # layer1.0, layer2.0, layer3.0, layer4.0 bottlenecks
PROJ_PICK = [1, 5, 10, 17]   # the 1x1 projections (stride 2 from layer2 on, up to 2048 channels)


@pytest.mark.parametrize("variant", ["fic", "fic_af"])
@pytest.mark.parametrize("ci", CHAIN_PICK + PROJ_PICK, ids=lambda i: f"chain{i}")
def test_resnet50_bottleneck_chain(ref, ci, variant):
    from bench import resnet50_chains
    chain = resnet50_chains(4)[ci]
    if len(chain) == 1 and variant == "fic_af":
        pytest.skip("a single-layer chain has no producer epilogue to tap")
    plans, filt = [], []
    bias = []
    for li, ls in enumerate(chain):
        f = api.fill_random_i8(ls.k * ls.c * ls.r * ls.s, api.derive_seed(700 + 7 * ci + li, 2)).view(ls.filter_dims())
        pl = api.ConvPlan(ls, f, abi.CHECK_FIC)
        if variant == "fic_af" and li > 0:
            pl.set_af_input(True)
        plans.append(pl)
        filt.append(f.cpu().numpy())
        bias.append(np.linspace(-1.0, 1.0, ls.k).astype(np.float32))
    ls0 = chain[0]
    x = api.fill_random_i8(ls0.n * ls0.c * ls0.h * ls0.w, api.derive_seed(700 + 7 * ci, 1)).view(ls0.input_dims())
    nl = len(chain)
    bufs = [plans[0].pack(x)] + [plans[i].packed_buffer() for i in range(1, nl)]
    last = chain[-1]
    out = torch.zeros(identity_out_bytes(last), dtype=torch.int8, device="cuda")
    for i, pl in enumerate(plans):
        pl.run(bufs[i], bufs[i + 1] if i < nl - 1 else out, abi.OUT_I8_PACKED,
               ep=pl.epilog_params(0.02, bias[i].tolist(), True), next_plan=plans[i + 1] if i < nl - 1 else None)
    ps = api.PlanSet(plans)
    ps.finalize()
    torch.cuda.synchronize()
    h = x.cpu().numpy()
    sums = []
    for ls, fh, b in zip(chain, filt, bias):
        conv = ref_conv(ref, h, fh, ls)
        sums.append(int(conv.astype(np.int64).sum()))
        h = ref_epilog(ref, conv, 0.02, b)
    oc = ps.outcomes()
    for i in range(nl):  # FIC of every layer: pass, lhs = rhs = the reference's ConvOut sum
        assert oc[i][1].status == 0 and oc[i][1].lhs == oc[i][1].rhs == sums[i], (i, oc[i][1].lhs, sums[i])
    got = unpack_identity(out, last).squeeze(-1).cpu().numpy()
    assert np.array_equal(got, h)
