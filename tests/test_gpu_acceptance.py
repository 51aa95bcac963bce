"""The reference's acceptance criteria 1 and 6 (tests/acceptance/acceptance_main.cpp)
through the C ABI on the B200.

Criterion 1 (:59-128): every layer of the six builtin configs (vgg16 / resnet18 /
resnet50 at 224 and at 1080p capped to 64x64, network_config.hpp:310-316,
tensor.hpp:207) on the reference's seeds derive_seed(0xC1, (ci*1000 + li)*100 + s)
(input, then filters, from one SplitMix64 stream): fault-free FC, IC, ICBatch and
FIC verdicts all Pass -- all 20 seeds per layer, as the reference.

Criterion 6 (:285-316): 200 random small shapes from SplitMix64(0xC6) (n, c, k in
1..4, h, w in 1..8, 1x1 or 3x3, stride 1..2, pad 0..1) with the reference's data
(input then filters continuing the same stream): the fused tensor-core conv
equals the independent conv (torch f64 conv2d), the fused FC / FIC / IC verdicts
Pass."""
import ctypes as C
import json
import os

import pytest
import torch

from paper_2006_04984_b200 import abi, api
from splitmix import SplitMix64

pytestmark = pytest.mark.gpu
NETWORKS = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "networks.json")))["networks"]
SEEDS = 20


def protected_run(ls, x, f):
    plan = api.ConvPlan(ls, f, abi.CHECK_FC | abi.CHECK_FIC | abi.CHECK_IC)
    packed = plan.pack(x)
    out = torch.empty(ls.output_dims(), dtype=torch.int32, device="cuda")
    plan.run(packed, out, abi.OUT_I32_NCHW)
    plan.finalize()
    return out, plan.outcomes()


def units():
    for ci, net in enumerate(NETWORKS):
        cap = "1080p" in net["name"]
        for li, L in enumerate(net["layers"]):
            h, w = (min(L["h"], 64), min(L["w"], 64)) if cap else (L["h"], L["w"])
            dims = (L["n"], L["c"], h, w, L["k"], L["r"], L["s"], L["stride_h"], L["stride_w"], L["pad_h"], L["pad_w"])
            yield net["name"], ci, li, L["id"], dims


@pytest.mark.parametrize("net", [n["name"] for n in NETWORKS])
def test_criterion1_fault_free_identity_all_schemes(net):
    checked = 0
    for name, ci, li, lid, dims in units():
        if name != net:
            continue
        ls = api.layer_shape(*dims)
        for s in range(SEEDS):
            seed = api.derive_seed(0xC1, (ci * 1000 + li) * 100 + s)
            nx = ls.n * ls.c * ls.h * ls.w
            x = api.fill_random_i8(nx, seed).view(ls.input_dims())
            f = api.fill_random_i8(ls.k * ls.c * ls.r * ls.s, seed, nx).view(ls.filter_dims())
            out, (fc, fic, ic) = protected_run(ls, x, f)
            extra = api.conv_batch_checksum(api.ic_batch_checksum(x), f, ls)
            icb = api.ic_batch_verify(out, extra)
            assert (fc.status, fic.status, ic.status, icb.status) == (0, 0, 0, 0), (name, lid, s)
            assert fic.lhs == fic.rhs == int(out.to(torch.int64).sum())
            checked += 1
    assert checked > 0


def test_criterion6_random_shapes_exact():
    rng = SplitMix64(0xC6)
    checked = 0
    while checked < 200:
        n, c, k = 1 + rng.below(4), 1 + rng.below(4), 1 + rng.below(4)
        h, w = 1 + rng.below(8), 1 + rng.below(8)
        r = 3 if rng.below(2) else 1
        s = 3 if rng.below(2) else 1
        stride = 1 + rng.below(2)
        pad = rng.below(2)
        if r > h + 2 * pad or s > w + 2 * pad:
            continue
        ls = api.layer_shape(n, c, h, w, k, r, s, stride, stride, pad, pad)
        # input then filters continue the same stream (fill_random_i8, rng.hpp:46):
        # element i of a stream in state z is mix(z + (i+1) golden), so the device
        # fill from the current state reproduces the reference's data exactly
        nx, nf = n * c * h * w, k * c * r * s
        x = api.fill_random_i8(nx, rng.state).view(ls.input_dims())
        f = api.fill_random_i8(nf, rng.state, nx).view(ls.filter_dims())
        rng.state = (rng.state + (nx + nf) * 0x9E3779B97F4A7C15) % (1 << 64)
        out, (fc, fic, ic) = protected_run(ls, x, f)
        want = torch.nn.functional.conv2d(x.double(), f.double(), stride=stride, padding=pad).to(torch.int64)
        assert torch.equal(out.to(torch.int64), want), (n, c, h, w, k, r, s, stride, pad)
        assert (fc.status, fic.status, ic.status) == (0, 0, 0)
        checked += 1
