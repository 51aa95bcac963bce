"""GPU parity: every C-ABI entry point against the reference (golden vectors made
by the reference itself, tests/golden/golden.json) and the pinned C oracle, on
the same SplitMix64 inputs.  Bit-exact for all integer work and for the float
mode (the reference's sequential f32/f64 order is reproduced).  Runs on a B200.
"""
import hashlib
import json
import os

import numpy as np
import pytest
import torch

from oracle.pyoracle import Oracle
from paper_2006_04984_b200 import abi, api

pytestmark = pytest.mark.gpu
GOLDEN = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "golden.json")))
REF_KEYS = ("status", "locus", "lhs", "rhs", "lhs_f", "rhs_f")


def sha(t):
    a = t.cpu().numpy() if isinstance(t, torch.Tensor) else t
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def outcome(o):
    return {"status": o.status, "locus": list(o.locus) if o.has_locus else None, "lhs": o.lhs, "rhs": o.rhs,
            "lhs_f": o.lhs_f, "rhs_f": o.rhs_f}


@pytest.fixture(scope="module")
def ora():
    return Oracle("ora")


def device_data(ls, seed):
    """input = SplitMix64(derive_seed(seed,1)), filters = SplitMix64(derive_seed(seed,2)), generated on the GPU."""
    x = api.fill_random_i8(ls.n * ls.c * ls.h * ls.w, api.derive_seed(seed, 1)).view(ls.input_dims())
    f = api.fill_random_i8(ls.k * ls.c * ls.r * ls.s, api.derive_seed(seed, 2)).view(ls.filter_dims())
    return x, f


@pytest.mark.parametrize("case", GOLDEN["conv"], ids=lambda c: "x".join(map(str, c["dims"])))
def test_reference_functions_bit_exact(case, ora):
    ls = api.layer_shape(*case["dims"])
    x, f = device_data(ls, case["seed"])
    # device RNG == oracle RNG (index-parallel SplitMix64)
    xo = ora.random_i8(x.numel(), ora.derive_seed(case["seed"], 1))
    assert np.array_equal(x.cpu().numpy().ravel(), xo)
    conv = api.conv_direct(x, f, ls)
    assert sha(conv) == case["conv_sha"]
    bias = np.linspace(-3.0, 3.0, ls.k).astype(np.float32)
    assert sha(api.epilog(conv, 0.05, np.zeros(ls.k, np.float32))) == case["epilog_relu_sha"]
    assert sha(api.epilog(conv, 0.0123, bias)) == case["epilog_bias_sha"]
    assert sha(api.epilog(conv, 0.0123, bias, relu=False)) == case["epilog_ident_sha"]
    assert sha(api.epilog(conv, 0.0123, bias, relu=False, output_kind=api.F32)) == case["epilog_f32_sha"]
    fc = api.gen_filter_checksum(f)
    planes = api.decompose_checksum_filters(fc)
    extra = api.recombine_extra_fmaps(api.conv_checksum_planes(x, ls, planes))
    ic = api.gen_input_checksum(x, ls)
    batch = api.ic_batch_checksum(x)
    bext = api.conv_batch_checksum(batch, f, ls)  # tcgen05 digit-image route
    assert (sha(fc), sha(planes), sha(extra), sha(ic), sha(batch), sha(bext)) == (
        case["fc_sha"], case["planes_sha"], case["extra_sha"], case["ic_sha"], case["batch_sha"], case["batch_extra_sha"])
    assert torch.equal(api.conv_filter_checksum(x, ls, fc), extra)  # independent i64 route (checksum.hpp:201)
    assert api.fic_dot(fc, ic) == case["fic_dot"]
    got = {"fc": outcome(api.fc_verify(conv, extra)), "ic": outcome(api.ic_verify_k(conv, f, ic)),
           "icbatch": outcome(api.ic_batch_verify(conv, bext)), "fic": outcome(api.fic_verify(conv, case["fic_dot"]))}
    assert got == case["verify_pass"]
    bad = api.flip_bit(conv, case["flip"]["key"], case["flip"]["bit"])
    got = {"fc": outcome(api.fc_verify(bad, extra)), "ic": outcome(api.ic_verify_k(bad, f, ic)),
           "icbatch": outcome(api.ic_batch_verify(bad, bext)), "fic": outcome(api.fic_verify(bad, case["fic_dot"]))}
    assert got == case["verify_flip"]
    p = api.plan_precision(ls)
    assert {k: getattr(p, k) for k, _ in p._fields_} == case["plan"]
    if "fused" in case:
        out, cs, nic = api.fused_conv_epilog(x, f, ls, 0.02, bias, output_checksum=True,
                                             next_layer=api.layer_shape(ls.n, ls.k, ls.p, ls.q, 2, 3, 3, 1, 1, 1, 1))
        assert (sha(out), cs, sha(nic)) == (case["fused"]["out_sha"], case["fused"]["checksum"], case["fused"]["next_ic_sha"])


@pytest.mark.parametrize("case", GOLDEN["conv"], ids=lambda c: "x".join(map(str, c["dims"])))
def test_fused_protected_conv_matches_reference_verdicts(case):
    """The hot path: FC/FIC/IC verified inside the tcgen05 epilogue, fault-free and
    with the golden single ConvOut flip injected at the accumulator."""
    ls = api.layer_shape(*case["dims"])
    x, f = device_data(ls, case["seed"])
    plan = api.ConvPlan(ls, f, abi.CHECK_FC | abi.CHECK_FIC | abi.CHECK_IC)
    packed = plan.pack(x)
    out = torch.empty(ls.output_dims(), dtype=torch.int32, device="cuda")
    plan.run(packed, out, abi.OUT_I32_NCHW, ep=None)
    plan.finalize()
    fc, fic, ic = plan.outcomes()
    assert sha(out) == case["conv_sha"]
    vp = case["verify_pass"]
    assert (outcome(fc), outcome(fic), outcome(ic)) == (vp["fc"], vp["fic"], vp["ic"])
    plan.run(packed, out, abi.OUT_I32_NCHW, ep=None, fault_key=case["flip"]["key"], fault_bit=case["flip"]["bit"])
    plan.finalize()
    fc, fic, ic = plan.outcomes()
    vf = case["verify_flip"]
    assert (outcome(fc), outcome(fic), outcome(ic)) == (vf["fc"], vf["fic"], vf["ic"])
    # fused epilog output (bias + ReLU + requant) equals the reference epilog of the ConvOut
    bias = np.linspace(-3.0, 3.0, ls.k).astype(np.float32)
    y = torch.empty(ls.output_dims(), dtype=torch.int8, device="cuda")
    plan.run(packed, y, abi.OUT_I8_NCHW, scale=0.0123, bias=bias)
    assert sha(y) == case["epilog_bias_sha"]


@pytest.mark.parametrize("case", GOLDEN["float"], ids=lambda c: "x".join(map(str, c["dims"])))
def test_float_mode_bit_exact(case, ora):
    ls = api.layer_shape(*case["dims"])
    seed = case["seed"]
    if case["integers"]:
        x = ora.random_i8(ls.n * ls.c * ls.h * ls.w, seed).astype(np.float32).reshape(ls.input_dims())
        f = ora.random_i8(ls.k * ls.c * ls.r * ls.s, seed + 1).astype(np.float32).reshape(ls.filter_dims())
    else:
        x = ora.random_f32(ls.n * ls.c * ls.h * ls.w, ora.derive_seed(seed, 1)).reshape(ls.input_dims())
        f = ora.random_f32(ls.k * ls.c * ls.r * ls.s, ora.derive_seed(seed, 2)).reshape(ls.filter_dims())
    xd, fd = torch.from_numpy(x).cuda(), torch.from_numpy(f).cuda()
    conv = api.conv_direct_f32(xd, fd, ls)
    assert sha(conv) == case["conv_sha"]
    fs, ins = api.filter_checksum_f64(fd), api.input_checksum_f64(xd, ls)
    assert (sha(fs), sha(ins)) == (case["fs_sha"], case["is_sha"])
    exp = api.fic_dot_f64(fs, ins)
    lhs = api.reduce_all_f64(conv)
    assert lhs == float(np.add.accumulate(conv.cpu().numpy().ravel().astype(np.float64))[-1])  # sequential order
    tau = abs(lhs - exp)
    assert api.fic_verify_f32(conv, exp, tau).status == 0
    if tau > 0:
        assert api.fic_verify_f32(conv, exp, tau / 2).status == 1
    assert api.ic_verify_k_f32(conv, fd, ins, 1e-3).status == 0
    with pytest.raises(ValueError):
        api.float_verify(0.0, 0.0, -1.0)


def test_trials_match_reference():
    ls = api.layer_shape(1, 8, 12, 12, 8, 3, 3, 1, 1, 1, 1)
    xr, fr = device_data(ls, 4242)
    sets = {"ones": (torch.ones(ls.input_dims(), dtype=torch.int8, device="cuda"),
                     torch.ones(ls.filter_dims(), dtype=torch.int8, device="cuda")), "random": (xr, fr)}
    for t in GOLDEN["trials"]:
        x, f = sets[t["data"]]
        o = api.run_trial(ls, x, f, t["scheme"], t["target"], seed=t["seed"])
        got = {"classification": o.classification, "flat_index": o.flat_index, "bit": o.bit,
               "differs": o.final_output_differs, "verify": outcome(o.verify)}
        assert got == {k: t[k] for k in got}, t


@pytest.mark.parametrize("c", [c for c in GOLDEN["campaigns"]], ids=lambda c: f"{c['scheme']}-{c['target']}-{c['trials']}-{c['mode']}")
def test_campaign_counts_match_reference(c):
    """Includes the acceptance campaigns on the cfg1 layer (1000 trials each):
    FC filter 761/239/0/0, FC convout 932/68/0/0, FC input 0/0/743/257,
    FIC input 757/243/0/0, FIC filter 766/234/0/0, FIC convout 928/72/0/0."""
    ls = api.layer_shape(*c["dims"])
    r = api.run_campaign(ls, c["scheme"], c["target"], c["trials"], c["root_seed"], mode=c["mode"])
    assert [r.detected, r.detected_benign, r.sdc, r.masked] == c["counts"]


def test_campaign_sharding_is_deterministic():
    ls = api.layer_shape(1, 8, 12, 12, 8, 3, 3, 1, 1, 1, 1)
    whole = api.run_campaign(ls, abi.FIC, abi.TARGET_INPUT, 64, 4242, mode=abi.DATA_RANDOM_I8)
    parts = [api.run_campaign(ls, abi.FIC, abi.TARGET_INPUT, 64, 4242, mode=abi.DATA_RANDOM_I8, begin=b, end=e)
             for b, e in [(0, 13), (13, 40), (40, 64)]]
    assert whole.astuple() == tuple(map(sum, zip(*[p.astuple() for p in parts])))


def test_error_behaviour_mirrors_reference_exceptions():
    with pytest.raises(ValueError):
        api.layer_shape(0, 1, 1, 1, 1, 1, 1)
    with pytest.raises(ValueError):
        api.layer_shape(1, 1, 3, 3, 1, 5, 5)  # filter exceeds padded input
    wide = api.layer_shape(1, 131072, 1, 1, 1, 1, 1)
    with pytest.raises(ValueError):
        api.conv_direct(torch.zeros(wide.input_dims(), dtype=torch.int8, device="cuda"),
                        torch.zeros(wide.filter_dims(), dtype=torch.int8, device="cuda"), wide)
    t = torch.zeros((1, 1, 2, 2), dtype=torch.int32, device="cuda")
    with pytest.raises(IndexError):
        api.flip_bit(t, 4, 0)
    with pytest.raises(IndexError):
        api.flip_bit(t, 0, 32)
    assert api.flip_bit(t, 3, 31).flatten()[3].item() == -(2 ** 31)
    two = torch.full((1, 2, 1, 1), 10, dtype=torch.int32, device="cuda")
    with pytest.raises(ValueError):
        api.epilog(two, 1.0, [0.0])
    with pytest.raises(ValueError):
        api.epilog(two, float("inf"), [0.0, 0.0])
    ls = api.layer_shape(1, 1, 3, 3, 1, 3, 3)
    with pytest.raises(ValueError):
        api.run_trial(ls, torch.ones(ls.input_dims(), dtype=torch.int8, device="cuda"),
                      torch.ones(ls.filter_dims(), dtype=torch.int8, device="cuda"), abi.ICBATCH, abi.TARGET_FILTER)
    with pytest.raises(ValueError):
        api.run_campaign(ls, abi.FIC, abi.TARGET_CONVOUT, 0, 1)


def test_overflow_negative_control_on_gpu():
    # acceptance criterion 4: all-127 layer, true FIC sum 139,792,236,544; forced-32 falsely mismatches
    ls = api.layer_shape(1, 64, 16, 16, 64, 3, 3, 1, 1, 1, 1)
    x = torch.full(ls.input_dims(), 127, dtype=torch.int8, device="cuda")
    f = torch.full(ls.filter_dims(), 127, dtype=torch.int8, device="cuda")
    conv = api.conv_direct(x, f, ls)
    exp = api.fic_dot(api.gen_filter_checksum(f), api.gen_input_checksum(x, ls))
    assert exp == 139_792_236_544
    assert api.fic_verify(conv, exp).status == 0
    assert api.fic_verify_forced32(conv, exp).status == 1
    plan = api.ConvPlan(ls, f, abi.CHECK_FIC | abi.CHECK_FC)
    plan.run(plan.pack(x), None, abi.OUT_NONE, ep=None)
    plan.finalize()
    fc, fic, _ = plan.outcomes()
    assert fc.status == 0 and fic.status == 0 and fic.lhs == exp


def test_fic_convout_detection_exhaustive_on_gpu():
    # faults_test.cpp:189-206 through the fused kernel's accumulator fault hook
    ls = api.layer_shape(1, 2, 4, 4, 2, 3, 3, 1, 1, 1, 1)
    x, f = device_data(ls, 23)
    plan = api.ConvPlan(ls, f, abi.CHECK_FIC)
    packed = plan.pack(x)
    for idx in range(ls.nkpq()):
        for bit in range(32):
            plan.run(packed, None, abi.OUT_NONE, ep=None, fault_key=idx, fault_bit=bit)
            plan.finalize()
            assert plan.outcomes()[1].status == 1, (idx, bit)


def test_finalize_many_matches_per_plan_and_oracle(ora):
    # one verdict launch for a pass of several layers (abed_conv_plan_finalize_many)
    shapes = [(2, 64, 12, 12, 64, 3, 3, 1, 1, 1, 1), (1, 32, 9, 9, 256, 3, 3, 2, 2, 1, 1),
              (2, 16, 8, 8, 24, 1, 1, 1, 1, 0, 0)]
    plans, inputs = [], []
    for i, sh in enumerate(shapes):
        ls = api.layer_shape(*sh)
        x, f = device_data(ls, 40 + i)
        pl = api.ConvPlan(ls, f, abi.CHECK_FC | abi.CHECK_FIC)
        pl.run(pl.pack(x), None, abi.OUT_NONE, ep=None, fault_key=(5 if i == 1 else -1), fault_bit=30)
        plans.append(pl)
        inputs.append((ls, x, f))
    ps = api.PlanSet(plans)
    ps.finalize()
    many = ps.outcomes()
    for pl, got, (ls, x, f) in zip(plans, many, inputs):
        pl.finalize()
        one = pl.outcomes()
        for a, b in zip(got[:2], one[:2]):
            assert (a.status, a.has_locus, tuple(a.locus), a.lhs, a.rhs) == (b.status, b.has_locus, tuple(b.locus), b.lhs, b.rhs)
        xh, fh = x.cpu().numpy(), f.cpu().numpy()
        exp = ora.fic_dot(ora.gen_filter_checksum(fh), ora.gen_input_checksum(xh, ls))
        assert got[1].rhs == exp
    assert many[0][0].status == 0 and many[0][1].status == 0
    assert many[1][0].status == 1 and many[1][1].status == 1  # the injected ConvOut fault
    assert many[2][0].status == 0 and many[2][1].status == 0
