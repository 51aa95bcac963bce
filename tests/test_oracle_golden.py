"""Pins the C oracle (oracle/abed_oracle.c) before it is trusted as the GPU checker:

* against the reference's own known-answer tests (the assertions of
  /root/reference/proj/tests/{convolution,checksum,faults}_test.cpp restated), and
* against golden vectors produced by the reference implementation itself
  (tests/golden/golden.json, written by tests/golden/make_golden.py from oracle/_ref).
CPU only.
"""
import hashlib
import json
import os

import numpy as np
import pytest

from oracle.pyoracle import Oracle, ref_available

GOLDEN = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "golden.json")))


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


@pytest.fixture(scope="module")
def ora():
    return Oracle("ora")


def outcome(o):
    return {"status": o.status, "locus": list(o.locus) if o.has_locus else None, "lhs": o.lhs, "rhs": o.rhs,
            "lhs_f": o.lhs_f, "rhs_f": o.rhs_f}


def data(o, ls, seed):
    x = o.random_i8(ls.n * ls.c * ls.h * ls.w, o.derive_seed(seed, 1)).reshape(ls.input_dims())
    f = o.random_i8(ls.k * ls.c * ls.r * ls.s, o.derive_seed(seed, 2)).reshape(ls.filter_dims())
    return x, f


# ------------------------------------------------------------------ known answers
def test_conv_ones_window_and_linear_scaling(ora):
    # convolution_test.cpp:21-40
    ls = ora.layer_shape(1, 1, 3, 3, 1, 3, 3)
    assert ora.conv_i8(np.ones(ls.input_dims(), np.int8), np.ones(ls.filter_dims(), np.int8), ls).ravel().tolist() == [9]
    ls = ora.layer_shape(1, 1, 3, 3, 2, 3, 3)
    f = np.ones(ls.filter_dims(), np.int8)
    f[1] = 2
    assert ora.conv_i8(np.ones(ls.input_dims(), np.int8), f, ls).ravel().tolist() == [9, 18]


def test_conv_width_guard(ora):
    # convolution_test.cpp:50-60 (CRS > 65536 rejected)
    ls = ora.layer_shape(1, 131072, 1, 1, 1, 1, 1)
    with pytest.raises(Exception):
        ora.conv_i8(np.zeros(ls.input_dims(), np.int8), np.zeros(ls.filter_dims(), np.int8), ls)


def test_epilog_known_answers(ora):
    # convolution_test.cpp:208-246
    one = lambda v: np.array([v], np.int32).reshape(1, 1, 1, 1)
    assert ora.epilog(one(9), 1.0, [0.0])[0, 0, 0, 0] == 9
    assert ora.epilog(one(-5), 1.0, [0.0])[0, 0, 0, 0] == 0
    assert ora.epilog(one(300), 1.0, [0.5])[0, 0, 0, 0] == 127
    assert ora.epilog(one(-5), 0.5, [0.0], relu=False)[0, 0, 0, 0] == -2
    assert ora.epilog(one(5), 0.5, [0.0], relu=False)[0, 0, 0, 0] == 2
    two = np.full((1, 2, 1, 1), 10, np.int32)
    out = ora.epilog(two, 0.25, [0.5, -100.0], relu=False, out_f32=True).ravel()
    assert out.tolist() == [3.0, -97.5]
    with pytest.raises(Exception):
        ora.epilog(two, 1.0, [0.0])  # bias length
    with pytest.raises(Exception):
        ora.epilog(two, float("inf"), [0.0, 0.0])


def test_epilog_fma_probe(ora):
    # the reference's -march=native build returns 35 (FMA), 36 without
    acc = np.array([-21774], np.int32).reshape(1, 1, 1, 1)
    assert ora.epilog(acc, float.fromhex("0x1.cbe6dap-11"), [float.fromhex("0x1.b8ccccp+5")])[0, 0, 0, 0] == 35


def test_filter_checksum_and_decompose(ora):
    # checksum_test.cpp:29-69
    f = np.ones((2, 1, 3, 3), np.int8)
    f[1] = 2
    assert (ora.gen_filter_checksum(f) == 3).all()
    planes = ora.decompose_checksum_filters(np.array([0, 0x12345678], np.int32))
    assert planes[:, 0].tolist() == [0, 0, 0, 0]
    assert [int(v) & 0xFF for v in planes[:, 1]] == [0x78, 0x56, 0x34, 0x12]
    # round trip of extremes and random words through decompose -> planes conv == direct
    vals = np.array([0, -2**31, 2**31 - 1, 255, 256, -1, -256, 0x7F000000], np.int32)
    planes = ora.decompose_checksum_filters(vals)
    rec = (planes[0].view(np.uint8).astype(np.int64) + (planes[1].view(np.uint8).astype(np.int64) << 8)
           + (planes[2].view(np.uint8).astype(np.int64) << 16) + (planes[3].astype(np.int64) << 24))
    assert rec.tolist() == vals.tolist()


def test_fc_worked_example_and_flip(ora):
    # checksum_test.cpp:152-169
    ls = ora.layer_shape(1, 1, 3, 3, 2, 3, 3)
    x = np.ones(ls.input_dims(), np.int8)
    f = np.ones(ls.filter_dims(), np.int8)
    f[1] = 2
    conv = ora.conv_i8(x, f, ls)
    extra = ora.recombine_extra_fmaps(ora.conv_checksum_planes(x, ls, ora.decompose_checksum_filters(ora.gen_filter_checksum(f))))
    assert extra.ravel().tolist() == [27]
    assert ora.fc_verify(conv, extra).status == 0
    conv.ravel()[0] ^= 1 << 4
    bad = ora.fc_verify(conv, extra)
    assert bad.status == 1 and list(bad.locus) == [0, 0, 0]


def test_input_checksum_and_fic_worked_example(ora):
    # checksum_test.cpp:210-251
    ls = ora.layer_shape(1, 1, 3, 3, 2, 3, 3)
    x = np.ones(ls.input_dims(), np.int8)
    f = np.ones(ls.filter_dims(), np.int8)
    f[1] = 2
    ic = ora.gen_input_checksum(x, ls)
    assert (ic == 1).all()
    assert ora.fic_dot(ora.gen_filter_checksum(f), ic) == 27


def test_plan_precision_table_rows(ora):
    # checksum_test.cpp:381-419
    p = ora.plan_precision(ora.layer_shape(1, 64, 56, 56, 64, 3, 3, 1, 1, 1, 1))
    assert (p.bits_output_fmap, p.bits_reduced_fc, p.bits_filter_checksum, p.bits_input_checksum, p.bits_reduced_fic) == (26, 32, 14, 20, 43)
    assert p.reduced_fic_kind == 2  # I64
    assert ora.plan_precision(ora.layer_shape(1, 65536, 1, 1, 1, 1, 1)).bits_output_fmap == 32
    d = ora.plan_precision(ora.layer_shape(1, 1, 1, 1, 1, 1, 1))
    assert (d.bits_output_fmap, d.bits_reduced_fic, d.reduced_fic_kind) == (16, 16, 1)
    with pytest.raises(Exception):
        ora.plan_precision(ora.layer_shape(1, 1, 3, 3, 1, 3, 3), 16)
    with pytest.raises(Exception):
        ora.plan_precision(ora.layer_shape(16, 1024, 8192, 8192, 1024, 1, 1))


def test_overflow_negative_control(ora):
    # checksum_test.cpp:471-501; acceptance criterion 4 (true sum 139,792,236,544)
    ls = ora.layer_shape(1, 64, 16, 16, 64, 3, 3, 1, 1, 1, 1)
    x = np.full(ls.input_dims(), 127, np.int8)
    f = np.full(ls.filter_dims(), 127, np.int8)
    conv = ora.conv_i8(x, f, ls)
    expected = ora.fic_dot(ora.gen_filter_checksum(f), ora.gen_input_checksum(x, ls))
    assert expected == 139_792_236_544
    assert ora.fic_verify(conv, expected).status == 0
    assert ora.fic_verify(conv, expected, forced32=True).status == 1


def test_fic_convout_detection_exhaustive(ora):
    # faults_test.cpp:189-206: every bit of every ConvOut element is detected by FIC
    ls = ora.layer_shape(1, 2, 4, 4, 2, 3, 3, 1, 1, 1, 1)
    x, f = data(ora, ls, 23)
    conv = ora.conv_i8(x, f, ls)
    exp = ora.fic_dot(ora.gen_filter_checksum(f), ora.gen_input_checksum(x, ls))
    assert ora.fic_verify(conv, exp).status == 0
    for i in range(conv.size):
        for b in range(32):
            c2 = conv.copy().ravel()
            c2.view(np.uint32)[i] ^= np.uint32(1 << b)
            assert ora.fic_verify(c2, exp).status == 1


# ------------------------------------------------------------------ golden vectors
@pytest.mark.parametrize("case", GOLDEN["conv"], ids=lambda c: "x".join(map(str, c["dims"])))
def test_oracle_matches_reference_golden(ora, case):
    ls = ora.layer_shape(*case["dims"])
    x, f = data(ora, ls, case["seed"])
    conv = ora.conv_i8(x, f, ls)
    assert sha(conv) == case["conv_sha"]
    bias = np.linspace(-3.0, 3.0, ls.k).astype(np.float32)
    assert sha(ora.epilog(conv, 0.05, np.zeros(ls.k, np.float32))) == case["epilog_relu_sha"]
    assert sha(ora.epilog(conv, 0.0123, bias)) == case["epilog_bias_sha"]
    assert sha(ora.epilog(conv, 0.0123, bias, relu=False)) == case["epilog_ident_sha"]
    assert sha(ora.epilog(conv, 0.0123, bias, relu=False, out_f32=True)) == case["epilog_f32_sha"]
    fc = ora.gen_filter_checksum(f)
    planes = ora.decompose_checksum_filters(fc)
    extra = ora.recombine_extra_fmaps(ora.conv_checksum_planes(x, ls, planes))
    ic = ora.gen_input_checksum(x, ls)
    batch = ora.ic_batch_checksum(x)
    bext = ora.conv_batch_checksum(batch, f, ls)
    assert (sha(fc), sha(planes), sha(extra), sha(ic), sha(batch), sha(bext)) == (
        case["fc_sha"], case["planes_sha"], case["extra_sha"], case["ic_sha"], case["batch_sha"], case["batch_extra_sha"])
    assert ora.fic_dot(fc, ic) == case["fic_dot"]
    got = {"fc": outcome(ora.fc_verify(conv, extra)), "ic": outcome(ora.ic_verify_k(conv, f, ic)),
           "icbatch": outcome(ora.ic_batch_verify(conv, bext)), "fic": outcome(ora.fic_verify(conv, case["fic_dot"]))}
    assert got == case["verify_pass"]
    bad = conv.copy().ravel()
    bad.view(np.uint32)[case["flip"]["key"]] ^= np.uint32(1 << case["flip"]["bit"])
    bad = bad.reshape(conv.shape)
    got = {"fc": outcome(ora.fc_verify(bad, extra)), "ic": outcome(ora.ic_verify_k(bad, f, ic)),
           "icbatch": outcome(ora.ic_batch_verify(bad, bext)), "fic": outcome(ora.fic_verify(bad, case["fic_dot"]))}
    assert got == case["verify_flip"]
    p = ora.plan_precision(ls)
    assert {k: getattr(p, k) for k, _ in p._fields_} == case["plan"]
    if "fused" in case:
        out, cs, nic = ora.fused_conv_epilog(x, f, ls, 0.02, bias, checksum=True,
                                             next_ls=ora.layer_shape(ls.n, ls.k, ls.p, ls.q, 2, 3, 3, 1, 1, 1, 1))
        assert (sha(out), cs, sha(nic)) == (case["fused"]["out_sha"], case["fused"]["checksum"], case["fused"]["next_ic_sha"])


@pytest.mark.parametrize("case", GOLDEN["float"], ids=lambda c: "x".join(map(str, c["dims"])))
def test_oracle_float_mode_matches_reference(ora, case):
    ls = ora.layer_shape(*case["dims"])
    seed = case["seed"]
    if case["integers"]:
        x = ora.random_i8(ls.n * ls.c * ls.h * ls.w, seed).astype(np.float32).reshape(ls.input_dims())
        f = ora.random_i8(ls.k * ls.c * ls.r * ls.s, seed + 1).astype(np.float32).reshape(ls.filter_dims())
    else:
        x = ora.random_f32(ls.n * ls.c * ls.h * ls.w, ora.derive_seed(seed, 1)).reshape(ls.input_dims())
        f = ora.random_f32(ls.k * ls.c * ls.r * ls.s, ora.derive_seed(seed, 2)).reshape(ls.filter_dims())
    assert (sha(x), sha(f)) == (case["x_sha"], case["f_sha"])
    assert sha(ora.conv_f32(x, f, ls)) == case["conv_sha"]
    assert sha(ora.filter_checksum_f64(f)) == case["fs_sha"]
    assert sha(ora.input_checksum_f64(x, ls)) == case["is_sha"]


def test_oracle_trials_match_reference(ora):
    ls = ora.layer_shape(1, 8, 12, 12, 8, 3, 3, 1, 1, 1, 1)
    xr, fr = data(ora, ls, 4242)
    sets = {"ones": (np.ones(ls.input_dims(), np.int8), np.ones(ls.filter_dims(), np.int8)), "random": (xr, fr)}
    for t in GOLDEN["trials"]:
        x, f = sets[t["data"]]
        o = ora.run_trial(ls, x, f, t["scheme"], t["target"], seed=t["seed"])
        got = {"classification": o.classification, "flat_index": o.flat_index, "bit": o.bit,
               "differs": o.final_output_differs, "verify": outcome(o.verify)}
        want = {k: t[k] for k in got}
        assert got == want, t


def test_oracle_small_campaigns_match_reference(ora):
    for c in GOLDEN["campaigns"]:
        if c["trials"] > 200:
            continue
        ls = ora.layer_shape(*c["dims"])
        r = ora.run_campaign(ls, c["scheme"], c["target"], c["trials"], c["root_seed"], mode=c["mode"])
        assert [r.detected, r.detected_benign, r.sdc, r.masked] == c["counts"], c
        # sharded halves fold to the same report (trial order independence)
        a = ora.run_campaign(ls, c["scheme"], c["target"], c["trials"], c["root_seed"], mode=c["mode"], begin=0, end=77)
        b = ora.run_campaign(ls, c["scheme"], c["target"], c["trials"], c["root_seed"], mode=c["mode"], begin=77)
        assert [a.detected + b.detected, a.detected_benign + b.detected_benign, a.sdc + b.sdc, a.masked + b.masked] == c["counts"]


def test_golden_campaign_counts_are_the_published_acceptance_values():
    # BASELINE.md section 1 / SURVEY 8(c): cfg1 layer, 1000 trials, ones, scale 0.05, seeds 0xC2+i
    got = [(c["scheme"], c["target"], tuple(c["counts"])) for c in GOLDEN["campaigns"] if c["trials"] == 1000]
    assert got == [(0, 1, (761, 239, 0, 0)), (0, 2, (932, 68, 0, 0)), (0, 0, (0, 0, 743, 257)),
                   (3, 0, (757, 243, 0, 0)), (3, 1, (766, 234, 0, 0)), (3, 2, (928, 72, 0, 0))]


@pytest.mark.skipif(not ref_available(), reason="oracle/_ref not built")
def test_oracle_vs_reference_random_shapes(ora):
    """Fresh random shapes through both the restatement and the reference build."""
    ref = Oracle("ref")
    g = np.random.default_rng(0xAB)
    for _ in range(40):
        n, c, k = int(g.integers(1, 4)), int(g.integers(1, 20)), int(g.integers(1, 20))
        h, w = int(g.integers(1, 12)), int(g.integers(1, 12))
        r, s = int(g.choice([1, 3, 5])), int(g.choice([1, 3]))
        sh, sw, ph, pw = int(g.integers(1, 3)), int(g.integers(1, 3)), int(g.integers(0, 3)), int(g.integers(0, 2))
        try:
            ls = ref.layer_shape(n, c, h, w, k, r, s, sh, sw, ph, pw)
        except Exception:
            continue
        x, f = data(ref, ls, int(g.integers(1, 1 << 30)))
        assert np.array_equal(ora.conv_i8(x, f, ls), ref.conv_i8(x, f, ls))
        assert np.array_equal(ora.gen_input_checksum(x, ls), ref.gen_input_checksum(x, ls))
        planes = ref.decompose_checksum_filters(ref.gen_filter_checksum(f))
        assert np.array_equal(ora.conv_checksum_planes(x, ls, planes), ref.conv_checksum_planes(x, ls, planes))
        b = ref.ic_batch_checksum(x)
        assert np.array_equal(ora.conv_batch_checksum(b, f, ls), ref.conv_batch_checksum(b, f, ls))
