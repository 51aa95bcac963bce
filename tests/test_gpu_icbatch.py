"""Fused ICBatch (ABED_CHECK_ICBATCH) against the reference's unfused chain
ic_batch_checksum -> conv_batch_checksum -> ic_batch_verify (checksum.hpp:350-421).

The batch-sum image rides as balanced base-256 digit images after the N real
images of the packed input (written inside the conv kernel), the tensor-core
conv of those rows is the checksum row, and a scan after the kernel compares the
per-(k, p, q) batch sums of the outputs with it.  VerifyOutcome (status, locus
(k, p, q), lhs, rhs) must equal the reference's on fault-free runs and with a
flipped ConvOut element; outputs stay bit-exact.  Integer: no tolerance.
"""
import numpy as np
import pytest
import torch

from oracle.pyoracle import Oracle, ref_available
from paper_2006_04984_b200 import abi, api

pytestmark = pytest.mark.gpu

SHAPES = [
    (1, 64, 56, 56, 64, 3, 3, 1, 1, 1, 1),    # cfg1 (N = 1)
    (8, 64, 28, 28, 64, 3, 3, 1, 1, 1, 1),
    (4, 128, 28, 28, 128, 3, 3, 2, 2, 1, 1),  # stride 2 (4 phases)
    (4, 256, 14, 14, 256, 3, 3, 1, 1, 1, 1),  # two N tiles
    (2, 512, 7, 7, 512, 3, 3, 1, 1, 1, 1),    # streamed filters, 8 N tiles
    (3, 20, 13, 9, 24, 5, 5, 1, 1, 2, 2),     # 5x5, ragged channels
    (5, 48, 15, 17, 32, 1, 1, 2, 2, 0, 0),    # 1x1 stride 2
    (300, 16, 6, 6, 16, 3, 3, 1, 1, 1, 1),    # N > 256: three digit images
]


@pytest.fixture(scope="module")
def ora():
    return Oracle("ref") if ref_available() else Oracle("ora")


def data(dims, seed, extreme=False):
    ls = api.layer_shape(*dims)
    if extreme:
        x = torch.full(ls.input_dims(), -128, dtype=torch.int8)
        f = torch.full(ls.filter_dims(), -128, dtype=torch.int8)
        return ls, x, f
    g = torch.Generator().manual_seed(seed)
    x = torch.randint(-128, 128, ls.input_dims(), dtype=torch.int8, generator=g)
    f = torch.randint(-128, 128, ls.filter_dims(), dtype=torch.int8, generator=g)
    return ls, x, f


def run(ls, x, f, checks, fault_key=-1, fault_bit=0, runs=2):
    plan = api.ConvPlan(ls, f.cuda(), checks)
    packed = plan.pack(x.cuda())
    out = torch.empty(ls.output_dims(), dtype=torch.int32, device="cuda")
    for _ in range(runs):  # later runs start from the scan's reset accumulators
        plan.run(packed, out, abi.OUT_I32_NCHW, ep=None, fault_key=fault_key, fault_bit=fault_bit)
        plan.finalize()
    torch.cuda.synchronize()
    return out.cpu().numpy(), plan.outcomes()


def reference_outcome(ora, convout, x, f, ls):
    extra = ora.conv_batch_checksum(ora.ic_batch_checksum(x), f, ls)
    return ora.ic_batch_verify(convout, extra)


@pytest.mark.parametrize("checks", [abi.CHECK_ICBATCH, abi.CHECK_FC | abi.CHECK_FIC | abi.CHECK_ICBATCH],
                         ids=["icbatch", "fc+fic+icbatch"])
@pytest.mark.parametrize("dims", SHAPES, ids=["x".join(map(str, d[:5])) for d in SHAPES])
def test_icbatch_fault_free(ora, dims, checks):
    ls, x, f = data(dims, 11 + sum(dims))
    xh, fh = x.numpy(), f.numpy()
    want = ora.conv_i8(xh, fh, ls)
    got, oc = run(ls, x, f, checks)
    assert np.array_equal(got, want)
    ref = reference_outcome(ora, want, xh, fh, ls)
    assert ref.status == 0
    icb = oc[2]
    assert icb.status == 0 and icb.has_locus == 0 and icb.lhs == 0 and icb.rhs == 0 and icb.error_count == 0
    if checks & abi.CHECK_FIC:
        assert oc[1].status == 0 and oc[1].lhs == oc[1].rhs == int(want.astype(np.int64).sum())
    if checks & abi.CHECK_FC:
        assert oc[0].status == 0


@pytest.mark.parametrize("dims", SHAPES[:5] + SHAPES[7:], ids=lambda d: "x".join(map(str, d[:5])))
def test_icbatch_extreme_values(ora, dims):
    # all -128: the largest batch sums (digit range) and products
    ls, x, f = data(dims, 0, extreme=True)
    want = ora.conv_i8(x.numpy(), f.numpy(), ls)
    got, oc = run(ls, x, f, abi.CHECK_ICBATCH, runs=1)
    assert np.array_equal(got, want)
    assert oc[2].status == 0


@pytest.mark.parametrize("frac,bit", [(0.0, 0), (0.37, 9), (0.71, 31), (0.999, 30)])
@pytest.mark.parametrize("dims", [SHAPES[1], SHAPES[3], SHAPES[4], SHAPES[7]],
                         ids=lambda d: "x".join(map(str, d[:5])))
def test_icbatch_convout_fault(ora, dims, frac, bit):
    ls, x, f = data(dims, 5 + sum(dims))
    xh, fh = x.numpy(), f.numpy()
    want = ora.conv_i8(xh, fh, ls)
    key = min(int(frac * want.size), want.size - 1)
    got, oc = run(ls, x, f, abi.CHECK_ICBATCH, fault_key=key, fault_bit=bit)
    flipped = want.copy().reshape(-1)
    flipped[key] = np.int32(np.uint32(flipped[key].view(np.uint32) ^ np.uint32(1 << bit)).view(np.int32))
    flipped = flipped.reshape(want.shape)
    assert np.array_equal(got, flipped)  # the hook flips the stored ConvOut too
    ref = reference_outcome(ora, flipped, xh, fh, ls)
    icb = oc[2]
    assert ref.status == 1 and icb.status == 1
    assert tuple(icb.locus) == tuple(ref.locus) and icb.lhs == ref.lhs and icb.rhs == ref.rhs
    kpq = key % (ls.k * ls.p * ls.q)
    assert tuple(icb.locus) == (kpq // (ls.p * ls.q), (kpq % (ls.p * ls.q)) // ls.q, kpq % ls.q)
    assert icb.error_count == 1


def test_icbatch_argument_errors():
    ls, x, f = data((2, 16, 8, 8, 16, 3, 3, 1, 1, 1, 1), 1)
    with pytest.raises(abi.InvalidArgument):
        api.ConvPlan(ls, f.cuda(), abi.CHECK_IC | abi.CHECK_ICBATCH)
    with pytest.raises(abi.InvalidArgument):
        api.ConvPlan(ls, f.cuda(), 16)
    ff = torch.randn(ls.filter_dims(), device="cuda")
    with pytest.raises(abi.InvalidArgument):
        api.ConvPlanH(ls, ff, abi.F16, abi.CHECK_ICBATCH)
    # the packed buffer holds the two digit images after the batch
    plain = api.ConvPlan(ls, f.cuda(), 0)
    icb = api.ConvPlan(ls, f.cuda(), abi.CHECK_ICBATCH)
    assert icb.info.packed_input_bytes > plain.info.packed_input_bytes


def test_device_verdict_fold_equals_host_fold():
    """abed_verdict_records / abed_verdict_combine on the device (the bench's
    multi-GPU path) against the host fold, on a synthetic 3-rank gather."""
    import ctypes as C
    from paper_2006_04984_b200.dist import OUTCOME_BYTES, ShardedVerdicts, combine_host, records_host
    kinds = [abi.FC, abi.FIC, abi.ICBATCH, abi.FC, abi.FIC, abi.IC]
    ranks = []
    for r in range(3):
        outs = []
        for i, k in enumerate(kinds):
            o = abi.VerifyOutcome()
            fail = (r + i) % 3 == 0
            o.status, o.has_locus = int(fail and k != abi.FIC), int(fail and k != abi.FIC)
            o.locus[0], o.locus[1], o.locus[2] = r + i, 2 * i, 3
            o.lhs, o.rhs = 1000 * r + i, 1000 * r + (i if not fail else i + 7)
            o.error_count = 2 if o.status else 0
            outs.append(o)
        ranks.append(outs)
    gathered = [v for r, outs in enumerate(ranks) for v in records_host(outs, kinds, n_offset=4 * r)]
    want = combine_host(gathered, 3, kinds)
    dev = torch.zeros(len(kinds) * OUTCOME_BYTES, dtype=torch.uint8, device="cuda")
    host = (abi.VerifyOutcome * len(kinds))(*ranks[0])
    dev.copy_(torch.frombuffer(bytearray(host), dtype=torch.uint8))
    sv = ShardedVerdicts(dev, kinds, n_offset=0, force=True)
    sv.record()
    torch.cuda.synchronize()
    assert sv.rec.cpu().tolist() == gathered[: len(kinds) * 8]
    sv.gathered = torch.tensor(gathered, dtype=torch.int64, device="cuda")
    sv.world = 3
    sv._fold(C.c_void_p(torch.cuda.current_stream().cuda_stream))
    got = sv.outcomes_global()
    for a, b in zip(got, want):
        assert (a.status, a.has_locus, tuple(a.locus), a.lhs, a.rhs, a.error_count) == \
               (b.status, b.has_locus, tuple(b.locus), b.lhs, b.rhs, b.error_count)
