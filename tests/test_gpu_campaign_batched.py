"""Trial-parallel fault campaign (abed_run_campaign_batched / abed_campaign_*)
against the reference's run_campaign (faults.hpp:276-333).

Every trial of a campaign is evaluated in one launch from the golden ConvOut and
the elements its flip perturbs.  Parity: the 24 reference-generated golden
campaigns (including the six acceptance counts on the cfg1 layer), the reference
build itself (oracle/_ref) on strided / padded / ragged / 5x5 layers, and the
exhaustive GPU path (one fused protected conv per trial) on the epilog options
the oracle harness does not expose.  Integer classification counts: exact.
"""
import json
import os

import pytest
import torch

from oracle.pyoracle import Oracle, ref_available
from paper_2006_04984_b200 import abi, api

pytestmark = pytest.mark.gpu

GOLDEN = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "golden.json")))
SCHEMES = [abi.FC, abi.IC, abi.FIC]
TARGETS = [abi.TARGET_INPUT, abi.TARGET_FILTER, abi.TARGET_CONVOUT]


def counts(r):
    return [r.detected, r.detected_benign, r.sdc, r.masked]


@pytest.mark.parametrize("c", GOLDEN["campaigns"],
                         ids=lambda c: f"s{c['scheme']}-t{c['target']}-{c['trials']}-m{c['mode']}")
def test_batched_campaign_matches_reference_golden(c):
    ls = api.layer_shape(*c["dims"])
    r = api.run_campaign(ls, c["scheme"], c["target"], c["trials"], c["root_seed"], mode=c["mode"], batched=True)
    assert counts(r) == c["counts"] and r.trials == c["trials"]


SHAPES = [
    (2, 5, 9, 11, 7, 3, 3, 2, 2, 1, 1),    # stride 2, ragged channels
    (1, 20, 13, 9, 24, 5, 5, 1, 1, 2, 2),  # 5x5
    (3, 16, 8, 8, 16, 3, 3, 1, 1, 0, 0),   # no padding
    (2, 48, 7, 7, 32, 1, 1, 2, 2, 0, 0),   # 1x1 stride 2
]


@pytest.mark.skipif(not ref_available(), reason="oracle/_ref (the reference build) not present")
@pytest.mark.parametrize("dims", SHAPES, ids=lambda d: "x".join(map(str, d)))
@pytest.mark.parametrize("scheme", SCHEMES, ids=["FC", "IC", "FIC"])
@pytest.mark.parametrize("target", TARGETS, ids=["input", "filter", "convout"])
def test_batched_campaign_matches_reference_build(dims, scheme, target):
    ls = api.layer_shape(*dims)
    ref = Oracle("ref").run_campaign(ls, scheme, target, 300, 77 + scheme * 3 + target, mode=abi.DATA_RANDOM_I8)
    got = api.run_campaign(ls, scheme, target, 300, 77 + scheme * 3 + target, mode=abi.DATA_RANDOM_I8, batched=True)
    assert counts(got) == counts(ref)


@pytest.mark.parametrize("opts", [dict(relu=False), dict(output_kind=abi.F32), dict(bias=[0.5, -1.5, 2.0, 0.0, 1.0,
                                                                                          -0.25, 3.0, -2.0])],
                         ids=["identity", "f32-out", "bias"])
@pytest.mark.parametrize("scheme", SCHEMES, ids=["FC", "IC", "FIC"])
@pytest.mark.parametrize("target", TARGETS, ids=["input", "filter", "convout"])
def test_batched_equals_exhaustive_on_epilog_options(opts, scheme, target):
    ls = api.layer_shape(2, 8, 10, 10, 8, 3, 3, 1, 1, 1, 1)
    kw = dict(mode=abi.DATA_RANDOM_I8, scale=0.02, **opts)
    a = api.run_campaign(ls, scheme, target, 150, 9001, **kw)
    b = api.run_campaign(ls, scheme, target, 150, 9001, batched=True, **kw)
    assert counts(a) == counts(b)


def test_device_campaign_shards_sum_to_whole():
    """Trial ranges on separate 'ranks' add up to the whole campaign (the
    quantity the multi-GPU bench all-reduces)."""
    ls = api.layer_shape(4, 64, 28, 28, 64, 3, 3, 1, 1, 1, 1)
    camp = api.Campaign(ls, abi.FIC, abi.TARGET_INPUT, 1000, 5, mode=abi.DATA_RANDOM_I8)
    whole = torch.zeros(4, dtype=torch.int64, device="cuda")
    camp.run(whole)
    parts = torch.zeros(4, dtype=torch.int64, device="cuda")
    for b, e in [(0, 250), (250, 500), (500, 750), (750, 1000)]:
        camp.run(parts, b, e)
    assert torch.equal(whole, parts) and int(whole.sum()) == 1000
    rep = camp.report(whole, 1000)
    ref = api.run_campaign(ls, abi.FIC, abi.TARGET_INPUT, 1000, 5, mode=abi.DATA_RANDOM_I8, batched=True)
    assert counts(rep) == counts(ref)


def test_batched_guards_mirror_reference():
    ls = api.layer_shape(1, 4, 6, 6, 4, 3, 3, 1, 1, 1, 1)
    with pytest.raises(abi.InvalidArgument):
        api.run_campaign(ls, abi.FIC, abi.TARGET_CONVOUT, 0, 1, batched=True)
    with pytest.raises(abi.InvalidArgument):
        api.run_campaign(ls, abi.ICBATCH, abi.TARGET_CONVOUT, 10, 1, batched=True)


@pytest.mark.parametrize("scheme", SCHEMES, ids=["FC", "IC", "FIC"])
@pytest.mark.parametrize("target", TARGETS, ids=["input", "filter", "convout"])
def test_batch_sharded_records_sum_to_single_gpu_report(scheme, target):
    """configs[4]'s multi-GPU campaign: each rank holds a batch shard of the layer;
    per-trial records summed over the shards (the NCCL all-reduce) and classified
    equal the whole-batch report -- here with 3 uneven shards in one process."""
    ls = api.layer_shape(6, 16, 12, 12, 24, 3, 3, 1, 1, 1, 1)
    trials, seed = 400, 31 + 3 * scheme + target
    whole = api.run_campaign(ls, scheme, target, trials, seed, mode=abi.DATA_RANDOM_I8, batched=True)
    total = torch.zeros(trials, 3, dtype=torch.int64, device="cuda")
    for b, e in [(0, 1), (1, 4), (4, 6)]:
        camp = api.Campaign(ls, scheme, target, trials, seed, mode=abi.DATA_RANDOM_I8, images=(b, e))
        rec = torch.zeros(trials, 3, dtype=torch.int64, device="cuda")
        camp.run_records(rec)
        total += rec
    cnt = torch.zeros(4, dtype=torch.int64, device="cuda")
    camp.classify(total, cnt)
    c = cnt.tolist()  # indexed by ABED_DETECTED, _SDC, _MASKED, _DETECTED_BENIGN
    assert [c[abi.DETECTED], c[abi.DETECTED_BENIGN], c[abi.SDC], c[abi.MASKED]] == counts(whole)
