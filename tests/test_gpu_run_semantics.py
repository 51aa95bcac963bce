"""Run / finalize semantics that replace per-run memsets, and the one-shot plan
cache behind the reference's conv_fast_i8 / conv_direct / fused_conv_epilog.

* IC plans: a run's in-kernel sums are consumed (and zeroed) by its verdict; a
  second finalize of the same run repeats the outcome; a run that was never
  finalized is cleared before the next run accumulates; captured-graph replays of
  run + finalize stay correct (ic_verify_k, checksum.hpp:319-347).
* Compare runs (full duplication): the mismatch counter only grows and
  abed_conv_plan_compare_count reports the increase since the previous call.
* One-shot calls: the cached plan re-packs the filters on every call (same shape,
  different filters), and more shapes than the cache holds evict cleanly.
Integer results: exact against the C oracle.
"""
import ctypes

import numpy as np
import pytest
import torch

from oracle.pyoracle import Oracle
from paper_2006_04984_b200 import abi, api

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ora():
    return Oracle("ora")


def _data(ls, seed):
    g = torch.Generator().manual_seed(seed)
    x = torch.randint(-128, 128, ls.input_dims(), dtype=torch.int8, generator=g)
    f = torch.randint(-128, 128, ls.filter_dims(), dtype=torch.int8, generator=g)
    return x, f


def _ic_ref(ora, x, f, ls, fault_key=-1, fault_bit=0):
    conv = ora.conv_i8(x.numpy(), f.numpy(), ls)
    if fault_key >= 0:
        flat = conv.reshape(-1).view(np.uint32)
        flat[fault_key] ^= np.uint32(1 << fault_bit)
    ic = ora.gen_input_checksum(x.numpy(), ls)
    return ora.ic_verify_k(conv, f.numpy(), ic)


def _same(a, b):
    return (a.status, tuple(a.locus), a.lhs, a.rhs) == (b.status, tuple(b.locus), b.lhs, b.rhs)


def test_ic_consumed_sums_repeat_finalize_and_unfinalized_runs(ora):
    ls = api.layer_shape(4, 32, 14, 14, 48, 3, 3, 1, 1, 1, 1)
    x, f = _data(ls, 11)
    plan = api.ConvPlan(ls, f.cuda(), abi.CHECK_IC)
    packed = plan.pack(x.cuda())
    out = torch.empty(ls.output_dims(), dtype=torch.int32, device="cuda")
    key = 2 * ls.k * ls.p * ls.q + 7 * ls.p * ls.q + 3 * ls.q + 5
    good, bad = _ic_ref(ora, x, f, ls), _ic_ref(ora, x, f, ls, key, 20)
    assert good.status == 0 and bad.status == 1
    # fault, finalize twice (the second repeats the first)
    plan.run(packed, out, abi.OUT_I32_NCHW, ep=None, fault_key=key, fault_bit=20)
    plan.finalize()
    assert _same(plan.outcomes()[2], bad)
    plan.finalize()
    assert _same(plan.outcomes()[2], bad)
    # clean run after the consumed fault: passes (no stale sums)
    plan.run(packed, out, abi.OUT_I32_NCHW, ep=None)
    plan.finalize()
    assert _same(plan.outcomes()[2], good)
    # two runs without a finalize in between: the second starts from cleared sums
    plan.run(packed, out, abi.OUT_I32_NCHW, ep=None, fault_key=key, fault_bit=20)
    plan.run(packed, out, abi.OUT_I32_NCHW, ep=None)
    plan.finalize()
    assert _same(plan.outcomes()[2], good)


def test_ic_graph_replays_of_run_and_finalize(ora):
    ls = api.layer_shape(2, 16, 12, 12, 32, 3, 3, 1, 1, 1, 1)
    x, f = _data(ls, 12)
    plan = api.ConvPlan(ls, f.cuda(), abi.CHECK_IC)
    packed = plan.pack(x.cuda())
    out = torch.empty(ls.output_dims(), dtype=torch.int32, device="cuda")
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        plan.run(packed, out, abi.OUT_I32_NCHW, ep=None)
        plan.finalize()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        plan.run(packed, out, abi.OUT_I32_NCHW, ep=None)
        plan.finalize()
    good = _ic_ref(ora, x, f, ls)
    for _ in range(5):
        g.replay()
        torch.cuda.synchronize()
        assert _same(plan.outcomes()[2], good)


def test_ic_captured_runs_without_finalize_clear_their_sums(ora):
    """A graph that contains only the run, replayed several times, then one eager
    finalize: the verdict is the last run's (captured runs clear the sums unless the
    plan declared paired finalizes)."""
    ls = api.layer_shape(2, 16, 12, 12, 32, 3, 3, 1, 1, 1, 1)
    x, f = _data(ls, 14)
    plan = api.ConvPlan(ls, f.cuda(), abi.CHECK_IC)
    packed = plan.pack(x.cuda())
    out = torch.empty(ls.output_dims(), dtype=torch.int32, device="cuda")
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        plan.run(packed, out, abi.OUT_I32_NCHW, ep=None)
        plan.finalize()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        plan.run(packed, out, abi.OUT_I32_NCHW, ep=None)
    for _ in range(3):
        g.replay()
    plan.finalize()
    torch.cuda.synchronize()
    assert _same(plan.outcomes()[2], _ic_ref(ora, x, f, ls))


def test_compare_count_reports_the_increase():
    ls = api.layer_shape(2, 16, 10, 10, 16, 3, 3, 1, 1, 1, 1)
    x, f = _data(ls, 13)
    plan = api.ConvPlan(ls, f.cuda(), 0)
    packed = plan.pack(x.cuda())
    buf = torch.zeros(ls.n * 16 * (ls.p + 1) * (ls.q + 1) + (1 << 16), dtype=torch.int8, device="cuda")
    ep = plan.epilog_params(0.05, [0.0] * ls.k, True)
    plan.run(packed, buf, abi.OUT_I8_PACKED, ep=ep)
    n = ctypes.c_int64(-1)
    for _ in range(3):  # identical recomputations: no mismatches, every time
        plan.run(packed, buf, abi.OUT_I8_COMPARE, ep=ep)
        abi.call("abed_conv_plan_compare_count", plan.handle, ctypes.byref(n))
        assert n.value == 0
    buf.view(torch.uint8)[:4096].bitwise_xor_(1)  # corrupt stored outputs: the next compare counts them
    plan.run(packed, buf, abi.OUT_I8_COMPARE, ep=ep)
    abi.call("abed_conv_plan_compare_count", plan.handle, ctypes.byref(n))
    assert n.value > 0
    plan.run(packed, buf, abi.OUT_I8_PACKED, ep=ep)  # restore
    plan.run(packed, buf, abi.OUT_I8_COMPARE, ep=ep)
    abi.call("abed_conv_plan_compare_count", plan.handle, ctypes.byref(n))
    assert n.value == 0


def test_one_shot_cache_repacks_filters_and_evicts(ora):
    ls = api.layer_shape(2, 16, 9, 11, 24, 3, 3, 1, 1, 1, 1)
    for seed in (21, 22, 23):  # same shape, different filters each call
        x, f = _data(ls, seed)
        got = api.conv_direct(x.cuda(), f.cuda(), ls).cpu().numpy()
        assert np.array_equal(got, ora.conv_i8(x.numpy(), f.numpy(), ls))
    # more shapes than the cache holds (8 per device), then the first again
    shapes = [api.layer_shape(1, 8 + 8 * i, 6, 7, 16, 3, 3, 1, 1, 1, 1) for i in range(11)] + [ls]
    for i, s in enumerate(shapes):
        x, f = _data(s, 40 + i)
        got = api.conv_direct(x.cuda(), f.cuda(), s).cpu().numpy()
        assert np.array_equal(got, ora.conv_i8(x.numpy(), f.numpy(), s)), i


def test_fused_conv_epilog_tap_on_the_cached_fic_plan(ora):
    ls = api.layer_shape(2, 16, 8, 8, 16, 3, 3, 1, 1, 1, 1)
    bias = np.linspace(-1, 1, ls.k).astype(np.float32)
    for seed in (31, 32):
        x, f = _data(ls, seed)
        y, cs, _ = api.fused_conv_epilog(x.cuda(), f.cuda(), ls, 0.03, bias.tolist(), output_checksum=True)
        conv = ora.conv_i8(x.numpy(), f.numpy(), ls)
        assert cs == int(conv.astype(np.int64).sum())
        assert np.array_equal(y.cpu().numpy(), ora.epilog(conv, 0.03, bias))


def _icb_ref(ora, x, f, ls, fault_key=-1, fault_bit=0):
    conv = ora.conv_i8(x.numpy(), f.numpy(), ls)
    if fault_key >= 0:
        flat = conv.reshape(-1).view(np.uint32)
        flat[fault_key] ^= np.uint32(1 << fault_bit)
    extra = ora.conv_batch_checksum(ora.ic_batch_checksum(x.numpy()), f.numpy(), ls)
    return ora.ic_batch_verify(conv, extra)


def test_icbatch_scan_at_finalize_consumes_and_repeats(ora):
    """ICBatch: the scan of a run happens at the finalize that follows it (one launch
    for every plan of a pass); a second finalize repeats the outcome; a run that was
    never finalized is cleared before the next run accumulates (ic_batch_verify,
    checksum.hpp:398-421)."""
    ls = api.layer_shape(4, 32, 14, 14, 48, 3, 3, 1, 1, 1, 1)
    x, f = _data(ls, 15)
    plan = api.ConvPlan(ls, f.cuda(), abi.CHECK_ICBATCH)
    packed = plan.pack(x.cuda())
    out = torch.empty(ls.output_dims(), dtype=torch.int32, device="cuda")
    key = 1 * ls.k * ls.p * ls.q + 9 * ls.p * ls.q + 4 * ls.q + 2
    good, bad = _icb_ref(ora, x, f, ls), _icb_ref(ora, x, f, ls, key, 21)
    assert good.status == 0 and bad.status == 1
    plan.run(packed, out, abi.OUT_I32_NCHW, ep=None, fault_key=key, fault_bit=21)
    plan.finalize()
    assert _same(plan.outcomes()[2], bad)
    plan.finalize()
    assert _same(plan.outcomes()[2], bad)
    plan.run(packed, out, abi.OUT_I32_NCHW, ep=None)
    plan.finalize()
    assert _same(plan.outcomes()[2], good)
    plan.run(packed, out, abi.OUT_I32_NCHW, ep=None, fault_key=key, fault_bit=21)
    plan.run(packed, out, abi.OUT_I32_NCHW, ep=None)
    plan.finalize()
    assert _same(plan.outcomes()[2], good)


@pytest.mark.parametrize("paired", [False, True], ids=["run-only-graph", "paired-graph"])
def test_icbatch_graph_replays(ora, paired):
    """Captured ICBatch passes: run + finalize graphs (paired: no clearing memsets),
    and run-only graphs replayed several times before one eager finalize."""
    ls = api.layer_shape(3, 16, 12, 12, 32, 3, 3, 1, 1, 1, 1)
    x, f = _data(ls, 16)
    plans = [api.ConvPlan(ls, f.cuda(), abi.CHECK_ICBATCH) for _ in range(3)]
    ps = api.PlanSet(plans)
    for pl in plans:
        pl.set_paired_finalize(paired)
    packed = plans[0].pack(x.cuda())
    outs = [torch.empty(ls.output_dims(), dtype=torch.int32, device="cuda") for _ in plans]
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        for pl, o in zip(plans, outs):
            pl.run(packed, o, abi.OUT_I32_NCHW, ep=None)
        ps.finalize()
    torch.cuda.synchronize()
    good = _icb_ref(ora, x, f, ls)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        for pl, o in zip(plans, outs):
            pl.run(packed, o, abi.OUT_I32_NCHW, ep=None)
        if paired:
            ps.finalize()
    for _ in range(4):
        g.replay()
    if not paired:
        ps.finalize()
    torch.cuda.synchronize()
    for oc in ps.outcomes():
        assert _same(oc[2], good)
