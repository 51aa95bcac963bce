"""Batch-sharded protected conv on the GPU with two processes.

Two ranks (gloo process group, both on cuda:0 -- the pool offers one GPU per
box) each run the fused FC + FIC conv on their half of the batch, pack their
VerifyOutcomes into records, all-gather them and fold them on the device
(paper_2006_04984_b200/dist.py ShardedVerdicts: abed_verdict_records /
abed_verdict_combine).  The folded outcomes must equal one process running the
whole batch -- fault-free and with a ConvOut flip on rank 1 (global FC locus,
error counts, FIC lhs / rhs sums) -- i.e. the fold is the reference's
fc_verify / fic_verify (checksum.hpp:211-236, 287-294) of the whole batch.
"""
import os
import socket

import pytest
import torch
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu

SHAPE = (8, 32, 14, 14, 48, 3, 3, 1, 1, 1, 1)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _outcome_tuple(o):
    return (o.status, tuple(o.locus) if o.status else (), o.lhs, o.rhs, o.error_count)


def _run(ls, x, f, fault_key):
    from paper_2006_04984_b200 import abi, api
    plan = api.ConvPlan(ls, f, abi.CHECK_FC | abi.CHECK_FIC)
    packed = plan.pack(x)
    out = torch.empty(ls.output_dims(), dtype=torch.int32, device="cuda")
    plan.run(packed, out, abi.OUT_I32_NCHW, ep=None, fault_key=fault_key, fault_bit=17)
    ps = api.PlanSet([plan])
    ps.finalize()
    torch.cuda.synchronize()
    return ps


def _worker(rank, world, port, fault_global, q):
    import torch.distributed as dist

    from paper_2006_04984_b200 import abi, api
    from paper_2006_04984_b200.dist import ShardedVerdicts, shard_range
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    try:
        ls = api.layer_shape(*SHAPE)
        n0, n1 = shard_range(ls.n, rank, world)
        sub = api.layer_shape(n1 - n0, *SHAPE[1:])
        chw, kpq = ls.c * ls.h * ls.w, ls.k * ls.p * ls.q
        # the rank's slice of the global SplitMix64 input stream; filters replicated
        x = api.fill_random_i8((n1 - n0) * chw, api.derive_seed(5, 1), offset=n0 * chw).view(sub.input_dims())
        f = api.fill_random_i8(ls.k * ls.c * ls.r * ls.s, api.derive_seed(5, 2)).view(ls.filter_dims())
        key = -1
        if fault_global >= 0 and n0 * kpq <= fault_global < n1 * kpq:
            key = fault_global - n0 * kpq
        ps = _run(sub, x, f, key)
        sv = ShardedVerdicts(ps._out, [abi.FC, abi.FIC, abi.IC], n_offset=n0)
        sv.record()
        sv.reduce()
        torch.cuda.synchronize()
        g = sv.outcomes_global()
        q.put((rank, [_outcome_tuple(g[0]), _outcome_tuple(g[1])]))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("fault", [-1, 5 * 48 * 14 * 14 + 9 * 14 * 14 + 3 * 14 + 7], ids=["fault-free", "fault-on-rank1"])
def test_batch_sharded_verdicts_equal_single_process(fault):
    from paper_2006_04984_b200 import abi, api
    ls = api.layer_shape(*SHAPE)
    x = api.fill_random_i8(ls.n * ls.c * ls.h * ls.w, api.derive_seed(5, 1)).view(ls.input_dims())
    f = api.fill_random_i8(ls.k * ls.c * ls.r * ls.s, api.derive_seed(5, 2)).view(ls.filter_dims())
    whole = _run(ls, x, f, fault).outcomes()[0]
    want = [_outcome_tuple(whole[0]), _outcome_tuple(whole[1])]
    if fault >= 0:
        assert whole[0].status == 1 and whole[1].status == 1
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, fault, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = [q.get(timeout=300) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, g in got:
        assert g == want, (rank, g, want)
