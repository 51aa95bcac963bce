"""Multi-process (gloo, world_size 2, CPU) tests of the batch/trial sharding and
the single integer all-reduce that the multi-GPU path uses.  The per-shard
campaign runs through the C oracle here (no GPU); on the box the same helpers
drive abed_run_campaign over NCCL."""
import os
import socket

import pytest
import torch.multiprocessing as mp

from paper_2006_04984_b200.dist import shard_range


def test_shard_ranges_cover_exactly():
    for total in (0, 1, 7, 32, 1000, 1024):
        for world in (1, 2, 3, 4, 8):
            spans = [shard_range(total, r, world) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == total
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
            assert max(e - b for b, e in spans) - min(e - b for b, e in spans) <= 1


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import torch.distributed as dist

    from oracle.pyoracle import Oracle
    from paper_2006_04984_b200.dist import allreduce_counts, max_over_ranks, sharded_campaign
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    ora = Oracle("ora")
    ls = ora.layer_shape(1, 8, 12, 12, 8, 3, 3, 1, 1, 1, 1)

    def run_range(b, e):
        r = ora.run_campaign(ls, 3, 0, 96, 4242, mode=1, begin=b, end=e)
        return [r.detected, r.detected_benign, r.sdc, r.masked]

    counts = sharded_campaign(run_range, 96, rank, world)
    verdicts = allreduce_counts([1 if rank == 0 else 0, rank])  # per-shard error counts
    slowest = max_over_ranks(10.0 + rank)
    q.put((rank, counts, verdicts, slowest))
    dist.destroy_process_group()


def test_sharded_campaign_equals_single_process():
    from oracle.pyoracle import Oracle
    ora = Oracle("ora")
    ls = ora.layer_shape(1, 8, 12, 12, 8, 3, 3, 1, 1, 1, 1)
    whole = ora.run_campaign(ls, 3, 0, 96, 4242, mode=1)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=240) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    for rank, counts, verdicts, slowest in res:
        assert counts == [whole.detected, whole.detected_benign, whole.sdc, whole.masked]
        assert verdicts == [1, 1]
        assert slowest == 11.0


@pytest.mark.gpu
def test_bench_multi_rank_contract_single_gpu_visible():
    """bench.py's rank logic with WORLD_SIZE=1 (the driver's N=1 run)."""
    from bench import dist_setup
    assert dist_setup()[0] >= 1


# ---------------------------------------------------------------- batch-sharded verdicts
SHARD_LS = (4, 8, 10, 10, 8, 3, 3, 1, 1, 1, 1)


def _shard_outcomes(ora, x, f, ls, b, e, fault):
    """FC / FIC / ICBatch VerifyOutcomes of images [b, e) (the C oracle restating
    fc_verify, fic_verify and ic_batch_verify), with an optional ConvOut flip
    (global flat index, bit) applied to this shard's output."""
    import numpy as np
    sub = ora.layer_shape(e - b, *SHARD_LS[1:])
    xs = np.ascontiguousarray(x[b:e])
    conv = ora.conv_i8(xs, f, sub)
    if fault is not None:
        idx, bit = fault
        lo, hi = b * ls.k * ls.p * ls.q, e * ls.k * ls.p * ls.q
        if lo <= idx < hi:
            flat = conv.reshape(-1)
            flat[idx - lo] = np.int32(np.uint32(flat[idx - lo].view(np.uint32) ^ np.uint32(1 << bit)).view(np.int32))
    fsum = ora.gen_filter_checksum(f)
    extra = ora.recombine_extra_fmaps(ora.conv_checksum_planes(xs, sub, ora.decompose_checksum_filters(fsum)))
    fc = ora.fc_verify(conv, extra, ls.k)
    fic = ora.fic_verify(conv, ora.fic_dot(fsum, ora.gen_input_checksum(xs, sub)))
    icb = ora.ic_batch_verify(conv, ora.conv_batch_checksum(ora.ic_batch_checksum(xs), f, sub))
    return [fc, fic, icb]


def _verdict_worker(rank, world, port, fault, q):
    import torch.distributed as dist

    from oracle.pyoracle import Oracle
    from paper_2006_04984_b200 import abi
    from paper_2006_04984_b200.dist import combine_host, gather_records, records_host, shard_range
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    ora = Oracle("ora")
    ls = ora.layer_shape(*SHARD_LS)
    x = ora.random_i8(ls.n * ls.c * ls.h * ls.w, 99).reshape(ls.input_dims())
    f = ora.random_i8(ls.k * ls.c * ls.r * ls.s, 98).reshape(ls.filter_dims())
    b, e = shard_range(ls.n, rank, world)
    kinds = [abi.FC, abi.FIC, abi.ICBATCH]
    rec = records_host(_shard_outcomes(ora, x, f, ls, b, e, fault), kinds, b)
    glob = combine_host(gather_records(rec), world, kinds)
    q.put((rank, [(o.status, o.has_locus, tuple(o.locus), o.lhs, o.rhs, o.error_count) for o in glob]))
    dist.destroy_process_group()


@pytest.mark.parametrize("fault", [None, (3 * 8 * 100 + 5 * 100 + 42, 13), (1 * 8 * 100 + 7, 30)],
                         ids=["fault-free", "fault-on-rank1", "fault-on-rank0"])
def test_sharded_verdicts_equal_single_process(fault):
    """Two gloo ranks each verify half the batch; the all-gathered records fold into
    the single-process verdict: FC locus / lhs / rhs (global image index), FIC lhs and
    rhs (sums of the shards), ICBatch status and locus."""
    from oracle.pyoracle import Oracle
    ora = Oracle("ora")
    ls = ora.layer_shape(*SHARD_LS)
    x = ora.random_i8(ls.n * ls.c * ls.h * ls.w, 99).reshape(ls.input_dims())
    f = ora.random_i8(ls.k * ls.c * ls.r * ls.s, 98).reshape(ls.filter_dims())
    whole = _shard_outcomes(ora, x, f, ls, 0, ls.n, fault)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_verdict_worker, args=(r, 2, port, fault, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=240) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    assert res[0][1] == res[1][1]  # every rank holds the same global verdicts
    fc, fic, icb = res[0][1]
    wfc, wfic, wicb = whole
    assert fc[0] == wfc.status and fic[0] == wfic.status and icb[0] == wicb.status
    assert (fic[3], fic[4]) == (wfic.lhs, wfic.rhs)
    if fault is None:
        assert fc[0] == fic[0] == icb[0] == 0
    else:
        assert fc[0] == 1 and fc[2] == tuple(wfc.locus) and (fc[3], fc[4]) == (wfc.lhs, wfc.rhs)
        assert fc[5] == 1 and icb[2] == tuple(wicb.locus)
        n_glob = fault[0] // (ls.k * ls.p * ls.q)
        assert fc[2][0] == n_glob
