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
