"""Multi-GPU verdicts and sharding for the batch-sharded protected convolution
(SURVEY 8(e)).

Images are independent, so the batch shards across ranks (contiguous image
ranges: rank order is batch order) and every rank verifies its shard.  The only
data-path collective is ONE all-gather per step of the per-shard VerifyOutcome
records (8 int64 per outcome slot), folded on the device into the global
outcomes by abed_verdict_combine:

* FC (fc_verify, checksum.hpp:211-236): error counts add, the global first
  mismatch is the lowest failing rank's (its locus n made global by the rank's
  image offset);
* FIC (fic_verify, :287-294): lhs = sum of the outputs and rhs = fic_dot are both
  linear in the batch, so the per-shard sums add up to the single-GPU verdict;
* IC / ICBatch: per-shard restrictions of the check (any shard failing fails).

Campaign trials shard by trial index; trial seeds derive_seed(root, t) do not
depend on the GPU count, so the folded report is identical for any world size.
The same fold runs on host memory (abed_verdict_*_host) for the gloo CPU tests.
"""
from __future__ import annotations

import ctypes as C

import torch

from . import abi

REC_WORDS = 8
OUTCOME_BYTES = C.sizeof(abi.VerifyOutcome)


def shard_range(total: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous [begin, end) share of `total` items for `rank` (balanced to +-1)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    return total * rank // world, total * (rank + 1) // world


def _dist():
    import torch.distributed as dist
    return dist if dist.is_available() and dist.is_initialized() else None


def _kinds(kinds):
    arr = (C.c_int32 * len(kinds))(*kinds)
    return arr, C.cast(arr, C.c_void_p)


class ShardedVerdicts:
    """Global VerifyOutcomes of a batch-sharded pass.

    outcomes_dev: uint8 CUDA tensor holding n abed_verify_outcome of this rank
    (e.g. a PlanSet's outcome buffer, 3 slots per layer {FC, FIC, IC/ICBatch});
    kinds: scheme of each slot (abi.FC / abi.FIC / abi.IC / abi.ICBATCH);
    n_offset: index of this rank's first image in the global batch.
    record() (capturable) packs the records; reduce() runs the all-gather and the
    device fold into self.global_dev.  With one rank there is nothing to gather or
    fold (the global outcomes are the rank's own): record() and reduce() launch
    nothing unless force=True (tests of the device fold on one GPU)."""

    def __init__(self, outcomes_dev: torch.Tensor, kinds, n_offset: int, group=None, force: bool = False):
        self.n = len(kinds)
        assert outcomes_dev.numel() >= self.n * OUTCOME_BYTES
        self.outcomes = outcomes_dev
        self._karr, self._kptr = _kinds(kinds)
        self.n_offset = int(n_offset)
        self.group = group
        d = _dist()
        self.world = d.get_world_size(group) if d else 1
        self.active = self.world > 1 or force
        dev = outcomes_dev.device
        self.gathered = torch.zeros(self.world * self.n * REC_WORDS, dtype=torch.int64, device=dev)
        # one rank: the records are the gathered buffer
        self.rec = self.gathered if self.world == 1 else torch.zeros(self.n * REC_WORDS, dtype=torch.int64,
                                                                      device=dev)
        self.global_dev = torch.zeros(self.n * OUTCOME_BYTES, dtype=torch.uint8, device=dev)

    def record(self, stream=None):
        if not self.active:
            return
        st = C.c_void_p(stream if stream is not None else torch.cuda.current_stream().cuda_stream)
        abi.call("abed_verdict_records", C.c_void_p(self.outcomes.data_ptr()), self.n, self._kptr, self.n_offset,
                 C.c_void_p(self.rec.data_ptr()), st)
        if self.world == 1:
            self._fold(st)

    def _fold(self, st):
        abi.call("abed_verdict_combine", C.c_void_p(self.gathered.data_ptr()), self.world, self.n, self._kptr,
                 C.c_void_p(self.global_dev.data_ptr()), st)

    def reduce(self, stream=None):
        if self.world == 1:
            return
        d = _dist()
        d.all_gather_into_tensor(self.gathered, self.rec, group=self.group)
        self._fold(C.c_void_p(stream if stream is not None else torch.cuda.current_stream().cuda_stream))

    def outcomes_global(self):
        host = (self.global_dev if self.active else self.outcomes[: self.n * OUTCOME_BYTES]).cpu().numpy()
        res = (abi.VerifyOutcome * self.n)()
        C.memmove(res, host.ctypes.data, C.sizeof(res))
        return list(res)


def records_host(outcomes, kinds, n_offset: int) -> list[int]:
    """abed_verdict_records_host: this rank's records for a list of VerifyOutcome."""
    n = len(kinds)
    arr = (abi.VerifyOutcome * n)(*outcomes)
    rec = (C.c_int64 * (n * REC_WORDS))()
    karr, kp = _kinds(kinds)
    abi.call("abed_verdict_records_host", C.cast(arr, C.c_void_p), n, kp, n_offset, C.cast(rec, C.c_void_p))
    del karr
    return list(rec)


def combine_host(gathered: list[int], world: int, kinds) -> list:
    """abed_verdict_combine_host: fold world x n records (rank-major) into n outcomes."""
    n = len(kinds)
    g = (C.c_int64 * len(gathered))(*gathered)
    out = (abi.VerifyOutcome * n)()
    karr, kp = _kinds(kinds)
    abi.call("abed_verdict_combine_host", C.cast(g, C.c_void_p), world, n, kp, C.cast(out, C.c_void_p))
    del karr
    return list(out)


def gather_records(rec: list[int], group=None) -> list[int]:
    """All-gather this rank's int64 records (rank-major) over the process group."""
    d = _dist()
    t = torch.tensor(rec, dtype=torch.int64)
    if not d or d.get_world_size(group) == 1:
        return list(rec)
    parts = [torch.empty_like(t) for _ in range(d.get_world_size(group))]
    d.all_gather(parts, t, group=group)
    return [int(v) for p in parts for v in p.tolist()]


def allreduce_counts(counts, device=None) -> list[int]:
    """Sum small integer vectors (campaign class counts) over all ranks."""
    t = torch.as_tensor(list(counts), dtype=torch.int64, device=device)
    d = _dist()
    if d and d.get_world_size() > 1:
        d.all_reduce(t)
    return [int(v) for v in t.tolist()]


def max_over_ranks(value: float, device=None) -> float:
    """Multi-GPU timing rule: the step time is the slowest rank's."""
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    d = _dist()
    if d and d.get_world_size() > 1:
        d.all_reduce(t, op=d.ReduceOp.MAX)
    return float(t.item())


def sharded_campaign(run_range, trials: int, rank: int, world: int, device=None) -> list[int]:
    """run_range(begin, end) -> (detected, benign, sdc, masked) for this rank's trial
    shard; returns the global report counts."""
    b, e = shard_range(trials, rank, world)
    return allreduce_counts(run_range(b, e), device=device)
