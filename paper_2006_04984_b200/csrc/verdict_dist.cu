// Multi-GPU verdicts: the batch is sharded across ranks, every
// rank verifies its shard, and the per-shard VerifyOutcomes (checksum.hpp:30-51)
// are folded into the global ones with ONE small collective per step: each rank
// writes kRecWords int64 per outcome slot, the records of all ranks are
// all-gathered (NCCL over NVLink; gloo in the CPU tests), and a one-block
// kernel folds them.  The fold is the reference's verdict over the whole batch
// where linearity makes that exact, the reference's ordered fold otherwise:
//   FC  (fc_verify, :211-236): mismatch counts add; the first mismatch in the
//       reference's (n, p, q) order is the lowest rank's (shards are contiguous
//       image ranges, so rank order is batch order; locus n is made global by the
//       rank's image offset when the records are written)
//   FIC (fic_verify, :287-294): lhs and rhs add (the output sum and fic_dot are
//       both linear in the batch); status = lhs != rhs, pass reports lhs = rhs
//   IC / ICBatch (:319-347, :398-421): per-shard verdicts (each is the exact
//       restriction of the check to the shard): status = any shard failed, counts
//       add, locus / lhs / rhs of the lowest failing rank
// The same fold runs on host memory (abed_verdict_*_host) for the CPU tests.
#include <cuda_runtime.h>

#include "abed_internal.h"

namespace {

constexpr int kRecWords = 8;  // {status, has_locus, l0, l1, l2, lhs, rhs, error_count}
constexpr int kMaxSlots = 256;

struct Kinds {
  int n;
  int8_t kind[kMaxSlots];
};

__host__ __device__ inline void put_record(const abed_verify_outcome& o, int kind, int64_t n_offset, int64_t* r) {
  r[0] = o.status;
  r[1] = o.has_locus;
  r[2] = o.locus[0] + ((kind == ABED_FC && o.has_locus) ? n_offset : 0);
  r[3] = o.locus[1];
  r[4] = o.locus[2];
  r[5] = o.lhs;
  r[6] = o.rhs;
  r[7] = o.error_count;
}

__host__ __device__ inline void fold_slot(const int64_t* gathered, int world, int n, int slot, int kind,
                                          abed_verify_outcome* out) {
  abed_verify_outcome o{};
  if (kind == ABED_FIC) {
    int64_t lhs = 0, rhs = 0;
    for (int w = 0; w < world; ++w) {
      const int64_t* r = gathered + ((int64_t)w * n + slot) * kRecWords;
      lhs += r[5];
      rhs += r[6];
    }
    o.status = lhs != rhs ? 1 : 0;
    o.lhs = lhs;
    o.rhs = rhs;
    o.error_count = o.status;
  } else {
    int first = -1;
    int64_t count = 0;
    for (int w = 0; w < world; ++w) {
      const int64_t* r = gathered + ((int64_t)w * n + slot) * kRecWords;
      if (r[0]) {
        if (first < 0) first = w;
        count += r[7] > 0 ? r[7] : 1;
      }
    }
    if (first >= 0) {
      const int64_t* r = gathered + ((int64_t)first * n + slot) * kRecWords;
      o.status = 1;
      o.has_locus = (int32_t)r[1];
      o.locus[0] = r[2];
      o.locus[1] = r[3];
      o.locus[2] = r[4];
      o.lhs = r[5];
      o.rhs = r[6];
      o.error_count = count;
    }
  }
  out[slot] = o;
}

__global__ void records_kernel(const abed_verify_outcome* __restrict__ outc, Kinds k, int64_t n_offset,
                               int64_t* __restrict__ rec) {
  for (int i = threadIdx.x; i < k.n; i += blockDim.x) put_record(outc[i], k.kind[i], n_offset, rec + i * kRecWords);
}

__global__ void combine_kernel(const int64_t* __restrict__ gathered, int world, Kinds k, abed_verify_outcome* out) {
  for (int i = threadIdx.x; i < k.n; i += blockDim.x) fold_slot(gathered, world, k.n, i, k.kind[i], out);
}

Kinds make_kinds(int32_t n, const int32_t* kinds) {
  if (n < 0 || n > kMaxSlots) abed_host::throw_invalid("verdicts: 0..256 outcome slots");
  Kinds k{};
  k.n = n;
  for (int i = 0; i < n; ++i) {
    if (kinds[i] < ABED_FC || kinds[i] > ABED_FIC) abed_host::throw_invalid("verdicts: unknown scheme kind");
    k.kind[i] = (int8_t)kinds[i];
  }
  return k;
}

}  // namespace

extern "C" {

int abed_verdict_records(const abed_verify_outcome* outcomes_dev, int32_t n, const int32_t* kinds_host,
                         int64_t n_offset, int64_t* records_dev, void* stream) {
  return abed_host::guarded([&] {
    const Kinds k = make_kinds(n, kinds_host);
    records_kernel<<<1, 256, 0, (cudaStream_t)stream>>>(outcomes_dev, k, n_offset, records_dev);
    abed_host::cuda_check(cudaGetLastError(), "verdict records");
  });
}

int abed_verdict_combine(const int64_t* gathered_dev, int32_t world, int32_t n, const int32_t* kinds_host,
                         abed_verify_outcome* out_dev, void* stream) {
  return abed_host::guarded([&] {
    if (world < 1) abed_host::throw_invalid("verdicts: world size must be >= 1");
    const Kinds k = make_kinds(n, kinds_host);
    combine_kernel<<<1, 256, 0, (cudaStream_t)stream>>>(gathered_dev, world, k, out_dev);
    abed_host::cuda_check(cudaGetLastError(), "verdict combine");
  });
}

int abed_verdict_records_host(const abed_verify_outcome* outcomes, int32_t n, const int32_t* kinds, int64_t n_offset,
                              int64_t* records) {
  return abed_host::guarded([&] {
    const Kinds k = make_kinds(n, kinds);
    for (int i = 0; i < n; ++i) put_record(outcomes[i], k.kind[i], n_offset, records + i * kRecWords);
  });
}

int abed_verdict_combine_host(const int64_t* gathered, int32_t world, int32_t n, const int32_t* kinds,
                              abed_verify_outcome* out) {
  return abed_host::guarded([&] {
    if (world < 1) abed_host::throw_invalid("verdicts: world size must be >= 1");
    const Kinds k = make_kinds(n, kinds);
    for (int i = 0; i < n; ++i) fold_slot(gathered, world, n, i, k.kind[i], out);
  });
}

}  // extern "C"
