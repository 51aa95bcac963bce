// Row/column-checksum ABFT for an int8 GEMM (the classical scheme the paper
// compares ABED against; reference abft_gemm.hpp:41-152) on the B200.
//
// The GEMM itself runs on the tcgen05 implicit-GEMM conv kernel as a 1x1 conv:
// A (m x k, row-major) is m pixels of k channels -- exactly the strip-plane
// layout (16 channels per 16-byte pixel), so packing A is a straight copy --
// and B (k x n) is n filters of k channels.  The checksum row of A (column sums,
// up to 8 + log2 m bits) and the checksum column of B (row sums) do not fit the
// int8 operands, so each is appended as FOUR balanced base-256 digit rows /
// filters (every digit in [-128, 127]; the digits of an int32 v recombine as
// d0 + 256 d1 + 65536 d2 + 2^24 d3 exactly).  The GEMM then produces an
// (m + 4) x (n + 4) int32 block whose digit rows / columns recombine, in int64,
// into the reference's augmented product c_aug = gemm(a_aug, b_aug, I64)
// (abft_gemm.hpp:139) bit for bit.
//
// The online tasks stay separate passes, as in the reference's cost accounting
// (abft_costs, abft_gemm.hpp:41-55): (2) copy into the augmented operands,
// (3) input checksums, (4) the larger GEMM, (5) dual output-checksum generation
// and comparison (abft_check, :70-96: rows 0..m, then columns 0..n, first
// mismatch in loop order), (6) trimmed copy-out of c.  That is the point of the
// comparison: ABED fuses its check into the conv epilogue, classical ABFT pays
// these passes over HBM.
//
// Modes of abed_abft_plan_run: ABED_ABFT_CHECKED (the reference's abft_gemm),
// ABED_ABFT_PLAIN (same GEMM pipeline, no checksums: the unprotected baseline)
// and ABED_ABFT_FUSED_ROW (the ABED-style alternative: the row check only, as the
// filter-checksum column verified inside the GEMM epilogue).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstring>

#include "abed_internal.h"

using namespace abed_dev;

namespace abed_host {
int ceil_log2_i64(int64_t v);
}

namespace {

constexpr int kDigits = 4;  // balanced base-256 digits of an int32 checksum

__device__ __forceinline__ int digit_of(int32_t v, int d) {
  int64_t rest = v;
  int dig = 0;
  for (int i = 0; i <= d; ++i) {
    dig = (int)(((rest + 128) & 0xFF) - 128);
    rest = (rest - dig) / 256;
  }
  return dig;
}

// row sums of B (k x n): the checksum column of B (task 3), one warp per row
__global__ void abft_rowsum_kernel(const int8_t* __restrict__ b, int64_t rows, int64_t cols, int32_t* __restrict__ out) {
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (warp >= rows) return;
  const int8_t* row = b + warp * cols;
  int32_t s = 0;
  for (int64_t j = lane; j < cols; j += 32) s += row[j];
  for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if (lane == 0) out[warp] = s;
}

// f[j][t] (filters KCRS, 1x1) = B[t][j] for j < n; rows n..n+3 the digits of the
// B row sums (task 2 + the B half of task 3).  32x32 tile transpose via smem.
__global__ void abft_build_filters_kernel(const int8_t* __restrict__ b, int64_t k, int64_t n,
                                          const int32_t* __restrict__ rowsum, int digits, int8_t* __restrict__ f) {
  __shared__ int8_t tile[32][33];
  const int64_t t0 = (int64_t)blockIdx.y * 32, j0 = (int64_t)blockIdx.x * 32;
  for (int r = threadIdx.y; r < 32; r += blockDim.y) {
    const int64_t t = t0 + r, j = j0 + threadIdx.x;
    int8_t v = 0;
    if (t < k) {
      if (j < n) v = b[t * n + j];
      else if (j < n + digits) v = (int8_t)digit_of(rowsum[t], (int)(j - n));
    }
    tile[r][threadIdx.x] = v;
  }
  __syncthreads();
  for (int r = threadIdx.y; r < 32; r += blockDim.y) {
    const int64_t j = j0 + r, t = t0 + threadIdx.x;
    if (j < n + digits && t < k) f[j * k + t] = tile[threadIdx.x][r];
  }
}

// A (m x k) into the strip planes of the 1 x k x 1 x (m + digits) GEMM input:
// plane g, pixel i < m = A[i][16g .. 16g + 15]; pixels m .. m+3 = digits of the
// A column sums (task 2 + the A half of task 3); zero beyond.
__global__ void abft_pack_a_kernel(const int8_t* __restrict__ a, int64_t m, int64_t k, const int32_t* __restrict__ colsum,
                                   int digits, int c16, int64_t plane_len, int8_t* __restrict__ out) {
  const int64_t total = (int64_t)c16 * plane_len;
  const bool vec = (k % 16 == 0) && ((reinterpret_cast<uintptr_t>(a) & 15) == 0);
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = idx % plane_len;
    const int g = (int)(idx / plane_len);
    const int64_t c0 = (int64_t)g * 16;
    uint4 v = make_uint4(0, 0, 0, 0);
    if (i < m && c0 < k) {
      if (vec) {
        v = *reinterpret_cast<const uint4*>(a + i * k + c0);
      } else {
        uint32_t w4[4] = {0, 0, 0, 0};
        for (int e = 0; e < 16 && c0 + e < k; ++e) w4[e >> 2] |= (uint32_t)(uint8_t)a[i * k + c0 + e] << (8 * (e & 3));
        v = make_uint4(w4[0], w4[1], w4[2], w4[3]);
      }
    } else if (i >= m && i < m + digits && c0 < k) {
      uint32_t w4[4] = {0, 0, 0, 0};
      for (int e = 0; e < 16 && c0 + e < k; ++e)
        w4[e >> 2] |= (uint32_t)(uint8_t)digit_of(colsum[c0 + e], (int)(i - m)) << (8 * (e & 3));
      v = make_uint4(w4[0], w4[1], w4[2], w4[3]);
    }
    reinterpret_cast<uint4*>(out)[idx] = v;
  }
}

// Checked mode, tasks (2) + (3) for A in ONE read of A: a block owns one 16-column
// group g and kRowsPerBlock rows; each thread copies its rows' 16-byte chunks into
// the strip planes and accumulates the 16 column sums as SIMD byte sums (x ^ 0x80
// split into two 16-bit lanes per word: 4 instr per 4 bytes, flushed to int32
// every 128 rows), then one shared-memory reduction and 16 integer atomics per
// block.  The digit pixels (m .. m+3) follow in abft_a_digits_kernel once the
// column sums are complete.
constexpr int kPackSumThreads = 256;
constexpr int kRowsPerBlock = 4096;
__global__ void __launch_bounds__(kPackSumThreads) abft_pack_a_sum_kernel(const int8_t* __restrict__ a, int64_t m,
                                                                           int64_t k, int c16, int64_t plane_len,
                                                                           int8_t* __restrict__ out,
                                                                           int32_t* __restrict__ colsum) {
  __shared__ int32_t red[16][kPackSumThreads / 32];
  const int g = blockIdx.y;
  const int64_t c0 = (int64_t)g * 16;
  const int64_t r0 = (int64_t)blockIdx.x * kRowsPerBlock;
  const int64_t r1 = min(m, r0 + kRowsPerBlock);
  const bool vec = (k % 16 == 0) && ((reinterpret_cast<uintptr_t>(a) & 15) == 0);
  int32_t acc[16];
#pragma unroll
  for (int e = 0; e < 16; ++e) acc[e] = 0;
  uint32_t ev[4] = {0, 0, 0, 0}, od[4] = {0, 0, 0, 0};
  int cnt = 0;
  int64_t rows_done = 0;
  uint4* dst = reinterpret_cast<uint4*>(out) + (int64_t)g * plane_len;
  for (int64_t i = r0 + threadIdx.x; i < r1; i += kPackSumThreads) {
    uint4 v;
    if (vec) {
      v = __ldcs(reinterpret_cast<const uint4*>(a + i * k + c0));
    } else {
      uint32_t w4[4] = {0, 0, 0, 0};
      for (int e = 0; e < 16 && c0 + e < k; ++e) w4[e >> 2] |= (uint32_t)(uint8_t)a[i * k + c0 + e] << (8 * (e & 3));
      v = make_uint4(w4[0], w4[1], w4[2], w4[3]);
    }
    dst[i] = v;
    const uint32_t w[4] = {v.x ^ 0x80808080u, v.y ^ 0x80808080u, v.z ^ 0x80808080u, v.w ^ 0x80808080u};
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      ev[q] += w[q] & 0x00FF00FFu;
      od[q] += (w[q] >> 8) & 0x00FF00FFu;
    }
    ++rows_done;
    if (++cnt == 128) {  // 128 * 255 < 2^16
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        acc[4 * q] += (int32_t)(ev[q] & 0xFFFFu);
        acc[4 * q + 1] += (int32_t)(od[q] & 0xFFFFu);
        acc[4 * q + 2] += (int32_t)(ev[q] >> 16);
        acc[4 * q + 3] += (int32_t)(od[q] >> 16);
        ev[q] = od[q] = 0;
      }
      cnt = 0;
    }
  }
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    acc[4 * q] += (int32_t)(ev[q] & 0xFFFFu);
    acc[4 * q + 1] += (int32_t)(od[q] & 0xFFFFu);
    acc[4 * q + 2] += (int32_t)(ev[q] >> 16);
    acc[4 * q + 3] += (int32_t)(od[q] >> 16);
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int e = 0; e < 16; ++e) {
    int32_t v = acc[e] - 128 * (int32_t)rows_done;  // un-bias x ^ 0x80 = x + 128
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (lane == 0) red[e][warp] = v;
  }
  __syncthreads();
  if (threadIdx.x < 16 && c0 + threadIdx.x < k) {
    int32_t t = 0;
    for (int w = 0; w < kPackSumThreads / 32; ++w) t += red[threadIdx.x][w];
    atomicAdd(colsum + c0 + threadIdx.x, t);
  }
}

// digit pixels m .. m+3 of every channel group, and zero pixels m+4 .. plane_len
__global__ void abft_a_digits_kernel(int64_t m, int64_t k, const int32_t* __restrict__ colsum, int digits, int c16,
                                     int64_t plane_len, int8_t* __restrict__ out) {
  const int64_t tail = plane_len - m;
  const int64_t total = (int64_t)c16 * tail;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int g = (int)(idx / tail);
    const int64_t i = m + idx % tail;
    const int64_t c0 = (int64_t)g * 16;
    uint4 v = make_uint4(0, 0, 0, 0);
    if (i < m + digits && c0 < k) {
      uint32_t w4[4] = {0, 0, 0, 0};
      for (int e = 0; e < 16 && c0 + e < k; ++e)
        w4[e >> 2] |= (uint32_t)(uint8_t)digit_of(colsum[c0 + e], (int)(i - m)) << (8 * (e & 3));
      v = make_uint4(w4[0], w4[1], w4[2], w4[3]);
    }
    reinterpret_cast<uint4*>(out)[(int64_t)g * plane_len + i] = v;
  }
}

// GEMM output o[j][i] (K-major: (n + dn) x (m + dm) int32) -> c_aug (m+1) x (n+1)
// int64 with the digit rows / columns recombined, and/or the trimmed c (m x n
// int32, task 6).  32x32 tiles over (i, j) of c_aug through shared memory.
__global__ void abft_assemble_kernel(const int32_t* __restrict__ o, int64_t m, int64_t n, int digits,
                                     int64_t* __restrict__ c_aug, int32_t* __restrict__ c) {
  __shared__ int64_t tile[32][33];
  const int64_t ld = m + digits;  // o row length
  const int64_t i0 = (int64_t)blockIdx.x * 32, j0 = (int64_t)blockIdx.y * 32;
  const int64_t mi = digits ? m + 1 : m, nj = digits ? n + 1 : n;
  // read: consecutive threads take consecutive i (coalesced in o)
  for (int r = threadIdx.y; r < 32; r += blockDim.y) {
    const int64_t j = j0 + r, i = i0 + threadIdx.x;
    int64_t v = 0;
    if (i < mi && j < nj) {
      if (i < m && j < n) {
        v = o[j * ld + i];
      } else if (i < m) {  // checksum column: sum_d 256^d o[n+d][i]
        for (int d = digits - 1; d >= 0; --d) v = v * 256 + o[(n + d) * ld + i];
      } else if (j < n) {  // checksum row: sum_e 256^e o[j][m+e]
        for (int e = digits - 1; e >= 0; --e) v = v * 256 + o[j * ld + m + e];
      } else {             // corner: sum_{d,e} 256^(d+e) o[n+d][m+e]
        for (int d = digits - 1; d >= 0; --d) {
          int64_t row = 0;
          for (int e = digits - 1; e >= 0; --e) row = row * 256 + o[(n + d) * ld + m + e];
          v = v * 256 + row;
        }
      }
    }
    tile[r][threadIdx.x] = v;
  }
  __syncthreads();
  // write: consecutive threads take consecutive j (coalesced in c_aug / c)
  for (int r = threadIdx.y; r < 32; r += blockDim.y) {
    const int64_t i = i0 + r, j = j0 + threadIdx.x;
    if (i < mi && j < nj) {
      const int64_t v = tile[threadIdx.x][r];
      if (c_aug) c_aug[i * (n + 1) + j] = v;
      if (c && i < m && j < n) c[i * n + j] = (int32_t)v;
    }
  }
}

// task 5, pass 1: row i (0..m) sum over j < n vs c_aug[i][n]; one warp per row
// (unsigned arithmetic: the reference's int64 sums, wrapped deterministically)
__global__ void abft_row_check_kernel(const int64_t* __restrict__ c_aug, int64_t m, int64_t n,
                                      unsigned long long* __restrict__ rsum, unsigned long long* __restrict__ ws) {
  const int64_t i = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (i > m) return;
  const unsigned long long* row = reinterpret_cast<const unsigned long long*>(c_aug) + i * (n + 1);
  unsigned long long s = 0;
  for (int64_t j = lane; j < n; j += 32) s += row[j];
  for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if (lane == 0) {
    rsum[i] = s;
    if (s != row[n]) {
      atomicMin(ws + 0, (unsigned long long)i);
      atomicAdd(ws + 1, 1ull);
    }
  }
}

// task 5, pass 2: column sums over i < m (blocks split the rows, integer atomics)
__global__ void abft_col_sum_kernel(const int64_t* __restrict__ c_aug, int64_t m, int64_t n, int64_t rows_per,
                                    unsigned long long* __restrict__ csum) {
  __shared__ unsigned long long part[8][33];
  const int64_t j = (int64_t)blockIdx.x * 32 + threadIdx.x;
  const int64_t r0 = (int64_t)blockIdx.y * rows_per, r1 = min(m, r0 + rows_per);
  unsigned long long s = 0;
  if (j <= n)
    for (int64_t i = r0 + threadIdx.y; i < r1; i += blockDim.y)
      s += reinterpret_cast<const unsigned long long*>(c_aug)[i * (n + 1) + j];
  part[threadIdx.y][threadIdx.x] = s;
  __syncthreads();
  if (threadIdx.y == 0 && j <= n) {
    for (int y = 1; y < (int)blockDim.y; ++y) s += part[y][threadIdx.x];
    atomicAdd(csum + j, s);
  }
}

__global__ void abft_col_cmp_kernel(const int64_t* __restrict__ c_aug, int64_t m, int64_t n,
                                    const unsigned long long* __restrict__ csum, unsigned long long* __restrict__ ws) {
  const int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (j > n) return;
  if (csum[j] != reinterpret_cast<const unsigned long long*>(c_aug)[m * (n + 1) + j]) {
    atomicMin(ws + 2, (unsigned long long)j);
    atomicAdd(ws + 3, 1ull);
  }
}

__device__ void put_outcome(abed_verify_outcome* o, unsigned long long first, unsigned long long count, int64_t lhs,
                            int64_t rhs) {
  abed_verify_outcome v;
  memset(&v, 0, sizeof(v));
  if (count) {
    v.status = 1;
    v.has_locus = 1;
    v.locus[0] = (int64_t)first;
    v.locus[1] = -1;
    v.locus[2] = -1;
    v.lhs = lhs;
    v.rhs = rhs;
    v.error_count = (int64_t)count;
  }
  *o = v;
}

// VerifyOutcome::fail(sum, want, {index, -1, -1}) for the first mismatching row
// and column (abft_gemm.hpp:76-94); ok() (all zero) otherwise
__global__ void abft_finalize_kernel(const int64_t* __restrict__ c_aug, int64_t m, int64_t n,
                                     const unsigned long long* __restrict__ rsum, const unsigned long long* __restrict__ csum,
                                     const unsigned long long* __restrict__ ws, abed_verify_outcome* out) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  const unsigned long long ri = ws[0], ci = ws[2];
  put_outcome(out + 0, ri, ws[1], ws[1] ? (int64_t)rsum[ri] : 0, ws[1] ? c_aug[ri * (n + 1) + n] : 0);
  put_outcome(out + 1, ci, ws[3], ws[3] ? (int64_t)csum[ci] : 0, ws[3] ? c_aug[m * (n + 1) + ci] : 0);
}

// fused-row mode: the conv plan's FC verdict (locus (0, 0, i) of the 1 x n x 1 x m
// output) restated as the ABFT row check (locus (i, -1, -1)); no column check
__global__ void abft_fc_to_row_kernel(const abed_verify_outcome* fc, abed_verify_outcome* out) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  abed_verify_outcome v = *fc;
  if (v.status) {
    v.locus[0] = v.locus[2];
    v.locus[1] = -1;
    v.locus[2] = -1;
  }
  out[0] = v;
  abed_verify_outcome z;
  memset(&z, 0, sizeof(z));
  out[1] = z;
}

// ---------------------------------------------------------------- check workspace
struct CheckWs {
  unsigned long long* rsum = nullptr;  // m + 1
  unsigned long long* csum = nullptr;  // n + 1
  unsigned long long* ws = nullptr;    // {first row, rows bad, first col, cols bad}
};

void check_ws_alloc(CheckWs& w, int64_t m, int64_t n) {
  abed_host::cuda_check(cudaMalloc(&w.rsum, (size_t)(m + 1) * 8), "cudaMalloc(abft rsum)");
  abed_host::cuda_check(cudaMalloc(&w.csum, (size_t)(n + 1) * 8), "cudaMalloc(abft csum)");
  abed_host::cuda_check(cudaMalloc(&w.ws, 4 * 8), "cudaMalloc(abft ws)");
}
void check_ws_free(CheckWs& w) {
  cudaFree(w.rsum);
  cudaFree(w.csum);
  cudaFree(w.ws);
  w = CheckWs{};
}

// abft_check (abft_gemm.hpp:70-96) on a device c_aug, asynchronous
void launch_check(const int64_t* c_aug, int64_t m, int64_t n, CheckWs& w, abed_verify_outcome* out_dev, cudaStream_t st) {
  using abed_host::cuda_check;
  // ws = {first bad row = ~0, rows bad = 0, first bad column = ~0, columns bad = 0}
  cuda_check(cudaMemsetAsync(w.ws, 0xFF, 8 * 4, st), "abft ws");
  cuda_check(cudaMemsetAsync(w.ws + 1, 0, 8, st), "abft ws");
  cuda_check(cudaMemsetAsync(w.ws + 3, 0, 8, st), "abft ws");
  cuda_check(cudaMemsetAsync(w.csum, 0, (size_t)(n + 1) * 8, st), "abft csum");
  const int64_t rows = m + 1;
  abft_row_check_kernel<<<(unsigned)((rows * 32 + 255) / 256), 256, 0, st>>>(c_aug, m, n, w.rsum, w.ws);
  // column pass: ~8 resident blocks per SM over the row range
  const int64_t col_tiles = (n + 1 + 31) / 32;
  int64_t splits = std::max<int64_t>(1, (int64_t)abed_host::num_sms() * 8 / col_tiles);
  int64_t rows_per = std::max<int64_t>(64, (m + splits - 1) / splits);
  splits = (m + rows_per - 1) / rows_per;
  abft_col_sum_kernel<<<dim3((unsigned)col_tiles, (unsigned)splits), dim3(32, 8), 0, st>>>(c_aug, m, n, rows_per, w.csum);
  abft_col_cmp_kernel<<<(unsigned)((n + 1 + 255) / 256), 256, 0, st>>>(c_aug, m, n, w.csum, w.ws);
  abft_finalize_kernel<<<1, 32, 0, st>>>(c_aug, m, n, w.rsum, w.csum, w.ws, out_dev);
  cuda_check(cudaGetLastError(), "abft_check");
}

void validate_abft(int64_t m, int64_t n, int64_t k) {
  using abed_host::throw_invalid;
  if (m < 1 || n < 1 || k < 1) throw_invalid("abft_gemm: extents must be >= 1");
  // abft_gemm.hpp:108-111
  if (16 + abed_host::ceil_log2_i64(m * n * k) > 63)
    throw_invalid("abft_gemm: checksum accumulation would overflow i64");
  if (16 + abed_host::ceil_log2_i64(k) > 31)
    throw_invalid("abft_gemm: product accumulation would overflow the i32 output");
  // device plan: four int8 digits hold any int32 checksum; the GEMM row count is an int
  if (m > (int64_t(1) << 24) || n > (int64_t(1) << 24))
    throw_invalid("abft_gemm: m and n are limited to 2^24 on the device plan");
}

}  // namespace

namespace abed_host {
int ceil_log2_i64(int64_t v) {  // checksum.hpp:53-62
  int b = 0;
  while (b < 63 && (int64_t(1) << b) < v) ++b;
  return b;
}
}  // namespace abed_host

struct abed_abft_plan {
  int64_t m = 0, n = 0, k = 0;
  abed_conv_plan* aug = nullptr;    // (m+4)-pixel x (n+4)-filter GEMM, no checks
  abed_conv_plan* plain = nullptr;  // m x n GEMM, no checks
  abed_conv_plan* fused = nullptr;  // m x n GEMM, FC row check in the epilogue
  int8_t* f = nullptr;              // transposed (n+4) x k filters
  int8_t* packed = nullptr;         // packed A (sized for the augmented plan)
  int32_t* colsum = nullptr;        // k
  int32_t* rowsum = nullptr;        // k
  int32_t* out = nullptr;           // (n+4) x (m+4) GEMM output
  abed_verify_outcome* fc_out = nullptr;  // 3 outcomes of the fused plan
  CheckWs ws;
  int b_packed[3] = {0, 0, 0};      // per mode: B already packed by an earlier run
};

namespace {
using namespace abed_host;

abed_layer_shape gemm_shape(int64_t m, int64_t n, int64_t k, int digits) {
  abed_layer_shape s{};
  s.n = 1; s.c = k; s.h = 1; s.w = m + digits; s.k = n + digits; s.r = 1; s.s = 1;
  s.stride_h = 1; s.stride_w = 1; s.pad_h = 0; s.pad_w = 0; s.p = 1; s.q = m + digits;
  return s;
}

void destroy(abed_abft_plan* p) {
  if (!p) return;
  if (p->aug) abed_conv_plan_destroy(p->aug);
  if (p->plain) abed_conv_plan_destroy(p->plain);
  if (p->fused) abed_conv_plan_destroy(p->fused);
  cudaFree(p->f);
  cudaFree(p->packed);
  cudaFree(p->colsum);
  cudaFree(p->rowsum);
  cudaFree(p->out);
  cudaFree(p->fc_out);
  check_ws_free(p->ws);
  delete p;
}

abed_conv_plan* gemm_plan(abed_abft_plan* p, int digits, int checks) {
  // the plan packs its filters again on every run; create it from zeros
  const abed_layer_shape s = gemm_shape(p->m, p->n, p->k, digits);
  cuda_check(cudaMemset(p->f, 0, (size_t)(p->n + kDigits) * p->k), "abft zero filters");
  return plan_create(s, p->f, checks, 0);
}

void run(abed_abft_plan* p, const int8_t* a, const int8_t* b, int32_t* c, int64_t* c_aug,
         abed_verify_outcome* out_dev, int mode, cudaStream_t st) {
  const int64_t m = p->m, n = p->n, k = p->k;
  const int digits = mode == ABED_ABFT_CHECKED ? kDigits : 0;
  abed_conv_plan* pl = mode == ABED_ABFT_CHECKED ? p->aug : mode == ABED_ABFT_PLAIN ? p->plain : p->fused;
  const ActGeom& g = pl->g;
  if (b) {
    // B side (skipped when b == NULL: B stays packed from an earlier run, i.e. the
    // weights-offline setting ABED's filter checksum assumes)
    if (digits) abft_rowsum_kernel<<<(unsigned)((k * 32 + 255) / 256), 256, 0, st>>>(b, k, n, p->rowsum);
    // task 2: B into filters (transposed) with the checksum column's digits
    abft_build_filters_kernel<<<dim3((unsigned)((n + digits + 31) / 32), (unsigned)((k + 31) / 32)), dim3(32, 8), 0, st>>>(
        b, k, n, p->rowsum, digits, p->f);
    const ConvTcParams& cp = pl->base;
    const int64_t frows = (int64_t)cp.n_tiles * cp.k_stages * cp.ntaps * cp.gps * cp.block_n_tot;
    pack_filters_kernel<<<grid_for(frows, 256), 256, 0, st>>>(p->f, g, cp.block_n, cp.block_n_tot, cp.n_tiles, cp.gps,
                                                             cp.k_stages, (pl->checks & ABED_CHECK_FC) ? 1 : 0, pl->d_wpk);
    p->b_packed[mode] = 1;
  } else if (!p->b_packed[mode]) {
    throw_invalid("abft plan: b == NULL before B was packed by a run in this mode");
  }
  if (digits) {
    // tasks 2 + 3 for A in one read: strip-plane copy + column sums, then the
    // checksum row's digit pixels
    cuda_check(cudaMemsetAsync(p->colsum, 0, (size_t)k * 4, st), "abft colsum");
    const dim3 grid((unsigned)((m + kRowsPerBlock - 1) / kRowsPerBlock), (unsigned)g.c16);
    abft_pack_a_sum_kernel<<<grid, kPackSumThreads, 0, st>>>(a, m, k, g.c16, g.plane_len, p->packed, p->colsum);
    const int64_t nt = (int64_t)g.c16 * (g.plane_len - m);
    abft_a_digits_kernel<<<grid_for(nt, 256), 256, 0, st>>>(m, k, p->colsum, digits, g.c16, g.plane_len, p->packed);
  } else {
    // task 2: A into the strip planes
    const int64_t n16 = (int64_t)g.c16 * g.plane_len;
    abft_pack_a_kernel<<<grid_for(n16, 256), 256, 0, st>>>(a, m, k, p->colsum, 0, g.c16, g.plane_len, p->packed);
  }
  cuda_check(cudaGetLastError(), "abft operands");
  // task 4: the (larger) GEMM on tcgen05
  plan_run(pl, p->packed, nullptr, ABED_OUT_I32_NCHW, p->out, nullptr, -1, 0, st);
  // task 5 (+ 6): assemble c_aug / c, then the dual output-checksum comparison
  const int64_t mi = digits ? m + 1 : m, nj = digits ? n + 1 : n;
  abft_assemble_kernel<<<dim3((unsigned)((mi + 31) / 32), (unsigned)((nj + 31) / 32)), dim3(32, 8), 0, st>>>(
      p->out, m, n, digits, digits ? c_aug : nullptr, c);
  cuda_check(cudaGetLastError(), "abft assemble");
  if (mode == ABED_ABFT_CHECKED) {
    launch_check(c_aug, m, n, p->ws, out_dev, st);
  } else if (mode == ABED_ABFT_FUSED_ROW && out_dev) {
    plan_finalize(pl, p->fc_out, st);
    abft_fc_to_row_kernel<<<1, 32, 0, st>>>(p->fc_out, out_dev);
    cuda_check(cudaGetLastError(), "abft fused verdict");
  }
}

// all_modes: build the plain and fused GEMM plans too (abed_abft_plan_create, so
// later runs in any mode stay allocation- and sync-free for graph capture); the
// one-shot abed_abft_gemm_i8 runs only the checked mode and builds only `aug`.
abed_abft_plan* create(int64_t m, int64_t n, int64_t k, bool all_modes) {
  require_device();
  validate_abft(m, n, k);
  auto* p = new abed_abft_plan();
  p->m = m; p->n = n; p->k = k;
  try {
      cuda_check(cudaMalloc(&p->f, (size_t)(n + kDigits) * k), "cudaMalloc(abft f)");
      cuda_check(cudaMalloc(&p->colsum, (size_t)k * 4), "cudaMalloc(abft colsum)");
      cuda_check(cudaMalloc(&p->rowsum, (size_t)k * 4), "cudaMalloc(abft rowsum)");
      cuda_check(cudaMalloc(&p->out, (size_t)(n + kDigits) * (m + kDigits) * 4), "cudaMalloc(abft out)");
      cuda_check(cudaMalloc(&p->fc_out, 3 * sizeof(abed_verify_outcome)), "cudaMalloc(abft fc)");
      check_ws_alloc(p->ws, m, n);
      p->aug = gemm_plan(p, kDigits, 0);
      if (all_modes) {
        p->plain = gemm_plan(p, 0, 0);
        p->fused = gemm_plan(p, 0, ABED_CHECK_FC);
      }
      cuda_check(cudaMalloc(&p->packed, (size_t)geom_packed_bytes(p->aug->g)), "cudaMalloc(abft packed)");
  } catch (...) {
    destroy(p);
    throw;
  }
  return p;
}

}  // namespace

extern "C" {

int abed_abft_plan_create(int64_t m, int64_t n, int64_t k, abed_abft_plan** plan) {
  return guarded([&] { *plan = create(m, n, k, true); });
}

int abed_abft_plan_destroy(abed_abft_plan* plan) {
  return guarded([&] { destroy(plan); });
}

int abed_abft_plan_run(abed_abft_plan* plan, const int8_t* a, const int8_t* b, int32_t* c, int64_t* c_aug,
                       abed_verify_outcome* outcomes_dev, int32_t mode, void* stream) {
  return guarded([&] {
    if (!plan) throw_invalid("abft plan is null");
    if (mode != ABED_ABFT_CHECKED && mode != ABED_ABFT_PLAIN && mode != ABED_ABFT_FUSED_ROW)
      throw_invalid("abft mode must be ABED_ABFT_CHECKED / _PLAIN / _FUSED_ROW");
    if (mode == ABED_ABFT_CHECKED && (!c_aug || !outcomes_dev))
      throw_invalid("abft_gemm: the checked mode needs c_aug and the outcome buffer");
    run(plan, a, b, c, c_aug, outcomes_dev, mode, (cudaStream_t)stream);
  });
}

int abed_abft_gemm_i8(const int8_t* a, int64_t m, int64_t k, const int8_t* b, int64_t kb, int64_t n, int32_t* c,
                      int64_t* c_aug, abed_verify_outcome* row_check, abed_verify_outcome* col_check) {
  return guarded([&] {
    if (k != kb) throw_invalid("abft_gemm: inner dimensions do not match");
    abed_abft_plan* p = create(m, n, k, false);
    abed_verify_outcome* d_out = nullptr;
    try {
      cuda_check(cudaMalloc(&d_out, 2 * sizeof(abed_verify_outcome)), "cudaMalloc(abft outcomes)");
      run(p, a, b, c, c_aug, d_out, ABED_ABFT_CHECKED, nullptr);
      abed_verify_outcome h[2];
      cuda_check(cudaMemcpy(h, d_out, sizeof(h), cudaMemcpyDeviceToHost), "abft outcomes d2h");
      if (row_check) *row_check = h[0];
      if (col_check) *col_check = h[1];
    } catch (...) {
      cudaFree(d_out);
      destroy(p);
      throw;
    }
    cudaFree(d_out);
    destroy(p);
  });
}

int abed_abft_check(const int64_t* c_aug, int64_t rows, int64_t cols, abed_verify_outcome* row_check,
                    abed_verify_outcome* col_check) {
  return guarded([&] {
    const int64_t m = rows - 1, n = cols - 1;
    if (m < 1 || n < 1) throw_invalid("abft_check: matrix too small");  // abft_gemm.hpp:73
    require_device();
    CheckWs w;
    abed_verify_outcome* d_out = nullptr;
    try {
      check_ws_alloc(w, m, n);
      cuda_check(cudaMalloc(&d_out, 2 * sizeof(abed_verify_outcome)), "cudaMalloc(abft outcomes)");
      launch_check(c_aug, m, n, w, d_out, nullptr);
      abed_verify_outcome h[2];
      cuda_check(cudaMemcpy(h, d_out, sizeof(h), cudaMemcpyDeviceToHost), "abft outcomes d2h");
      if (row_check) *row_check = h[0];
      if (col_check) *col_check = h[1];
    } catch (...) {
      check_ws_free(w);
      cudaFree(d_out);
      throw;
    }
    check_ws_free(w);
    cudaFree(d_out);
  });
}

}  // extern "C"
