// C ABI: the reference-facing L0-L2 functions other than the tensor-core conv.
// Each kernel restates one reference function on the device; integer
// reductions are exact (order-independent) and float-mode reductions keep the
// reference's sequential order so results are bit-identical to its -march=native
// build (FMA contraction spelled out with fma/fmaf).
#include <cooperative_groups.h>
#include <cuda_runtime.h>
#include <cstdlib>

#include <cmath>
#include <cstring>
#include <type_traits>
#include <vector>

#include "abed_internal.h"

using namespace abed_host;

namespace abed_host {
int grid_for(int64_t n, int threads);
void require_device();
void validate_shape(const abed_layer_shape& s);
}  // namespace abed_host

namespace {

constexpr uint64_t kGolden = 0x9E3779B97F4A7C15ULL;

__host__ __device__ inline uint64_t mix64(uint64_t z) {  // rng.hpp:16-19
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

// ------------------------------------------------------------------- rng
// fill_random_i8 (rng.hpp:46): element i of a stream is mix(seed + (i+1)*golden),
// so the fill is embarrassingly parallel.
__global__ void fill_i8_kernel(int8_t* t, int64_t n, uint64_t seed, uint64_t off, int extreme) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t v = mix64(seed + (uint64_t)(off + i + 1) * kGolden);
    t[i] = extreme ? ((v & 1) ? (int8_t)127 : (int8_t)-128) : (int8_t)(v & 0xFF);
  }
}

// ------------------------------------------------------------- direct conv
// conv_reference (convolution.hpp:78-111) for the widened instantiations the
// reference uses off the int8 hot path; one thread per output, window walked in
// (c,r,s) order.
template <typename TX, typename TW, typename TA>
__global__ void conv_direct_kernel(const TX* __restrict__ x, const TW* __restrict__ f, abed_layer_shape s,
                                   TA* __restrict__ out) {
  const int64_t total = s.n * s.k * s.p * s.q;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total; idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t q = idx % s.q, p = (idx / s.q) % s.p, k = (idx / (s.q * s.p)) % s.k, n = idx / (s.q * s.p * s.k);
    TA acc = 0;
    for (int64_t c = 0; c < s.c; ++c)
      for (int64_t r = 0; r < s.r; ++r) {
        const int64_t hi = p * s.stride_h - s.pad_h + r;
        if (hi < 0 || hi >= s.h) continue;
        for (int64_t ss = 0; ss < s.s; ++ss) {
          const int64_t wi = q * s.stride_w - s.pad_w + ss;
          if (wi < 0 || wi >= s.w) continue;
          const TA xv = (TA)x[((n * s.c + c) * s.h + hi) * s.w + wi];
          const TA fv = (TA)f[((k * s.c + c) * s.r + r) * s.s + ss];
          if constexpr (std::is_same<TA, float>::value) acc = __fmaf_rn(xv, fv, acc);
          else acc += xv * fv;
        }
      }
    out[idx] = acc;
  }
}

// conv_checksum_planes (checksum.hpp:134-176): 4 plane filters, planes 0-2 as u8, 3 as s8
__global__ void planes_conv_kernel(const int8_t* __restrict__ x, abed_layer_shape s, const int8_t* __restrict__ planes,
                                   int32_t* __restrict__ extra) {
  const int64_t npq = s.n * s.p * s.q, crs = s.c * s.r * s.s;
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < npq; j += (int64_t)gridDim.x * blockDim.x) {
    const int64_t q = j % s.q, p = (j / s.q) % s.p, n = j / (s.q * s.p);
    uint32_t a0 = 0, a1 = 0, a2 = 0, a3 = 0;
    for (int64_t c = 0; c < s.c; ++c)
      for (int64_t r = 0; r < s.r; ++r) {
        const int64_t hi = p * s.stride_h - s.pad_h + r;
        if (hi < 0 || hi >= s.h) continue;
        for (int64_t ss = 0; ss < s.s; ++ss) {
          const int64_t wi = q * s.stride_w - s.pad_w + ss;
          if (wi < 0 || wi >= s.w) continue;
          const int32_t xv = x[((n * s.c + c) * s.h + hi) * s.w + wi];
          const int64_t i = (c * s.r + r) * s.s + ss;
          a0 += (uint32_t)(xv * (int32_t)(uint8_t)planes[i]);
          a1 += (uint32_t)(xv * (int32_t)(uint8_t)planes[crs + i]);
          a2 += (uint32_t)(xv * (int32_t)(uint8_t)planes[2 * crs + i]);
          a3 += (uint32_t)(xv * (int32_t)planes[3 * crs + i]);
        }
      }
    extra[j] = (int32_t)a0;
    extra[npq + j] = (int32_t)a1;
    extra[2 * npq + j] = (int32_t)a2;
    extra[3 * npq + j] = (int32_t)a3;
  }
}

// ------------------------------------------------------------------ epilog
__global__ void epilog_kernel(const int32_t* __restrict__ in, abed_dims4 d, float scale, const float* __restrict__ bias,
                              int relu, int f32out, void* __restrict__ out) {
  const int64_t total = d.d0 * d.d1 * d.d2 * d.d3, pq = d.d2 * d.d3;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t k = (i / pq) % d.d1;
    float v = __fmaf_rn((float)in[i], scale, bias[k]);  // convolution.hpp:374 (FMA-contracted)
    if (relu && v < 0.0f) v = 0.0f;
    if (f32out) {
      static_cast<float*>(out)[i] = v;
    } else {
      v = fminf(127.0f, fmaxf(-128.0f, v));
      static_cast<int8_t*>(out)[i] = (int8_t)truncf(v);
    }
  }
}

// The same epilog on 16 consecutive outputs per thread (P*Q % 16 == 0, aligned
// buffers): one channel per vector, 64-byte loads, 16-byte (i8) or 64-byte (f32)
// stores -- HBM-bound, so the vector width is what sets the achieved bandwidth.
__device__ __forceinline__ float epilog_one(int32_t a, float scale, float b, int relu) {
  float v = __fmaf_rn(static_cast<float>(a), scale, b);
  if (relu && v < 0.0f) v = 0.0f;
  return v;
}
__global__ void __launch_bounds__(256) epilog_v16_kernel(const int32_t* __restrict__ in, abed_dims4 d, float scale,
                                                         const float* __restrict__ bias, int relu, int f32out,
                                                         void* __restrict__ out) {
  const int64_t total16 = d.d0 * d.d1 * d.d2 * d.d3 / 16, pq16 = d.d2 * d.d3 / 16;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total16; i += (int64_t)gridDim.x * blockDim.x) {
    const float b = __ldg(bias + (i / pq16) % d.d1);
    const int4* src = reinterpret_cast<const int4*>(in) + i * 4;
    int4 a[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) a[u] = __ldcs(src + u);
    float v[16];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      v[4 * u] = epilog_one(a[u].x, scale, b, relu);
      v[4 * u + 1] = epilog_one(a[u].y, scale, b, relu);
      v[4 * u + 2] = epilog_one(a[u].z, scale, b, relu);
      v[4 * u + 3] = epilog_one(a[u].w, scale, b, relu);
    }
    if (f32out) {
      float4* dst = reinterpret_cast<float4*>(out) + i * 4;
#pragma unroll
      for (int u = 0; u < 4; ++u) dst[u] = make_float4(v[4 * u], v[4 * u + 1], v[4 * u + 2], v[4 * u + 3]);
    } else {
      uint32_t w[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        uint32_t acc = 0;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const int32_t q = static_cast<int32_t>(truncf(fminf(127.0f, fmaxf(-128.0f, v[4 * u + j]))));
          acc |= (static_cast<uint32_t>(q) & 0xFFu) << (8 * j);
        }
        w[u] = acc;
      }
      reinterpret_cast<uint4*>(out)[i] = make_uint4(w[0], w[1], w[2], w[3]);
    }
  }
}

// ---------------------------------------------------------- checksum kernels
__global__ void decompose_kernel(const int32_t* __restrict__ sums, int64_t n, int8_t* __restrict__ planes) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t u = (uint32_t)sums[i];  // checksum.hpp:93-97
    for (int b = 0; b < 4; ++b) planes[b * n + i] = (int8_t)(uint8_t)(u >> (8 * b));
  }
}
__global__ void recombine_kernel(const int32_t* __restrict__ e, int64_t n, int64_t* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = (int64_t)e[i] + ((int64_t)e[n + i] << 8) + ((int64_t)e[2 * n + i] << 16) + ((int64_t)e[3 * n + i] << 24);
}
// Column sums of a rows x len int8 matrix into int32 -- the shape of both
// gen_filter_checksum (rows = K filters of len = C*R*S, checksum.hpp:75-90) and
// ic_batch_checksum (rows = N images of len = C*H*W, :350-362).  HBM-bound.  A
// block owns 512 adjacent columns (32 lanes x one 16-byte vector) of a range of
// rows; its 8 warps stride the rows (each warp load is 512 contiguous bytes, four
// rows in flight per thread), reduce through shared memory, and write each column
// once -- with an integer atomic only when several blocks split the rows (exact
// and deterministic either way).  `out` must be zeroed when row_splits > 1.
constexpr int kColsumWarps = 8;
// Cluster variant (no atomics, no memset): the row splits of one 512-column tile
// form a thread-block cluster; every CTA reduces its rows into shared memory, then
// each CTA sums its share of the tile's columns across the cluster's CTAs through
// distributed shared memory and stores them.  One launch, plain stores.
__global__ void __launch_bounds__(kColsumWarps * 32) colsum_i8_cluster_kernel(const int8_t* __restrict__ x,
                                                                            int64_t rows, int64_t len,
                                                                            int64_t rows_per,
                                                                            int32_t* __restrict__ out) {
  namespace cg = cooperative_groups;
  cg::cluster_group cluster = cg::this_cluster();
  __shared__ int32_t red[kColsumWarps][16][32];
  __shared__ int32_t s_part[512];
  const int cs = static_cast<int>(cluster.num_blocks());
  const int rank = static_cast<int>(cluster.block_rank());
  const int64_t cols16 = len >> 4;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t tile = blockIdx.x / cs;
  const int64_t c16 = tile * 32 + lane;
  const int64_t r0 = rank * rows_per, r1 = r0 + rows_per < rows ? r0 + rows_per : rows;
  int32_t acc[16];
#pragma unroll
  for (int j = 0; j < 16; ++j) acc[j] = 0;
  if (c16 < cols16) {
    // the warp's rows r0 + warp, + 8, ...: batches of 16 rows with every load
    // issued before use (pointer increments, no predicates), then a masked batch
    const int64_t step = (int64_t)kColsumWarps * cols16;  // uint4 stride between a warp's rows
    const uint4* ptr = reinterpret_cast<const uint4*>(x) + c16 + (r0 + warp) * cols16;
    const int64_t mine = r1 - r0 > warp ? (r1 - r0 - warp + kColsumWarps - 1) / kColsumWarps : 0;
    int64_t done = 0;
    while (done < mine) {
      uint32_t ev[4] = {0u, 0u, 0u, 0u}, od[4] = {0u, 0u, 0u, 0u};
      int64_t batch_end = done + 256 < mine ? done + 256 : mine;  // 16-bit lanes: <= 256 rows per flush
      for (; done + 16 <= batch_end; done += 16) {  // 16 x 16 B in flight per thread
        uint4 v[16];
#pragma unroll
        for (int u = 0; u < 16; ++u) v[u] = __ldcs(ptr + u * step);
        ptr += 16 * step;
#pragma unroll
        for (int u = 0; u < 16; ++u) {
          const uint32_t w[4] = {v[u].x ^ 0x80808080u, v[u].y ^ 0x80808080u, v[u].z ^ 0x80808080u,
                                 v[u].w ^ 0x80808080u};
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            ev[q] += w[q] & 0x00FF00FFu;
            od[q] += (w[q] >> 8) & 0x00FF00FFu;
          }
        }
      }
      if (done < batch_end) {  // masked last batch: every load still issued before use
        const int rem = static_cast<int>(batch_end - done);
        uint4 v[16];
#pragma unroll
        for (int u = 0; u < 16; ++u)
          v[u] = u < rem ? __ldcs(ptr + u * step) : make_uint4(0x80808080u, 0x80808080u, 0x80808080u, 0x80808080u);
        ptr += rem * step;
        done = batch_end;
#pragma unroll
        for (int u = 0; u < 16; ++u) {  // padding slots add (0x80 ^ 0x80) = 0
          const uint32_t w[4] = {v[u].x ^ 0x80808080u, v[u].y ^ 0x80808080u, v[u].z ^ 0x80808080u,
                                 v[u].w ^ 0x80808080u};
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            ev[q] += w[q] & 0x00FF00FFu;
            od[q] += (w[q] >> 8) & 0x00FF00FFu;
          }
        }
      }
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        acc[4 * q] += static_cast<int32_t>(ev[q] & 0xFFFFu);
        acc[4 * q + 1] += static_cast<int32_t>(od[q] & 0xFFFFu);
        acc[4 * q + 2] += static_cast<int32_t>(ev[q] >> 16);
        acc[4 * q + 3] += static_cast<int32_t>(od[q] >> 16);
      }
    }
#pragma unroll
    for (int j = 0; j < 16; ++j) acc[j] -= static_cast<int32_t>(128 * mine);
  }
#pragma unroll
  for (int j = 0; j < 16; ++j) red[warp][j][lane] = acc[j];
  __syncthreads();
  for (int e = threadIdx.x; e < 512; e += kColsumWarps * 32) {
    const int j = e >> 5, ln = e & 31;
    int32_t sum = 0;
#pragma unroll
    for (int q = 0; q < kColsumWarps; ++q) sum += red[q][j][ln];
    s_part[ln * 16 + j] = sum;  // column tile * 512 + ln * 16 + j
  }
  cluster.sync();
  const int per = (512 + cs - 1) / cs;
  for (int cl = rank * per + threadIdx.x; cl < (rank + 1) * per && cl < 512; cl += kColsumWarps * 32) {
    const int64_t col = tile * 512 + cl;
    if (col >= len) continue;
    int32_t sum = 0;
    for (int q = 0; q < cs; ++q) sum += cluster.map_shared_rank(s_part, q)[cl];
    out[col] = sum;
  }
  cluster.sync();  // keep this CTA's partials alive until every peer has read them
}

// Wide variant for long rows (the batch checksum: 256 images x 200704 bytes): a
// CTA owns 4096 adjacent columns (256 threads x one 16-byte vector, so one load
// instruction of the CTA reads 4 KB contiguous of one row -- whole DRAM pages,
// where the 512-column tiles above touch 512 bytes per row and page) and a row
// range; each thread sums its 16 columns over the rows (no cross-warp reduction).
// Row splits of a tile form a cluster and are summed through DSMEM as above.
constexpr int kColsumWideCols = 4096;
#ifndef ABED_COLSUM_WIDE_U
#define ABED_COLSUM_WIDE_U 16  // rows (16-byte loads) in flight per thread
#endif
#ifndef ABED_COLSUM_WIDE_MINB
#define ABED_COLSUM_WIDE_MINB 4
#endif
__global__ void __launch_bounds__(256, ABED_COLSUM_WIDE_MINB) colsum_i8_wide_kernel(const int8_t* __restrict__ x, int64_t rows,
                                                                int64_t len, int64_t rows_per,
                                                                int32_t* __restrict__ out) {
  namespace cg = cooperative_groups;
  cg::cluster_group cluster = cg::this_cluster();
  __shared__ __align__(16) int32_t s_part[kColsumWideCols];
  const int cs = static_cast<int>(cluster.num_blocks());
  const int rank = static_cast<int>(cluster.block_rank());
  const int64_t cols16 = len >> 4;
  const int64_t tile = blockIdx.x / cs;
  const int64_t c16 = tile * 256 + threadIdx.x;
  const int64_t r0 = rank * rows_per, r1 = r0 + rows_per < rows ? r0 + rows_per : rows;
  int32_t acc[16];
#pragma unroll
  for (int j = 0; j < 16; ++j) acc[j] = 0;
  if (c16 < cols16 && r1 > r0) {
    const uint4* ptr = reinterpret_cast<const uint4*>(x) + c16 + r0 * cols16;
    const int64_t mine = r1 - r0;
    int64_t done = 0;
    while (done < mine) {
      uint32_t ev[4] = {0u, 0u, 0u, 0u}, od[4] = {0u, 0u, 0u, 0u};
      const int64_t batch_end = done + 256 < mine ? done + 256 : mine;  // 16-bit lanes: <= 256 rows per flush
      while (done < batch_end) {  // batches of U rows, every load issued before use
        constexpr int U = ABED_COLSUM_WIDE_U;
        const int rem = batch_end - done < U ? static_cast<int>(batch_end - done) : U;
        uint4 v[U];
#pragma unroll
        for (int u = 0; u < U; ++u)
          v[u] = u < rem ? __ldcs(ptr + u * cols16) : make_uint4(0x80808080u, 0x80808080u, 0x80808080u, 0x80808080u);
        ptr += rem * cols16;
        done += rem;
#pragma unroll
        for (int u = 0; u < U; ++u) {  // padding slots add (0x80 ^ 0x80) = 0
          const uint32_t w[4] = {v[u].x ^ 0x80808080u, v[u].y ^ 0x80808080u, v[u].z ^ 0x80808080u,
                                 v[u].w ^ 0x80808080u};
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            ev[q] += w[q] & 0x00FF00FFu;
            od[q] += (w[q] >> 8) & 0x00FF00FFu;
          }
        }
      }
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        acc[4 * q] += static_cast<int32_t>(ev[q] & 0xFFFFu);
        acc[4 * q + 1] += static_cast<int32_t>(od[q] & 0xFFFFu);
        acc[4 * q + 2] += static_cast<int32_t>(ev[q] >> 16);
        acc[4 * q + 3] += static_cast<int32_t>(od[q] >> 16);
      }
    }
#pragma unroll
    for (int j = 0; j < 16; ++j) acc[j] -= static_cast<int32_t>(128 * mine);
  }
  if (cs == 1) {
    if (c16 < cols16) {
      int4* o = reinterpret_cast<int4*>(out + c16 * 16);
#pragma unroll
      for (int j = 0; j < 4; ++j) o[j] = make_int4(acc[4 * j], acc[4 * j + 1], acc[4 * j + 2], acc[4 * j + 3]);
    }
    return;
  }
  int4* sp = reinterpret_cast<int4*>(s_part + threadIdx.x * 16);
#pragma unroll
  for (int j = 0; j < 4; ++j) sp[j] = make_int4(acc[4 * j], acc[4 * j + 1], acc[4 * j + 2], acc[4 * j + 3]);
  cluster.sync();
  const int per = (kColsumWideCols + cs - 1) / cs;
  for (int cl = rank * per + threadIdx.x; cl < (rank + 1) * per && cl < kColsumWideCols; cl += 256) {
    const int64_t col = tile * kColsumWideCols + cl;
    if (col >= len) continue;
    int32_t sum = 0;
    for (int q = 0; q < cs; ++q) sum += cluster.map_shared_rank(s_part, q)[cl];
    out[col] = sum;
  }
  cluster.sync();  // keep this CTA's partials alive until every peer has read them
}

// Tall variant for short rows (the filter checksum: 512 filters x 4608 bytes): a
// CTA owns 32 adjacent columns of EVERY row (128 row groups x two 16-byte
// vectors), so ~one CTA per SM covers the matrix with all its loads in flight at
// once and no row split, cluster or atomic: the rows are summed in registers
// (16-bit lanes), then across the 128 row groups in shared memory.
template <int NV>  // 16-byte vectors per row and CTA: 16 * NV columns, 256 / NV row groups
__global__ void __launch_bounds__(256) colsum_i8_tall_kernel(const int8_t* __restrict__ x, int64_t rows, int64_t len,
                                                             int32_t* __restrict__ out) {
  constexpr int RG = 256 / NV, CC = 16 * NV, SL = 256 / CC;
  __shared__ int32_t part[RG][CC + 1];
  __shared__ int32_t red2[SL][CC];
  const int64_t cols16 = len >> 4;
  const int vec = threadIdx.x % NV, g = threadIdx.x / NV;
  const int64_t c16 = (int64_t)blockIdx.x * NV + vec;
  int32_t acc[16];
#pragma unroll
  for (int j = 0; j < 16; ++j) acc[j] = 0;
  if (c16 < cols16 && g < rows) {
    const int64_t mine = (rows - g + RG - 1) / RG;  // rows g, g + RG, ...
    const uint4* ptr = reinterpret_cast<const uint4*>(x) + c16 + g * cols16;
    const int64_t step = RG * cols16;
    int64_t done = 0;
    while (done < mine) {
      uint32_t ev[4] = {0u, 0u, 0u, 0u}, od[4] = {0u, 0u, 0u, 0u};
      const int64_t batch_end = done + 256 < mine ? done + 256 : mine;  // 16-bit lanes: <= 256 rows per flush
      while (done < batch_end) {  // batches of 8 rows, every load issued before use
        const int rem = batch_end - done < 8 ? static_cast<int>(batch_end - done) : 8;
        uint4 v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u)
          v[u] = u < rem ? __ldcs(ptr + u * step) : make_uint4(0x80808080u, 0x80808080u, 0x80808080u, 0x80808080u);
        ptr += rem * step;
        done += rem;
#pragma unroll
        for (int u = 0; u < 8; ++u) {  // padding slots add (0x80 ^ 0x80) = 0
          const uint32_t w[4] = {v[u].x ^ 0x80808080u, v[u].y ^ 0x80808080u, v[u].z ^ 0x80808080u,
                                 v[u].w ^ 0x80808080u};
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            ev[q] += w[q] & 0x00FF00FFu;
            od[q] += (w[q] >> 8) & 0x00FF00FFu;
          }
        }
      }
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        acc[4 * q] += static_cast<int32_t>(ev[q] & 0xFFFFu);
        acc[4 * q + 1] += static_cast<int32_t>(od[q] & 0xFFFFu);
        acc[4 * q + 2] += static_cast<int32_t>(ev[q] >> 16);
        acc[4 * q + 3] += static_cast<int32_t>(od[q] >> 16);
      }
    }
#pragma unroll
    for (int j = 0; j < 16; ++j) acc[j] -= static_cast<int32_t>(128 * mine);
  }
#pragma unroll
  for (int j = 0; j < 16; ++j) part[g][vec * 16 + j] = acc[j];
  __syncthreads();
  const int c = threadIdx.x % CC, sl = threadIdx.x / CC;
  int32_t sum = 0;
#pragma unroll
  for (int i = 0; i < RG / SL; ++i) sum += part[sl * (RG / SL) + i][c];
  red2[sl][c] = sum;
  __syncthreads();
  if (threadIdx.x < CC) {
    int32_t tot = 0;
#pragma unroll
    for (int i = 0; i < SL; ++i) tot += red2[i][c];
    const int64_t col = (int64_t)blockIdx.x * CC + c;
    if (col < len) out[col] = tot;
  }
}

// any length / alignment: one column per thread, the same row split
__global__ void colsum_i8_kernel(const int8_t* __restrict__ x, int64_t rows, int64_t len, int64_t rows_per,
                                 int32_t* __restrict__ out) {
  const int64_t chunks = (rows + rows_per - 1) / rows_per;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < len * chunks;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t c = idx % len, chunk = idx / len;
    const int64_t r0 = chunk * rows_per, r1 = r0 + rows_per < rows ? r0 + rows_per : rows;
    int32_t acc = 0;
    for (int64_t r = r0; r < r1; ++r) acc += x[r * len + c];
    if (acc != 0) atomicAdd(out + c, acc);
  }
}

// gen_input_checksum (checksum.hpp:248-266) from the batch-summed image: one
// block per (c, r, s), lattice sum over every window position.
__global__ void input_checksum_kernel(const int32_t* __restrict__ bsum, abed_layer_shape s, int32_t* __restrict__ ic) {
  const int64_t crs = s.c * s.r * s.s;
  for (int64_t e = blockIdx.x; e < crs; e += gridDim.x) {
    const int64_t c = e / (s.r * s.s), r = (e / s.s) % s.r, ss = e % s.s;
    int32_t acc = 0;
    for (int64_t t = threadIdx.x; t < s.p * s.q; t += blockDim.x) {
      const int64_t p = t / s.q, q = t % s.q;
      const int64_t hi = p * s.stride_h - s.pad_h + r, wi = q * s.stride_w - s.pad_w + ss;
      if (hi >= 0 && hi < s.h && wi >= 0 && wi < s.w) acc += bsum[(c * s.h + hi) * s.w + wi];
    }
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    __shared__ int32_t red[32];
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
    __syncthreads();
    if (threadIdx.x == 0) {
      int32_t tot = 0;
      for (int w = 0; w < (int)(blockDim.x >> 5); ++w) tot += red[w];
      ic[e] = tot;
    }
    __syncthreads();
  }
}
__global__ void reduce_i64_kernel(const int32_t* __restrict__ c, int64_t n, unsigned long long* __restrict__ out,
                                  unsigned int* __restrict__ wrap32) {
  long long s = 0;
  uint32_t w = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    s += c[i];
    w += (uint32_t)c[i];
  }
  for (int o = 16; o > 0; o >>= 1) {
    s += __shfl_xor_sync(0xffffffffu, s, o);
    w += __shfl_xor_sync(0xffffffffu, w, o);
  }
  if ((threadIdx.x & 31) == 0) {
    atomicAdd(out, (unsigned long long)s);
    atomicAdd(wrap32, w);
  }
}
__global__ void dot_i64_kernel(const int32_t* __restrict__ a, const int32_t* __restrict__ b, int64_t n,
                               unsigned long long* __restrict__ out) {
  long long s = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    s += (long long)a[i] * b[i];
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if ((threadIdx.x & 31) == 0) atomicAdd(out, (unsigned long long)s);
}

// First-mismatch search: key = reference loop position; atomicMin gives the
// first locus, atomicAdd the mismatch count (both exact and deterministic).
struct Mism {
  unsigned long long first;
  unsigned long long count;
};
__global__ void fc_verify_kernel(const int32_t* __restrict__ cv, abed_dims4 d, const int64_t* __restrict__ ev,
                                 int64_t k_lim, Mism* m) {
  const int64_t pq = d.d2 * d.d3, rows = d.d0 * pq;  // checksum.hpp:224-234 order (n, j)
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < rows; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t n = t / pq, j = t % pq;
    long long sum = 0;
    for (int64_t k = 0; k < k_lim; ++k) sum += cv[(n * d.d1 + k) * pq + j];
    if (sum != ev[t]) {
      atomicMin(&m->first, (unsigned long long)t);
      atomicAdd(&m->count, 1ull);
    }
  }
}
__global__ void icb_verify_kernel(const int32_t* __restrict__ cv, abed_dims4 d, const int64_t* __restrict__ ev, Mism* m) {
  const int64_t kpq = d.d1 * d.d2 * d.d3;  // checksum.hpp:409-419 order (k,p,q)
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < kpq; i += (int64_t)gridDim.x * blockDim.x) {
    long long sum = 0;
    for (int64_t n = 0; n < d.d0; ++n) sum += cv[n * kpq + i];
    if (sum != ev[i]) {
      atomicMin(&m->first, (unsigned long long)i);
      atomicAdd(&m->count, 1ull);
    }
  }
}
// ic_verify_k: one block per k: out_sum over (n, j) and dot(f[k], ic)
__global__ void ick_sums_kernel(const int32_t* __restrict__ cv, abed_dims4 d, const int8_t* __restrict__ f, int64_t crs,
                                const int32_t* __restrict__ ic, long long* __restrict__ lhs, long long* __restrict__ rhs) {
  const int64_t k = blockIdx.x, pq = d.d2 * d.d3;
  long long s = 0, dot = 0;
  for (int64_t t = threadIdx.x; t < d.d0 * pq; t += blockDim.x) s += cv[((t / pq) * d.d1 + k) * pq + t % pq];
  for (int64_t i = threadIdx.x; i < crs; i += blockDim.x) dot += (long long)f[k * crs + i] * ic[i];
  for (int o = 16; o > 0; o >>= 1) {
    s += __shfl_xor_sync(0xffffffffu, s, o);
    dot += __shfl_xor_sync(0xffffffffu, dot, o);
  }
  __shared__ long long rs[32], rd[32];
  if ((threadIdx.x & 31) == 0) { rs[threadIdx.x >> 5] = s; rd[threadIdx.x >> 5] = dot; }
  __syncthreads();
  if (threadIdx.x == 0) {
    long long a = 0, b = 0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) { a += rs[w]; b += rd[w]; }
    lhs[k] = a;
    rhs[k] = b;
  }
}

// ------------------------------------------------------------- float mode
// Sequential reductions (single thread per output) keep the reference's order.
__global__ void filter_sum_f64_kernel(const float* __restrict__ f, abed_dims4 fd, double* __restrict__ out) {
  const int64_t crs = fd.d1 * fd.d2 * fd.d3;  // checksum.hpp:483-494
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < crs; i += (int64_t)gridDim.x * blockDim.x) {
    double s = 0.0;
    for (int64_t k = 0; k < fd.d0; ++k) s += (double)f[k * crs + i];
    out[i] = s;
  }
}
__global__ void input_sum_f64_kernel(const float* __restrict__ x, abed_layer_shape s, double* __restrict__ out) {
  const int64_t crs = s.c * s.r * s.s;  // checksum.hpp:496-522, additions in (n, p, q) order
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < crs; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t c = e / (s.r * s.s), r = (e / s.s) % s.r, ss = e % s.s;
    double acc = 0.0;
    for (int64_t n = 0; n < s.n; ++n)
      for (int64_t p = 0; p < s.p; ++p) {
        const int64_t hi = p * s.stride_h - s.pad_h + r;
        if (hi < 0 || hi >= s.h) continue;
        for (int64_t q = 0; q < s.q; ++q) {
          const int64_t wi = q * s.stride_w - s.pad_w + ss;
          if (wi < 0 || wi >= s.w) continue;
          acc += (double)x[((n * s.c + c) * s.h + hi) * s.w + wi];
        }
      }
    out[e] = acc;
  }
}
__global__ void seq_f64_kernel(const float* __restrict__ c, int64_t n, double* out) {
  if (blockIdx.x || threadIdx.x) return;  // checksum.hpp:524-528
  double s = 0.0;
  for (int64_t i = 0; i < n; ++i) s += (double)c[i];
  *out = s;
}
__global__ void dot_f64_kernel(const double* __restrict__ a, const double* __restrict__ b, int64_t n, double* out) {
  if (blockIdx.x || threadIdx.x) return;  // checksum.hpp:530-535 (acc += a*b -> fma)
  double s = 0.0;
  for (int64_t i = 0; i < n; ++i) s = fma(a[i], b[i], s);
  *out = s;
}
__global__ void fc_rows_f64_kernel(const float* __restrict__ cv, abed_dims4 d, const float* __restrict__ ev, double* lhs,
                                   double* rhs) {
  const int64_t pq = d.d2 * d.d3, rows = d.d0 * pq;  // checksum.hpp:551-556
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < rows; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t n = t / pq, j = t % pq;
    double s = 0.0;
    for (int64_t k = 0; k < d.d1; ++k) s += (double)cv[(n * d.d1 + k) * pq + j];
    lhs[t] = s;
    rhs[t] = (double)ev[t];
  }
}
__global__ void ick_f64_kernel(const float* __restrict__ cv, abed_dims4 d, const float* __restrict__ f, int64_t crs,
                               const double* __restrict__ ic, double* lhs, double* rhs) {
  const int64_t pq = d.d2 * d.d3;  // checksum.hpp:579-587, per k sequential
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < d.d1; k += (int64_t)gridDim.x * blockDim.x) {
    double s = 0.0, dot = 0.0;
    for (int64_t n = 0; n < d.d0; ++n)
      for (int64_t j = 0; j < pq; ++j) s += (double)cv[(n * d.d1 + k) * pq + j];
    for (int64_t i = 0; i < crs; ++i) dot = fma((double)f[k * crs + i], ic[i], dot);
    lhs[k] = s;
    rhs[k] = dot;
  }
}

__global__ void flip_kernel(uint8_t* data, int64_t byte, uint8_t mask) { data[byte] ^= mask; }

// ------------------------------------------------------------- helpers
template <typename T>
struct DevBuf {
  T* p = nullptr;
  explicit DevBuf(size_t n) { cuda_check(cudaMalloc(&p, (n ? n : 1) * sizeof(T)), "cudaMalloc(tmp)"); }
  ~DevBuf() { cudaFree(p); }
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
};
template <typename T>
T d2h(const T* d) {
  T h;
  cuda_check(cudaMemcpy(&h, d, sizeof(T), cudaMemcpyDeviceToHost), "d2h");
  return h;
}
void sync() { cuda_check(cudaDeviceSynchronize(), "synchronize"); }
void launched(const char* what) { cuda_check(cudaGetLastError(), what); }
int64_t count4(abed_dims4 d) { return d.d0 * d.d1 * d.d2 * d.d3; }
void check_dims(abed_dims4 d) {
  if (d.d0 < 1 || d.d1 < 1 || d.d2 < 1 || d.d3 < 1) throw_invalid("Tensor4D: all extents must be >= 1");
}
void set_fail(abed_verify_outcome* o, int64_t lhs, int64_t rhs, bool locus, int64_t l0, int64_t l1, int64_t l2,
              int64_t count) {
  std::memset(o, 0, sizeof(*o));
  o->status = 1;
  o->lhs = lhs;
  o->rhs = rhs;
  o->has_locus = locus ? 1 : 0;
  o->locus[0] = l0; o->locus[1] = l1; o->locus[2] = l2;
  o->error_count = count;
}
void set_ok(abed_verify_outcome* o) { std::memset(o, 0, sizeof(*o)); }
int ceil_log2_host(int64_t v) {
  int bits = 0;
  uint64_t u = (uint64_t)v - 1;
  while (u) { ++bits; u >>= 1; }
  return bits;
}
void float_verify_host(double lhs, double rhs, double tau, abed_verify_outcome* o) {
  if (!(tau >= 0.0)) throw_invalid("float_verify: tau must be >= 0");  // checksum.hpp:474-481
  std::memset(o, 0, sizeof(*o));
  o->lhs_f = lhs;
  o->rhs_f = rhs;
  if (!(std::fabs(lhs - rhs) <= tau)) { o->status = 1; o->error_count = 1; }
}

}  // namespace

namespace abed_host {
int set_error(int code, const std::string& msg);
template <typename Fn>
int guarded2(Fn&& fn) {
  try {
    fn();
    return ABED_OK;
  } catch (const AbedError& e) {
    return set_error(e.code, e.what());
  } catch (const std::exception& e) {
    return set_error(ABED_ERR_RUNTIME, e.what());
  }
}
// exported to campaign.cu / abi_core.cu
void dev_colsum_i8(const int8_t* x, int64_t rows, int64_t len, int32_t* out, cudaStream_t st) {
  const bool v16 = (len % 16 == 0) && (reinterpret_cast<uintptr_t>(x) % 16 == 0);
  if (v16) {
    const int64_t wide_tiles = (len + kColsumWideCols - 1) / kColsumWideCols;
    // tuning / tests: 1 wide, 2 not wide, 3 tall, 4 cluster (2 and 4: the 512-column tiles)
    const char* force_s = getenv("ABED_COLSUM_KERNEL");
    const int force = force_s ? atoi(force_s) : 0;
    if (force == 1 || (force == 0 && wide_tiles * 16 >= num_sms())) {
      // row splits: a power-of-two cluster <= 8 (measured on the 256 x 200704 batch
      // checksum: cs 8 13.3 us, 4 15.4, 16 17.9, 12 20.5), one wave of <= 4 CTAs
      // per SM, >= 8 rows per split
      int64_t cs = 8;
      while (cs > 1 && (wide_tiles * cs > (int64_t)num_sms() * ABED_COLSUM_WIDE_MINB || (rows + cs - 1) / cs < 8))
        cs >>= 1;
      const char* cs_s = getenv("ABED_COLSUM_CS");  // tuning experiments
      if (cs_s && atoi(cs_s) > 0) cs = atoi(cs_s);
      if (cs < 1) cs = 1;
      const int64_t rows_per = (rows + cs - 1) / cs;
      static bool wattr[64] = {};
      int dev = 0;
      cudaGetDevice(&dev);
      if (dev < 0 || dev >= 64 || !wattr[dev]) {
        cuda_check(cudaFuncSetAttribute(colsum_i8_wide_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1),
                   "colsum cluster attr");
        if (dev >= 0 && dev < 64) wattr[dev] = true;
      }
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3((unsigned)(wide_tiles * cs));
      cfg.blockDim = dim3(256);
      cfg.stream = st;
      cudaLaunchAttribute la[1];
      la[0].id = cudaLaunchAttributeClusterDimension;
      la[0].val.clusterDim.x = (unsigned)cs;
      la[0].val.clusterDim.y = 1;
      la[0].val.clusterDim.z = 1;
      cfg.attrs = la;
      cfg.numAttrs = 1;
      cuda_check(cudaLaunchKernelEx(&cfg, colsum_i8_wide_kernel, x, rows, len, rows_per, out), "colsum launch");
      launched("colsum_i8");
      return;
    }
    // short rows: 32-column CTAs over all rows when they fill the SMs without
    // more than ~4 CTAs per SM
    const int64_t tall_tiles = (len / 16 + 1) / 2;
    if (force != 4 && (force == 3 || (tall_tiles <= (int64_t)num_sms() * 4 && tall_tiles * 2 >= num_sms() && rows >= 64))) {
      // 16-byte vectors per row and CTA (tuning: 1, 2, 4, 8 measured 4.1 / 4.1 / 5.1 / 7.7 us on K6)
      const char* nv_s = getenv("ABED_COLSUM_TALL_NV");
      const int nv = nv_s ? atoi(nv_s) : 2;
      const int64_t c16n = len / 16;
      if (nv == 8)
        colsum_i8_tall_kernel<8><<<(unsigned)((c16n + 7) / 8), 256, 0, st>>>(x, rows, len, out);
      else if (nv == 4)
        colsum_i8_tall_kernel<4><<<(unsigned)((c16n + 3) / 4), 256, 0, st>>>(x, rows, len, out);
      else if (nv == 1)
        colsum_i8_tall_kernel<1><<<(unsigned)c16n, 256, 0, st>>>(x, rows, len, out);
      else
        colsum_i8_tall_kernel<2><<<(unsigned)((c16n + 1) / 2), 256, 0, st>>>(x, rows, len, out);
      launched("colsum_i8");
      return;
    }
    // row splits of a 512-column tile = one cluster (<= 16 CTAs, DSMEM reduction):
    // about 8 resident CTAs per SM in one wave, at least one row per warp
    const int64_t col_tiles = (len / 16 + 31) / 32;
    // clusters only when the column tiles alone leave SMs idle (their co-scheduling
    // and DSMEM hand-off cost more than they save once every SM has a tile:
    // measured 26.7 -> 18.5 us on the 256 x 200704 batch checksum)
    int64_t cs = col_tiles >= num_sms() ? 1 : ((int64_t)num_sms() * 8) / col_tiles;
    const int64_t max_cs = (rows + kColsumWarps - 1) / kColsumWarps;
    if (cs > max_cs) cs = max_cs;
    static const int cs_cap = [] {
      const char* e = getenv("ABED_COLSUM_MAX_CLUSTER");  // tuning experiments
      const int v = e ? atoi(e) : 16;
      return v >= 1 && v <= 16 ? v : 16;
    }();
    if (cs > cs_cap) cs = cs_cap;
    if (cs < 1) cs = 1;
    const int64_t rows_per = (rows + cs - 1) / cs;
    static bool attr[64] = {};
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 0 || dev >= 64 || !attr[dev]) {
      cuda_check(cudaFuncSetAttribute(colsum_i8_cluster_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1),
                 "colsum cluster attr");
      if (dev >= 0 && dev < 64) attr[dev] = true;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)(col_tiles * cs));
    cfg.blockDim = dim3(kColsumWarps * 32);
    cfg.stream = st;
    cudaLaunchAttribute la[1];
    la[0].id = cudaLaunchAttributeClusterDimension;
    la[0].val.clusterDim.x = (unsigned)cs;
    la[0].val.clusterDim.y = 1;
    la[0].val.clusterDim.z = 1;
    cfg.attrs = la;
    cfg.numAttrs = 1;
    cuda_check(cudaLaunchKernelEx(&cfg, colsum_i8_cluster_kernel, x, rows, len, rows_per, out), "colsum launch");
  } else {
    cuda_check(cudaMemsetAsync(out, 0, (size_t)len * 4, st), "colsum memset");
    const int64_t want = (int64_t)num_sms() * 4 * 256;
    int64_t rows_per = (rows * len + want - 1) / want;
    if (rows_per < 16) rows_per = 16;
    if (rows_per > rows) rows_per = rows;
    const int64_t work = len * ((rows + rows_per - 1) / rows_per);
    colsum_i8_kernel<<<grid_for(work, 256), 256, 0, st>>>(x, rows, len, rows_per, out);
  }
  launched("colsum_i8");
}
void dev_gen_input_checksum(const int8_t* x, const abed_layer_shape& s, int32_t* sums, cudaStream_t st) {
  if (8 + ceil_log2_host(s.n * s.p * s.q) > 32)
    throw_invalid("gen_input_checksum: PQN too large for i32 checksums; a wider plan is required");
  DevBuf<int32_t> b((size_t)(s.c * s.h * s.w));
  dev_colsum_i8(x, s.n, s.c * s.h * s.w, b.p, st);
  input_checksum_kernel<<<(int)std::min<int64_t>(s.c * s.r * s.s, 65535), 256, 0, st>>>(b.p, s, sums);
  launched("gen_input_checksum");
  cuda_check(cudaStreamSynchronize(st), "gen_input_checksum sync");
}
void dev_epilog(const int32_t* in, abed_dims4 d, const abed_epilog_params* p, void* out, cudaStream_t st) {
  check_dims(d);
  if (p->bias_len != d.d1) throw_invalid("epilog: bias length must equal the channel count");
  if (!std::isfinite(p->scale)) throw_invalid("epilog: non-finite scale");
  if (p->bias_len > 0) {
    std::vector<float> hb((size_t)p->bias_len);
    cuda_check(cudaMemcpy(hb.data(), p->bias, hb.size() * 4, cudaMemcpyDeviceToHost), "bias d2h");
    for (float b : hb)
      if (!std::isfinite(b)) throw_invalid("epilog: non-finite bias");
  }
  if (p->output_kind != ABED_I8 && p->output_kind != ABED_F32) throw_invalid("epilog: output kind must be i8 or f32");
  const bool v16 = (d.d2 * d.d3) % 16 == 0 && reinterpret_cast<uintptr_t>(in) % 16 == 0 &&
                   reinterpret_cast<uintptr_t>(out) % 16 == 0;
  if (v16)
    epilog_v16_kernel<<<grid_for(count4(d) / 16, 256), 256, 0, st>>>(in, d, p->scale, p->bias,
                                                                     p->activation == ABED_RELU,
                                                                     p->output_kind == ABED_F32, out);
  else
    epilog_kernel<<<grid_for(count4(d), 256), 256, 0, st>>>(in, d, p->scale, p->bias, p->activation == ABED_RELU,
                                                             p->output_kind == ABED_F32, out);
  launched("epilog");
}
}  // namespace abed_host

#define GUARD(...) return guarded2([&] { require_device(); __VA_ARGS__; })

extern "C" {

uint64_t abed_derive_seed(uint64_t root, uint64_t index) {  // rng.hpp:41-44
  return mix64((root ^ (0xA02E9D4BD1C96D4FULL + index * kGolden)) + kGolden);
}
int abed_fill_random_i8(int8_t* t, int64_t n, uint64_t seed, uint64_t off, void* stream) {
  GUARD(fill_i8_kernel<<<grid_for(n, 256), 256, 0, (cudaStream_t)stream>>>(t, n, seed, off, 0); launched("fill_random_i8"));
}
int abed_fill_random_extreme(int8_t* t, int64_t n, uint64_t seed, uint64_t off, void* stream) {
  GUARD(fill_i8_kernel<<<grid_for(n, 256), 256, 0, (cudaStream_t)stream>>>(t, n, seed, off, 1); launched("fill_random_extreme"));
}

int abed_conv_f32(const float* x, const float* f, const abed_layer_shape* s, float* out, void* stream) {
  GUARD(validate_shape(*s);
        conv_direct_kernel<float, float, float><<<grid_for(s->n * s->k * s->p * s->q, 128), 128, 0, (cudaStream_t)stream>>>(x, f, *s, out);
        launched("conv_f32"); cuda_check(cudaStreamSynchronize((cudaStream_t)stream), "conv_f32"));
}
int abed_epilog(const int32_t* convout, abed_dims4 d, const abed_epilog_params* p, void* out, void* stream) {
  GUARD(dev_epilog(convout, d, p, out, (cudaStream_t)stream));
}
int abed_gen_filter_checksum(const int8_t* f, abed_dims4 fd, int32_t* sums, void* stream) {
  GUARD(check_dims(fd);
        if (fd.d0 > (int64_t(1) << 24)) throw_invalid("gen_filter_checksum: K too large for i32 checksums");
        const int64_t crs = fd.d1 * fd.d2 * fd.d3;
        dev_colsum_i8(f, fd.d0, crs, sums, (cudaStream_t)stream));
}
int abed_decompose_checksum_filters(const int32_t* sums, int64_t n, int8_t* planes, void* stream) {
  GUARD(decompose_kernel<<<grid_for(n, 256), 256, 0, (cudaStream_t)stream>>>(sums, n, planes); launched("decompose"));
}
int abed_conv_checksum_planes(const int8_t* x, const abed_layer_shape* s, const int8_t* planes, int32_t* extra, void* stream) {
  GUARD(validate_shape(*s);
        if (s->c * s->r * s->s > 65536) throw_invalid("conv_checksum_planes: CRS > 65536 exceeds the i32 plan");
        planes_conv_kernel<<<grid_for(s->n * s->p * s->q, 128), 128, 0, (cudaStream_t)stream>>>(x, *s, planes, extra);
        launched("conv_checksum_planes"));
}
int abed_recombine_extra_fmaps(const int32_t* e, int64_t n, int64_t* out, void* stream) {
  GUARD(recombine_kernel<<<grid_for(n, 256), 256, 0, (cudaStream_t)stream>>>(e, n, out); launched("recombine"));
}
int abed_conv_filter_checksum(const int8_t* x, const abed_layer_shape* s, const int32_t* sums, int64_t* out, void* stream) {
  GUARD(validate_shape(*s); abed_layer_shape one = *s; one.k = 1;
        conv_direct_kernel<int8_t, int32_t, int64_t><<<grid_for(s->n * s->p * s->q, 128), 128, 0, (cudaStream_t)stream>>>(x, sums, one, out);
        launched("conv_filter_checksum"));
}
int abed_fc_verify(const int32_t* cv, abed_dims4 d, const int64_t* extra, int64_t original_k, abed_verify_outcome* o) {
  GUARD(check_dims(d);
        const int64_t k_lim = original_k < 0 ? d.d1 : original_k;
        if (k_lim < 1 || k_lim > d.d1) throw_invalid("fc_verify: bad original_k");
        DevBuf<Mism> m(1); const Mism init{~0ull, 0ull};
        cuda_check(cudaMemcpy(m.p, &init, sizeof(init), cudaMemcpyHostToDevice), "h2d");
        fc_verify_kernel<<<grid_for(d.d0 * d.d2 * d.d3, 256), 256>>>(cv, d, extra, k_lim, m.p); launched("fc_verify");
        const Mism r = d2h(m.p);
        if (r.count == 0) { set_ok(o); return; }
        const int64_t t = (int64_t)r.first, pq = d.d2 * d.d3, n = t / pq, j = t % pq;
        // lhs/rhs at the first mismatch, recomputed exactly on the host from two small reads
        std::vector<int32_t> col((size_t)k_lim);
        for (int64_t k = 0; k < k_lim; ++k)
          cuda_check(cudaMemcpy(&col[(size_t)k], cv + (n * d.d1 + k) * pq + j, 4, cudaMemcpyDeviceToHost), "d2h");
        int64_t lhs = 0; for (int32_t v : col) lhs += v;
        const int64_t rhs = d2h(extra + t);
        set_fail(o, lhs, rhs, true, n, j / d.d3, j % d.d3, (int64_t)r.count));
}
int abed_gen_input_checksum(const int8_t* x, const abed_layer_shape* s, int32_t* sums, void* stream) {
  GUARD(validate_shape(*s); dev_gen_input_checksum(x, *s, sums, (cudaStream_t)stream));
}
int abed_reduce_all_i64(const int32_t* c, int64_t n, int64_t* result) {
  GUARD(DevBuf<unsigned long long> acc(2); cuda_check(cudaMemset(acc.p, 0, 16), "memset");
        reduce_i64_kernel<<<grid_for(n, 256), 256>>>(c, n, acc.p, reinterpret_cast<unsigned int*>(acc.p + 1));
        launched("reduce_all_i64"); *result = (int64_t)d2h(acc.p));
}
int abed_reduce_all_wrap32(const int32_t* c, int64_t n, int32_t* result) {
  GUARD(DevBuf<unsigned long long> acc(2); cuda_check(cudaMemset(acc.p, 0, 16), "memset");
        reduce_i64_kernel<<<grid_for(n, 256), 256>>>(c, n, acc.p, reinterpret_cast<unsigned int*>(acc.p + 1));
        launched("reduce_all_wrap32"); *result = (int32_t)d2h(reinterpret_cast<unsigned int*>(acc.p + 1)));
}
int abed_fic_dot(const int32_t* fc, const int32_t* ic, int64_t n, int64_t* result) {
  GUARD(DevBuf<unsigned long long> acc(1); cuda_check(cudaMemset(acc.p, 0, 8), "memset");
        dot_i64_kernel<<<grid_for(n, 256), 256>>>(fc, ic, n, acc.p); launched("fic_dot");
        *result = (int64_t)d2h(acc.p));
}
static void fic_common(const int32_t* c, int64_t n, int64_t expected, abed_verify_outcome* o, bool forced32) {
  DevBuf<unsigned long long> acc(2);
  cuda_check(cudaMemset(acc.p, 0, 16), "memset");
  reduce_i64_kernel<<<grid_for(n, 256), 256>>>(c, n, acc.p, reinterpret_cast<unsigned int*>(acc.p + 1));
  launched("fic_verify");
  const int64_t sum = forced32 ? (int64_t)(int32_t)d2h(reinterpret_cast<unsigned int*>(acc.p + 1)) : (int64_t)d2h(acc.p);
  if (sum != expected) {
    set_fail(o, sum, expected, false, 0, 0, 0, 1);
  } else {
    set_ok(o);  // checksum.hpp:290-293: Pass reports lhs = rhs = sum
    o->lhs = sum;
    o->rhs = expected;
  }
}
int abed_fic_verify(const int32_t* c, int64_t n, int64_t expected, abed_verify_outcome* o) {
  GUARD(fic_common(c, n, expected, o, false));
}
int abed_fic_verify_forced32(const int32_t* c, int64_t n, int64_t expected, abed_verify_outcome* o) {
  GUARD(fic_common(c, n, expected, o, true));
}
int abed_ic_verify_k(const int32_t* cv, abed_dims4 d, const int8_t* f, abed_dims4 fd, const int32_t* ic, abed_verify_outcome* o) {
  GUARD(check_dims(d); check_dims(fd);
        if (fd.d0 != d.d1) throw_invalid("ic_verify_k: filter count does not match convout");
        const int64_t crs = fd.d1 * fd.d2 * fd.d3;
        DevBuf<long long> lhs((size_t)d.d1), rhs((size_t)d.d1);
        ick_sums_kernel<<<(unsigned)d.d1, 256>>>(cv, d, f, crs, ic, lhs.p, rhs.p); launched("ic_verify_k");
        std::vector<long long> hl((size_t)d.d1), hr((size_t)d.d1);
        cuda_check(cudaMemcpy(hl.data(), lhs.p, hl.size() * 8, cudaMemcpyDeviceToHost), "d2h");
        cuda_check(cudaMemcpy(hr.data(), rhs.p, hr.size() * 8, cudaMemcpyDeviceToHost), "d2h");
        int64_t first = -1, cnt = 0;
        for (int64_t k = 0; k < d.d1; ++k) if (hl[(size_t)k] != hr[(size_t)k]) { if (first < 0) first = k; ++cnt; }
        if (first < 0) set_ok(o); else set_fail(o, hl[(size_t)first], hr[(size_t)first], true, first, -1, -1, cnt));
}
int abed_ic_batch_checksum(const int8_t* x, abed_dims4 d, int32_t* out, void* stream) {
  GUARD(check_dims(d);
        dev_colsum_i8(x, d.d0, d.d1 * d.d2 * d.d3, out, (cudaStream_t)stream));
}
int abed_ic_batch_verify(const int32_t* cv, abed_dims4 d, const int64_t* extra, abed_verify_outcome* o) {
  GUARD(check_dims(d);
        DevBuf<Mism> m(1); const Mism init{~0ull, 0ull};
        cuda_check(cudaMemcpy(m.p, &init, sizeof(init), cudaMemcpyHostToDevice), "h2d");
        icb_verify_kernel<<<grid_for(d.d1 * d.d2 * d.d3, 256), 256>>>(cv, d, extra, m.p); launched("ic_batch_verify");
        const Mism r = d2h(m.p);
        if (r.count == 0) { set_ok(o); return; }
        const int64_t i = (int64_t)r.first, kpq = d.d1 * d.d2 * d.d3, pq = d.d2 * d.d3;
        int64_t lhs = 0;
        for (int64_t n = 0; n < d.d0; ++n) lhs += d2h(cv + n * kpq + i);
        set_fail(o, lhs, d2h(extra + i), true, i / pq, (i % pq) / d.d3, i % d.d3, (int64_t)r.count));
}
int abed_plan_precision(const abed_layer_shape* s, int32_t b, abed_precision_plan* p) {
  return guarded2([&] {  // checksum.hpp:451-468 (host arithmetic only)
    if (b != 4 && b != 8) throw_invalid("plan_precision: operand width must be 4 or 8 bits");
    const int64_t crs = s->c * s->r * s->s, npq = s->n * s->p * s->q;
    auto kind = [](int bits) {
      if (bits <= 32) return (int32_t)ABED_I32;
      if (bits <= 64) return (int32_t)ABED_I64;
      throw_invalid("plan_precision: requirement exceeds 64 bits");
    };
    std::memset(p, 0, sizeof(*p));
    p->operand_bits = b;
    p->bits_output_fmap = 2 * b + ceil_log2_host(crs);
    p->bits_reduced_fc = 2 * b + ceil_log2_host(crs * s->k);
    p->bits_reduced_fic = 2 * b + ceil_log2_host(npq * s->k * crs);
    p->bits_filter_checksum = b + ceil_log2_host(s->k);
    p->bits_input_checksum = b + ceil_log2_host(npq);
    p->output_fmap_kind = kind(p->bits_output_fmap);
    p->reduced_fc_kind = kind(p->bits_reduced_fc);
    p->reduced_fic_kind = kind(p->bits_reduced_fic);
    p->filter_checksum_kind = kind(p->bits_filter_checksum);
    p->input_checksum_kind = kind(p->bits_input_checksum);
  });
}

// ------------------------------------------------------------- float mode
int abed_float_verify(double lhs, double rhs, double tau, abed_verify_outcome* o) {
  return guarded2([&] { float_verify_host(lhs, rhs, tau, o); });
}
int abed_filter_checksum_f64(const float* f, abed_dims4 fd, double* sums, void* stream) {
  GUARD(check_dims(fd);
        filter_sum_f64_kernel<<<grid_for(fd.d1 * fd.d2 * fd.d3, 128), 128, 0, (cudaStream_t)stream>>>(f, fd, sums);
        launched("filter_checksum_f64"));
}
int abed_input_checksum_f64(const float* x, const abed_layer_shape* s, double* sums, void* stream) {
  GUARD(validate_shape(*s);
        input_sum_f64_kernel<<<grid_for(s->c * s->r * s->s, 64), 64, 0, (cudaStream_t)stream>>>(x, *s, sums);
        launched("input_checksum_f64"));
}
int abed_reduce_all_f64(const float* c, int64_t n, double* result) {
  GUARD(DevBuf<double> r(1); seq_f64_kernel<<<1, 1>>>(c, n, r.p); launched("reduce_all_f64"); *result = d2h(r.p));
}
int abed_fic_dot_f64(const double* a, const double* b, int64_t n, double* result) {
  GUARD(DevBuf<double> r(1); dot_f64_kernel<<<1, 1>>>(a, b, n, r.p); launched("fic_dot_f64"); *result = d2h(r.p));
}
int abed_fic_verify_f32(const float* c, int64_t n, double expected, double tau, abed_verify_outcome* o) {
  GUARD(DevBuf<double> r(1); seq_f64_kernel<<<1, 1>>>(c, n, r.p); launched("fic_verify_f32");
        float_verify_host(d2h(r.p), expected, tau, o));
}
int abed_fc_verify_f32(const float* cv, abed_dims4 d, const float* extra, double tau, abed_verify_outcome* o) {
  GUARD(check_dims(d);
        const int64_t rows = d.d0 * d.d2 * d.d3;
        DevBuf<double> l((size_t)rows), r((size_t)rows);
        fc_rows_f64_kernel<<<grid_for(rows, 256), 256>>>(cv, d, extra, l.p, r.p); launched("fc_verify_f32");
        std::vector<double> hl((size_t)rows), hr((size_t)rows);
        cuda_check(cudaMemcpy(hl.data(), l.p, (size_t)rows * 8, cudaMemcpyDeviceToHost), "d2h");
        cuda_check(cudaMemcpy(hr.data(), r.p, (size_t)rows * 8, cudaMemcpyDeviceToHost), "d2h");
        const int64_t pq = d.d2 * d.d3;
        for (int64_t t = 0; t < rows; ++t)
          if (!(std::fabs(hl[(size_t)t] - hr[(size_t)t]) <= tau)) {
            float_verify_host(hl[(size_t)t], hr[(size_t)t], tau, o);
            o->has_locus = 1; o->locus[0] = t / pq; o->locus[1] = (t % pq) / d.d3; o->locus[2] = t % d.d3;
            return;
          }
        set_ok(o));
}
int abed_ic_verify_k_f32(const float* cv, abed_dims4 d, const float* f, abed_dims4 fd, const double* ic, double tau,
                         abed_verify_outcome* o) {
  GUARD(check_dims(d); check_dims(fd);
        DevBuf<double> l((size_t)d.d1), r((size_t)d.d1);
        ick_f64_kernel<<<grid_for(d.d1, 32), 32>>>(cv, d, f, fd.d1 * fd.d2 * fd.d3, ic, l.p, r.p); launched("ic_verify_k_f32");
        std::vector<double> hl((size_t)d.d1), hr((size_t)d.d1);
        cuda_check(cudaMemcpy(hl.data(), l.p, hl.size() * 8, cudaMemcpyDeviceToHost), "d2h");
        cuda_check(cudaMemcpy(hr.data(), r.p, hr.size() * 8, cudaMemcpyDeviceToHost), "d2h");
        for (int64_t k = 0; k < d.d1; ++k)
          if (!(std::fabs(hl[(size_t)k] - hr[(size_t)k]) <= tau)) {
            float_verify_host(hl[(size_t)k], hr[(size_t)k], tau, o);
            o->has_locus = 1; o->locus[0] = k; o->locus[1] = -1; o->locus[2] = -1;
            return;
          }
        set_ok(o));
}

// --------------------------------------------------------------- faults
int abed_flip_bit(void* data, int32_t kind, int64_t count, int64_t flat_index, int32_t bit, void* stream) {
  GUARD(  // faults.hpp:53-62
      const int64_t es = kind == ABED_I8 ? 1 : kind == ABED_I64 ? 8 : 4;
      if (flat_index < 0 || flat_index >= count) throw_range("flip_bit: flat index out of bounds");
      if (bit < 0 || bit >= 8 * es) throw_range("flip_bit: bit position out of range for element kind");
      flip_kernel<<<1, 1, 0, (cudaStream_t)stream>>>(static_cast<uint8_t*>(data), flat_index * es + bit / 8,
                                                     (uint8_t)(1u << (bit % 8)));
      launched("flip_bit"));
}

}  // extern "C"
