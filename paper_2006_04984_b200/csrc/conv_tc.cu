// tcgen05 implicit-GEMM INT8 convolution with fused ABED checks and epilog.
//
// Replaces, on the device, the reference's int8 convolution
// (convolution.hpp:224 detail::conv_fast_i8 == :237 conv_direct) and, when a
// check is requested, the FC extra-fmap convolution + fc_verify
// (checksum.hpp:134-236), the FIC output reduction (:268, :287) and the IC
// per-channel reduction (:319-347), all inside the accumulator epilogue, before
// the fused scale/bias/ReLU/requantise (convolution.hpp:353-387).
//
// CTA = 10 warps, one CTA per SM, persistent over (M tile, N tile) work units:
//   warp 0      producer: one thread issues 1-D bulk copies (cp.async.bulk) of
//               the activation strips (and B blocks unless B is resident)
//   warp 1      TMEM allocator + single-thread tcgen05.mma issuer
//   warps 2..9  epilogue: tcgen05.ld (thread = GEMM row = output pixel), two
//               warps per TMEM lane quarter splitting the 16-column chunks;
//               checks, epilog, stores; double-buffered TMEM accumulators.
#include <cuda_runtime.h>

#include <cstdint>

#include "conv_tc.cuh"
#include "ptx.cuh"

namespace abed_dev {

constexpr int kEpiWarps = 8;
constexpr int kEpiThreads = kEpiWarps * 32;
constexpr int kConvThreads = 64 + kEpiThreads;
constexpr int kBiasSmem = 2048;

// compile-time output flavours
enum EpiKind : int { EPI_NONE = 0, EPI_NCHW = 1, EPI_PACKED = 2, EPI_COMPARE = 3 };

struct SmemLayout {
  uint32_t a_off, a_stage_bytes, b_off, bar_off, tab_off, total;
};

__host__ __device__ inline SmemLayout smem_layout(const ConvTcParams& p) {
  SmemLayout L;
  L.a_stage_bytes = static_cast<uint32_t>(p.n_phase) * p.gps * p.strip_pix * 16u;
  L.a_off = 0;
  uint32_t off = L.a_stage_bytes * p.n_stages;
  off = (off + 127u) & ~127u;
  L.b_off = off;
  off += p.b_resident ? p.b_stage_bytes * p.k_stages : p.b_stage_bytes * p.n_stages;
  off = (off + 127u) & ~127u;
  L.bar_off = off;
  off += 8 * (2 * kStages + 5) + 16;
  L.tab_off = off;  // per-stage MMA operand offset table (uint2 per MMA)
  off += 8u * p.ntaps * (p.gps / 2);
  L.total = off;
  return L;
}

__device__ __forceinline__ void decode_tile(const ConvTcParams& p, int tile_seq, int& mt, int& nt) {
  // b_resident with several N tiles: each CTA owns one N tile (blockIdx % n_tiles)
  if (p.b_resident) {
    nt = blockIdx.x % p.n_tiles;
    mt = blockIdx.x / p.n_tiles + tile_seq * (gridDim.x / p.n_tiles);
  } else {
    const int t = blockIdx.x + tile_seq * gridDim.x;
    mt = t / p.n_tiles;
    nt = t % p.n_tiles;
  }
}

// convolution.hpp:374-381 under the reference's -march=native build: the
// multiply-add contracts to one fused FMA, then ReLU, clamp, truncate.
__device__ __forceinline__ int32_t requant_i8(int32_t acc, float scale, float bias, int relu) {
  float v = __fmaf_rn(static_cast<float>(acc), scale, bias);
  if (relu) {
    // v < 0 -> 0 (reference keeps -0.0, which truncates to 0 as well)
    v = fminf(fmaxf(v, 0.0f), 127.0f);
    // 2^23 + v rounded toward zero puts trunc(v) in the low mantissa bits
    return static_cast<int32_t>(__float_as_uint(__fadd_rz(v, 8388608.0f)) & 0xFFu);
  }
  v = fminf(127.0f, fmaxf(-128.0f, v));
  return __float2int_rz(v);
}

__device__ __forceinline__ uint32_t pack4(int32_t a, int32_t b, int32_t c, int32_t d) {
  const uint32_t lo = __byte_perm(static_cast<uint32_t>(a), static_cast<uint32_t>(b), 0x0040u);
  const uint32_t hi = __byte_perm(static_cast<uint32_t>(c), static_cast<uint32_t>(d), 0x0040u);
  return __byte_perm(lo, hi, 0x5410u);
}

__device__ __forceinline__ void epi_bar() { asm volatile("bar.sync 1, %0;" ::"n"(kEpiThreads) : "memory"); }

template <int EPI, bool FC, bool FIC>
__global__ void __launch_bounds__(kConvThreads, 1) conv_i8_tc_kernel(const __grid_constant__ ConvTcParams p) {
  extern __shared__ __align__(128) uint8_t smem[];
  const SmemLayout L = smem_layout(p);
  uint8_t* sA = smem + L.a_off;
  uint8_t* sB = smem + L.b_off;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L.bar_off);
  uint64_t* full = bars;
  uint64_t* empty = bars + kStages;
  uint64_t* tfull = bars + 2 * kStages;
  uint64_t* tempty = bars + 2 * kStages + 2;
  uint64_t* bres = bars + 2 * kStages + 4;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * kStages + 5);
  __shared__ float s_bias[kBiasSmem];
  __shared__ int64_t s_red[kEpiWarps][4];
  __shared__ int64_t s_rowsum[kBlockM];

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  int64_t* const trace = p.trace ? p.trace + static_cast<int64_t>(blockIdx.x) * kTraceSlots : nullptr;
  const long long t_entry = clock64();
  if (trace && threadIdx.x == 0) {
    uint64_t gt;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(gt));
    trace[0] = static_cast<int64_t>(gt);
    trace[1] = t_entry;
  }

  // accumulator stages: columns per stage (multiple of 32), 2 stages when they fit
  const int acc_cols = (p.block_n_tot + 31) & ~31;
  const int n_acc = (2 * acc_cols <= 512) ? 2 : 1;
  uint32_t tmem_cols = 32;
  while (tmem_cols < static_cast<uint32_t>(n_acc * acc_cols)) tmem_cols <<= 1;

  if (threadIdx.x == 0) {
    for (int i = 0; i < kStages; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&tfull[i], 1);
      mbar_init(&tempty[i], kEpiWarps);
    }
    mbar_init(bres, 1);
    fence_mbar_init();
  }
  if (EPI != EPI_NONE && p.K <= kBiasSmem) {
    for (int i = threadIdx.x; i < p.K; i += blockDim.x) s_bias[i] = p.bias[i];
  }
  if (warp == 1) tmem_alloc(tmem_slot, tmem_cols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  if (trace && threadIdx.x == 0) trace[2] = clock64() - t_entry;

  // number of work units for this CTA
  int n_units;
  if (p.b_resident) {
    const int per = gridDim.x / p.n_tiles;
    const int mt0 = blockIdx.x / p.n_tiles;
    n_units = (static_cast<int>(blockIdx.x) < per * p.n_tiles && mt0 < p.m_tiles) ? (p.m_tiles - mt0 + per - 1) / per : 0;
  } else {
    const int total = p.m_tiles * p.n_tiles;
    n_units = static_cast<int>(blockIdx.x) < total ? (total - blockIdx.x + gridDim.x - 1) / gridDim.x : 0;
  }

  if (warp == 0) {
    // ------------------------------------------------------------ producer
    // warp-uniform loop; one elected lane issues each copy (ptx.cuh *_w)
    if (n_units > 0) {
      const uint64_t pol_b = policy_evict_last();
      if (p.b_resident) {
        const int nt = blockIdx.x % p.n_tiles;
        const uint32_t bytes = p.b_stage_bytes * p.k_stages;
        mbar_arrive_expect_tx_w(bres, bytes);
        const int8_t* src = p.wpk + static_cast<int64_t>(nt) * p.k_stages * p.b_stage_bytes;
        for (uint32_t o = 0; o < bytes; o += 65536u) {
          const uint32_t sz = (bytes - o) < 65536u ? (bytes - o) : 65536u;
          bulk_g2s_evict_last_w(sB + o, src + o, sz, bres, pol_b);
        }
      }
      int stage = 0;
      uint32_t phase = 0;
      const uint32_t strip_bytes = p.strip_pix * 16u;
      const uint32_t bytes = L.a_stage_bytes + (p.b_resident ? 0u : p.b_stage_bytes);
      if (trace && lane == 0) trace[8] = clock64() - t_entry;
      for (int u = 0; u < n_units; ++u) {
        int mt, nt;
        decode_tile(p, u, mt, nt);
        const int64_t m0 = static_cast<int64_t>(mt) * kBlockM;
        for (int ks = 0; ks < p.k_stages; ++ks) {
          mbar_wait(&empty[stage], phase ^ 1u);
          mbar_arrive_expect_tx_w(&full[stage], bytes);
          uint8_t* dstA = sA + stage * L.a_stage_bytes;
          for (int ph = 0; ph < p.n_phase; ++ph) {
            for (int g = 0; g < p.gps; ++g) {
              const int64_t plane = static_cast<int64_t>(ph) * p.c16 + ks * p.gps + g;
              const int8_t* src = p.act + (plane * p.plane_len + m0) * 16;
              bulk_g2s_w(dstA + (ph * p.gps + g) * strip_bytes, src, strip_bytes, &full[stage]);
            }
          }
          if (!p.b_resident) {
            const int8_t* src = p.wpk + (static_cast<int64_t>(nt) * p.k_stages + ks) * p.b_stage_bytes;
            bulk_g2s_evict_last_w(sB + stage * p.b_stage_bytes, src, p.b_stage_bytes, &full[stage], pol_b);
          }
          if (++stage == p.n_stages) {
            stage = 0;
            phase ^= 1u;
          }
        }
      }
      if (trace && lane == 0) trace[7] = clock64() - t_entry;
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    // Per-MMA descriptor offsets (16-byte units) are tabulated once: the issue
    // loop is then one smem load, two adds and the tcgen05.mma per instruction.
    uint2* tab = reinterpret_cast<uint2*>(smem + L.tab_off);
    const int n_mma = p.ntaps * (p.gps / 2);
    const uint32_t strip_bytes = p.strip_pix * 16u;
    const uint32_t b_lbo = p.block_n_tot * 16u;
    for (int i = lane; i < n_mma; i += 32) {
      const int tap = i / (p.gps / 2), g = (i % (p.gps / 2)) * 2;
      const uint32_t a_off = p.tap_phase[tap] * p.gps * strip_bytes + static_cast<uint32_t>(p.tap_shift[tap]) * 16u +
                             g * strip_bytes;
      const uint32_t b_off = (tap * p.gps + g) * b_lbo;
      tab[i] = make_uint2(a_off >> 4, b_off >> 4);
    }
    __syncwarp();
    if (n_units > 0) {
      if (p.b_resident) mbar_wait(bres, 0);
      int stage = 0;
      uint32_t phase = 0;
      int as = 0;
      uint32_t aphase = 0;
      const uint32_t n_main = p.block_n_tot > 256 ? 256u : static_cast<uint32_t>(p.block_n_tot);
      const uint32_t n_rest = p.block_n_tot > 256 ? static_cast<uint32_t>(p.block_n_tot - 256) : 0u;
      const uint32_t idesc_main = make_idesc_i8(n_main);
      const uint32_t idesc_rest = make_idesc_i8(n_rest > 0 ? n_rest : 16u);
      for (int u = 0; u < n_units; ++u) {
        mbar_wait(&tempty[as], aphase ^ 1u);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + as * acc_cols;
        for (int ks = 0; ks < p.k_stages; ++ks) {
          if (trace) {
            const long long w0 = clock64();
            mbar_wait(&full[stage], phase);
            const long long w1 = clock64();
            if (lane == 0) {
              if (u == 0 && ks == 0) trace[3] = w1 - t_entry;
              trace[9] += w1 - w0;
            }
          } else {
            mbar_wait(&full[stage], phase);
          }
          tc_fence_after();
          // warp-uniform issue: every lane walks the table, one elected lane issues
          const uint64_t a0 = make_sdesc(smem_u32(sA + stage * L.a_stage_bytes), strip_bytes, 128u);
          const uint64_t b0 = make_sdesc(
              smem_u32(p.b_resident ? sB + ks * p.b_stage_bytes : sB + stage * p.b_stage_bytes), b_lbo, 128u);
          uint32_t accum = ks > 0 ? 1u : 0u;
          if (n_rest) {
            for (int i = 0; i < n_mma; ++i) {
              const uint2 o = tab[i];
              mma_i8_w(d_tmem, a0 + o.x, b0 + o.y, idesc_main, accum);
              mma_i8_w(d_tmem + 256u, a0 + o.x, b0 + o.y + 256u, idesc_rest, accum);
              accum = 1u;
            }
          } else {
#pragma unroll 6
            for (int i = 0; i < n_mma; ++i) {
              const uint2 o = tab[i];
              mma_i8_w(d_tmem, a0 + o.x, b0 + o.y, idesc_main, accum);
              accum = 1u;
            }
          }
          mma_commit_w(&empty[stage]);
          if (++stage == p.n_stages) {
            stage = 0;
            phase ^= 1u;
          }
        }
        mma_commit_w(&tfull[as]);
        if (trace && lane == 0 && u == n_units - 1) trace[4] = clock64() - t_entry;
        if (++as == n_acc) {
          as = 0;
          aphase ^= 1u;
        }
      }
    }
  } else {
    // ------------------------------------------------------------ epilogue
    const int ew = warp - 2;                // 0..7
    const int quarter = warp & 3;           // TMEM lane quarter this warp may access
    const int half = ew >> 2;               // which alternate 16-column chunks
    const int row = quarter * 32 + lane;
    int as = 0;
    uint32_t aphase = 0;
    const uint32_t HlWl = static_cast<uint32_t>(p.Hl) * p.Wl;
    const int64_t PQ = static_cast<int64_t>(p.P) * p.Q;
    const bool bias_in_smem = p.K <= kBiasSmem;
    const float scale = p.scale;
    // chunk-sum in int32 is exact when 16 * max|acc| < 2^31 (CRS < 8192)
    const bool chunk32 = p.ntaps * p.c16 * 16 < 8192;
    for (int u = 0; u < n_units; ++u) {
      int mt, nt;
      decode_tile(p, u, mt, nt);
      const uint32_t m = static_cast<uint32_t>(mt) * kBlockM + row;
      uint32_t n_img = 0, pp = 0, qq = 0;
      bool valid = m < static_cast<uint64_t>(p.m_total);
      if (valid) {
        n_img = m / HlWl;
        const uint32_t rem = m - n_img * HlWl;
        pp = rem / p.Wl;
        qq = rem - pp * p.Wl;
        valid = pp < static_cast<uint32_t>(p.P) && qq < static_cast<uint32_t>(p.Q);
      }
      // per-row output base addresses
      int8_t* pk_row = nullptr;
      int64_t nchw_row = 0;
      if (EPI == EPI_PACKED || EPI == EPI_COMPARE) {
        const int hh = pp + p.o_ph, ww = qq + p.o_pw;
        const int a_ph = hh % p.o_sh, b_ph = ww % p.o_sw;
        const int64_t t = (static_cast<int64_t>(n_img) * p.o_Hl + hh / p.o_sh) * p.o_Wl + ww / p.o_sw;
        pk_row = static_cast<int8_t*>(p.out) +
                 (static_cast<int64_t>(a_ph * p.o_nph_w + b_ph) * p.o_c16 * p.o_plane_len + t) * 16;
      } else if (EPI == EPI_NCHW) {
        nchw_row = static_cast<int64_t>(n_img) * p.K * PQ + static_cast<int64_t>(pp) * p.Q + qq;
      }

      if (trace && warp == 2) {
        const long long w0 = clock64();
        mbar_wait(&tfull[as], aphase);
        if (lane == 0) trace[10] += clock64() - w0;
      } else {
        mbar_wait(&tfull[as], aphase);
      }
      tc_fence_after();
      const uint32_t t_row = tmem_base + (static_cast<uint32_t>(quarter * 32) << 16) + as * acc_cols;

      int64_t row_sum = 0;  // this warp's channels of the row (FC lhs part, FIC)
      const int k_base = nt * p.block_n;
      for (int cb = half * 16; cb < p.block_n; cb += 32) {
        uint32_t v[16];
        tmem_ld16(t_row + cb, v);
        tmem_ld_wait();
        int32_t a[16];
#pragma unroll
        for (int j = 0; j < 16; ++j) a[j] = static_cast<int32_t>(v[j]);
        const int k0 = k_base + cb;
        if (p.fault_key >= 0 && valid) {
          // ConvOut fault hook (faults.hpp:230-233): flip before checks and epilog
#pragma unroll
          for (int j = 0; j < 16; ++j) {
            const int64_t key = (static_cast<int64_t>(n_img) * p.K + k0 + j) * PQ + static_cast<int64_t>(pp) * p.Q + qq;
            if (key == p.fault_key) a[j] = static_cast<int32_t>(static_cast<uint32_t>(a[j]) ^ (1u << p.fault_bit));
          }
        }
        const bool kfull = k0 + 16 <= p.K;
        if (!kfull) {
#pragma unroll
          for (int j = 0; j < 16; ++j)
            if (k0 + j >= p.K) a[j] = 0;
        }
        if (FC || FIC || (p.check & CHECK_IC)) {
          if (chunk32) {
            int32_t s = 0;
#pragma unroll
            for (int j = 0; j < 16; ++j) s += a[j];
            row_sum += s;
          } else {
#pragma unroll
            for (int j = 0; j < 16; ++j) row_sum += a[j];
          }
        }
        if (p.check & CHECK_IC) {
          // per-channel column sums over the 32 rows of this warp, one atomic per channel
#pragma unroll
          for (int j = 0; j < 16; ++j) {
            long long s = valid ? a[j] : 0;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
            if (lane == j && k0 + j < p.K && s != 0) atomicAdd(&p.ic_sum[k0 + j], static_cast<unsigned long long>(s));
          }
        }
        if (EPI == EPI_PACKED || EPI == EPI_COMPARE) {
          int32_t y[16];
          if (bias_in_smem) {
            const float4* b4 = reinterpret_cast<const float4*>(s_bias + k0);
#pragma unroll
            for (int j4 = 0; j4 < 4; ++j4) {
              const float4 bb = b4[j4];
              y[j4 * 4 + 0] = requant_i8(a[j4 * 4 + 0], scale, bb.x, p.relu);
              y[j4 * 4 + 1] = requant_i8(a[j4 * 4 + 1], scale, bb.y, p.relu);
              y[j4 * 4 + 2] = requant_i8(a[j4 * 4 + 2], scale, bb.z, p.relu);
              y[j4 * 4 + 3] = requant_i8(a[j4 * 4 + 3], scale, bb.w, p.relu);
            }
          } else {
#pragma unroll
            for (int j = 0; j < 16; ++j) y[j] = requant_i8(a[j], scale, __ldg(p.bias + k0 + j), p.relu);
          }
          if (!kfull) {
#pragma unroll
            for (int j = 0; j < 16; ++j)
              if (k0 + j >= p.K) y[j] = 0;
          }
          const uint4 val = make_uint4(pack4(y[0], y[1], y[2], y[3]), pack4(y[4], y[5], y[6], y[7]),
                                       pack4(y[8], y[9], y[10], y[11]), pack4(y[12], y[13], y[14], y[15]));
          if (valid) {
            uint4* dst = reinterpret_cast<uint4*>(pk_row + static_cast<int64_t>(k0 >> 4) * p.o_plane_len * 16);
            if (EPI == EPI_PACKED) {
              *dst = val;
            } else {
              const uint4 ref = *dst;
              if (ref.x != val.x || ref.y != val.y || ref.z != val.z || ref.w != val.w) atomicAdd(p.cmp_count, 1ull);
            }
          }
        } else if (EPI == EPI_NCHW) {
          if (valid) {
            const int64_t base = nchw_row + static_cast<int64_t>(k0) * PQ;
            switch (p.out_mode) {
              case OUT_I32_NCHW: {
                int32_t* o = static_cast<int32_t*>(p.out) + base;
#pragma unroll
                for (int j = 0; j < 16; ++j)
                  if (k0 + j < p.K) o[j * PQ] = a[j];
                break;
              }
              case OUT_I8_NCHW: {
                int8_t* o = static_cast<int8_t*>(p.out) + base;
#pragma unroll
                for (int j = 0; j < 16; ++j)
                  if (k0 + j < p.K) o[j * PQ] = static_cast<int8_t>(requant_i8(a[j], scale, __ldg(p.bias + k0 + j), p.relu));
                break;
              }
              default: {  // OUT_F32_NCHW
                float* o = static_cast<float*>(p.out) + base;
#pragma unroll
                for (int j = 0; j < 16; ++j)
                  if (k0 + j < p.K) {
                    float f = __fmaf_rn(static_cast<float>(a[j]), scale, __ldg(p.bias + k0 + j));
                    if (p.relu && f < 0.0f) f = 0.0f;
                    o[j * PQ] = f;
                  }
                break;
              }
            }
          }
        }
      }
      int64_t extra = 0;
      if (FC && half == 0) {
        uint32_t v[16];
        tmem_ld16(t_row + p.block_n, v);
        tmem_ld_wait();
        extra = static_cast<int64_t>(static_cast<int32_t>(v[0])) +
                (static_cast<int64_t>(static_cast<int32_t>(v[1])) << 8) +
                (static_cast<int64_t>(static_cast<int32_t>(v[2])) << 16);
      }
      // accumulator consumed: hand the TMEM stage back to the MMA warp
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[as]);
      if (!valid) row_sum = 0;

      const int tile_id = nt * p.m_tiles + mt;
      if (FC) {
        // combine the two column halves of each row
        if (half == 1) s_rowsum[row] = row_sum;
        epi_bar();
        if (half == 0) {
          const int64_t lhs = row_sum + s_rowsum[row];
          if (p.n_tiles > 1) {
            int64_t* part = p.fc_part + (static_cast<int64_t>(nt) * p.m_tiles * kBlockM + m) * 2;
            part[0] = valid ? lhs : 0;
            part[1] = valid ? extra : 0;
          } else {
            const bool bad = valid && (lhs != extra);
            const unsigned ballot = __ballot_sync(0xffffffffu, bad);
            int64_t key = -1, l = 0, r = 0;
            if (ballot) {
              const int src = __ffs(ballot) - 1;
              key = __shfl_sync(0xffffffffu, static_cast<int64_t>(n_img) * PQ + static_cast<int64_t>(pp) * p.Q + qq, src);
              l = __shfl_sync(0xffffffffu, lhs, src);
              r = __shfl_sync(0xffffffffu, extra, src);
            }
            if (lane == 0) {
              s_red[quarter][0] = __popc(ballot);
              s_red[quarter][1] = key;
              s_red[quarter][2] = l;
              s_red[quarter][3] = r;
            }
          }
        }
        epi_bar();
        if (p.n_tiles == 1 && ew == 0 && lane == 0) {
          int64_t c = 0, k = -1, l = 0, r = 0;
          for (int qd = 0; qd < 4; ++qd) {
            c += s_red[qd][0];
            if (k < 0 && s_red[qd][1] >= 0) {
              k = s_red[qd][1];
              l = s_red[qd][2];
              r = s_red[qd][3];
            }
          }
          int64_t* rec = p.fc_rec + static_cast<int64_t>(tile_id) * 4;
          rec[0] = c;
          rec[1] = k;
          rec[2] = l;
          rec[3] = r;
        }
      }
      if (FIC) {
        long long s = row_sum;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        epi_bar();  // s_red reuse guard
        if (lane == 0) s_red[ew][0] = s;
        epi_bar();
        if (ew == 0 && lane == 0) {
          int64_t tot = 0;
#pragma unroll
          for (int w = 0; w < kEpiWarps; ++w) tot += s_red[w][0];
          p.fic_part[tile_id] = tot;
        }
      }
      if (++as == n_acc) {
        as = 0;
        aphase ^= 1u;
      }
    }
  }

  if (trace && warp == 2 && lane == 0) {
    trace[5] = clock64() - t_entry;
    trace[6] = n_units;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem_base, tmem_cols);
  }
}

}  // namespace abed_dev

// --------------------------------------------------------------------------
// host side launcher
// --------------------------------------------------------------------------
namespace abed_host {

using abed_dev::ConvTcParams;

uint32_t conv_tc_smem_bytes(const ConvTcParams& p) { return abed_dev::smem_layout(p).total; }

template <int EPI, bool FC, bool FIC>
static cudaError_t launch_variant(const ConvTcParams& p, int grid, cudaStream_t stream) {
  static bool attr_done = false;
  auto kern = abed_dev::conv_i8_tc_kernel<EPI, FC, FIC>;
  if (!attr_done) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, abed_dev::kConvDynSmemMax);
    if (e != cudaSuccess) return e;
    attr_done = true;
  }
  kern<<<grid, abed_dev::kConvThreads, conv_tc_smem_bytes(p), stream>>>(p);
  return cudaGetLastError();
}

template <int EPI>
static cudaError_t launch_epi(const ConvTcParams& p, int grid, cudaStream_t st) {
  const bool fc = (p.check & abed_dev::CHECK_FC) != 0, fic = (p.check & abed_dev::CHECK_FIC) != 0;
  if (fc && fic) return launch_variant<EPI, true, true>(p, grid, st);
  if (fc) return launch_variant<EPI, true, false>(p, grid, st);
  if (fic) return launch_variant<EPI, false, true>(p, grid, st);
  return launch_variant<EPI, false, false>(p, grid, st);
}

cudaError_t conv_tc_launch(const ConvTcParams& p, int num_sms, cudaStream_t stream) {
  int grid;
  if (p.b_resident) {
    int per = num_sms / p.n_tiles;
    if (per < 1) per = 1;
    if (per > p.m_tiles) per = p.m_tiles;
    grid = per * p.n_tiles;
  } else {
    grid = p.m_tiles * p.n_tiles;
    if (grid > num_sms) grid = num_sms;
  }
  switch (p.out_mode) {
    case abed_dev::OUT_NONE: return launch_epi<abed_dev::EPI_NONE>(p, grid, stream);
    case abed_dev::OUT_I8_PACKED: return launch_epi<abed_dev::EPI_PACKED>(p, grid, stream);
    case abed_dev::OUT_I8_COMPARE: return launch_epi<abed_dev::EPI_COMPARE>(p, grid, stream);
    default: return launch_epi<abed_dev::EPI_NCHW>(p, grid, stream);
  }
}

}  // namespace abed_host
