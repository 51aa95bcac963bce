// tcgen05 implicit-GEMM INT8 convolution with fused ABED checks and epilog.
//
// Replaces, on the device, the reference's int8 convolution
// (convolution.hpp:224 detail::conv_fast_i8 == :237 conv_direct) and, when a
// check is requested, the FC extra-fmap convolution + fc_verify
// (checksum.hpp:134-236), the FIC output reduction (:268, :287) and the IC
// per-channel reduction (:319-347), all inside the accumulator epilogue, before
// the fused scale/bias/ReLU/requantise (convolution.hpp:353-387).
//
// CTA = 6 warps, one CTA per SM, persistent over (M tile, N tile) work units:
//   warp 0      producer: one thread issues 1-D bulk copies (cp.async.bulk) of
//               the activation strips (and B blocks unless B is resident)
//   warp 1      TMEM allocator + single-thread tcgen05.mma issuer
//   warps 2..5  epilogue: tcgen05.ld (thread = GEMM row = output pixel),
//               checks, epilog, stores; double-buffered TMEM accumulators.
#include <cuda_runtime.h>

#include <cstdint>

#include "conv_tc.cuh"
#include "ptx.cuh"

namespace abed_dev {

struct SmemLayout {
  uint32_t a_off, a_stage_bytes, b_off, b_stage_bytes_smem, bar_off, total;
};

__host__ __device__ inline SmemLayout smem_layout(const ConvTcParams& p) {
  SmemLayout L;
  L.a_stage_bytes = static_cast<uint32_t>(p.n_phase) * p.gps * p.strip_pix * 16u;
  L.a_off = 0;
  uint32_t off = L.a_stage_bytes * kStages;
  off = (off + 127u) & ~127u;
  L.b_off = off;
  L.b_stage_bytes_smem = p.b_stage_bytes;
  off += p.b_resident ? p.b_stage_bytes * p.k_stages : p.b_stage_bytes * kStages;
  off = (off + 127u) & ~127u;
  L.bar_off = off;
  off += 8 * (2 * kStages + 5) + 16;
  L.total = off;
  return L;
}

__device__ __forceinline__ void decode_tile(const ConvTcParams& p, int tile_seq, int& mt,
                                            int& nt) {
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

__device__ __forceinline__ int8_t requant(int32_t acc, float scale, float bias, int relu) {
  // convolution.hpp:374-381 under the reference's -march=native build: the
  // multiply-add contracts to one fused FMA, then ReLU, clamp, truncate.
  float v = __fmaf_rn(static_cast<float>(acc), scale, bias);
  if (relu && v < 0.0f) v = 0.0f;
  v = fminf(127.0f, fmaxf(-128.0f, v));
  return static_cast<int8_t>(__float2int_rz(v));
}

__global__ void __launch_bounds__(kThreads, 1) conv_i8_tc_kernel(const __grid_constant__ ConvTcParams p) {
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
  __shared__ int64_t red_s64[4][4];

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;

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
      mbar_init(&tempty[i], 4);
    }
    mbar_init(bres, 1);
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc(tmem_slot, tmem_cols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  // number of work units for this CTA
  int n_units;
  if (p.b_resident) {
    const int per = gridDim.x / p.n_tiles;
    const int mt0 = blockIdx.x / p.n_tiles;
    n_units = (blockIdx.x < per * p.n_tiles && mt0 < p.m_tiles) ? (p.m_tiles - mt0 + per - 1) / per : 0;
  } else {
    const int total = p.m_tiles * p.n_tiles;
    n_units = blockIdx.x < total ? (total - blockIdx.x + gridDim.x - 1) / gridDim.x : 0;
  }

  if (warp == 0) {
    // ------------------------------------------------------------ producer
    if (lane == 0 && n_units > 0) {
      const uint64_t pol_b = policy_evict_last();
      if (p.b_resident) {
        const int nt = blockIdx.x % p.n_tiles;
        const uint32_t bytes = p.b_stage_bytes * p.k_stages;
        mbar_arrive_expect_tx(bres, bytes);
        const int8_t* src = p.wpk + static_cast<int64_t>(nt) * p.k_stages * p.b_stage_bytes;
        // split into <= 64 KB pieces
        for (uint32_t o = 0; o < bytes; o += 65536u) {
          const uint32_t sz = (bytes - o) < 65536u ? (bytes - o) : 65536u;
          bulk_g2s_evict_last(sB + o, src + o, sz, bres, pol_b);
        }
      }
      int stage = 0;
      uint32_t phase = 0;
      const uint32_t strip_bytes = p.strip_pix * 16u;
      for (int u = 0; u < n_units; ++u) {
        int mt, nt;
        decode_tile(p, u, mt, nt);
        const int64_t m0 = static_cast<int64_t>(mt) * kBlockM;
        for (int ks = 0; ks < p.k_stages; ++ks) {
          mbar_wait(&empty[stage], phase ^ 1u);
          const uint32_t bytes =
              L.a_stage_bytes + (p.b_resident ? 0u : p.b_stage_bytes);
          mbar_arrive_expect_tx(&full[stage], bytes);
          uint8_t* dstA = sA + stage * L.a_stage_bytes;
          for (int ph = 0; ph < p.n_phase; ++ph) {
            for (int g = 0; g < p.gps; ++g) {
              const int64_t plane = static_cast<int64_t>(ph) * p.c16 + ks * p.gps + g;
              const int8_t* src = p.act + (plane * p.plane_len + m0) * 16;
              bulk_g2s(dstA + (ph * p.gps + g) * strip_bytes, src, strip_bytes, &full[stage]);
            }
          }
          if (!p.b_resident) {
            const int8_t* src =
                p.wpk + (static_cast<int64_t>(nt) * p.k_stages + ks) * p.b_stage_bytes;
            bulk_g2s_evict_last(sB + stage * p.b_stage_bytes, src, p.b_stage_bytes, &full[stage],
                                pol_b);
          }
          if (++stage == kStages) {
            stage = 0;
            phase ^= 1u;
          }
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    if (n_units > 0) {
      if (p.b_resident) {
        mbar_wait(bres, 0);
      }
      int stage = 0;
      uint32_t phase = 0;
      int as = 0;
      uint32_t aphase = 0;
      const uint32_t strip_bytes = p.strip_pix * 16u;
      const uint32_t n_main = p.block_n_tot > 256 ? 256u : static_cast<uint32_t>(p.block_n_tot);
      const uint32_t n_rest = p.block_n_tot > 256 ? static_cast<uint32_t>(p.block_n_tot - 256) : 0u;
      const uint32_t idesc_main = make_idesc_i8(n_main);
      const uint32_t idesc_rest = make_idesc_i8(n_rest > 0 ? n_rest : 16u);
      const uint32_t b_lbo = p.block_n_tot * 16u;
      for (int u = 0; u < n_units; ++u) {
        mbar_wait(&tempty[as], aphase ^ 1u);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + as * acc_cols;
        uint32_t accum = 0;
        for (int ks = 0; ks < p.k_stages; ++ks) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          if (lane == 0) {
            const uint32_t a_base = smem_u32(sA + stage * L.a_stage_bytes);
            const uint32_t b_base = smem_u32(
                p.b_resident ? sB + ks * p.b_stage_bytes : sB + stage * p.b_stage_bytes);
            for (int tap = 0; tap < p.ntaps; ++tap) {
              const uint32_t a_tap = a_base + p.tap_phase[tap] * p.gps * strip_bytes +
                                     static_cast<uint32_t>(p.tap_shift[tap]) * 16u;
              for (int g = 0; g < p.gps; g += 2) {
                const uint64_t adesc = make_sdesc(a_tap + g * strip_bytes, strip_bytes, 128u);
                const uint32_t b_off = (tap * p.gps + g) * b_lbo;
                const uint64_t bdesc = make_sdesc(b_base + b_off, b_lbo, 128u);
                mma_i8(d_tmem, adesc, bdesc, idesc_main, accum);
                if (n_rest) {
                  const uint64_t bdesc2 = make_sdesc(b_base + b_off + 256u * 16u, b_lbo, 128u);
                  mma_i8(d_tmem + 256u, adesc, bdesc2, idesc_rest, accum);
                }
                accum = 1;
              }
            }
            mma_commit(&empty[stage]);
          }
          __syncwarp();
          if (++stage == kStages) {
            stage = 0;
            phase ^= 1u;
          }
        }
        if (lane == 0) mma_commit(&tfull[as]);
        __syncwarp();
        if (++as == n_acc) {
          as = 0;
          aphase ^= 1u;
        }
      }
    }
  } else {
    // ------------------------------------------------------------ epilogue
    const int quarter = warp & 3;  // TMEM lane quarter this warp may access
    const int row = quarter * 32 + lane;
    const int ew = warp - 2;       // 0..3
    int as = 0;
    uint32_t aphase = 0;
    const int64_t PQ = static_cast<int64_t>(p.P) * p.Q;
    const int64_t HlWl = static_cast<int64_t>(p.Hl) * p.Wl;
    for (int u = 0; u < n_units; ++u) {
      int mt, nt;
      decode_tile(p, u, mt, nt);
      const int64_t m = static_cast<int64_t>(mt) * kBlockM + row;
      int n_img = 0, pp = 0, qq = 0;
      bool valid = m < p.m_total;
      if (valid) {
        n_img = static_cast<int>(m / HlWl);
        const int64_t rem = m - n_img * HlWl;
        pp = static_cast<int>(rem / p.Wl);
        qq = static_cast<int>(rem - static_cast<int64_t>(pp) * p.Wl);
        valid = pp < p.P && qq < p.Q;
      }
      const int64_t ref_pix = static_cast<int64_t>(n_img) * PQ + static_cast<int64_t>(pp) * p.Q + qq;

      mbar_wait(&tfull[as], aphase);
      tc_fence_after();
      const uint32_t t_row = tmem_base + (static_cast<uint32_t>(quarter * 32) << 16) + as * acc_cols;

      int64_t row_sum = 0;   // sum over this tile's channels (FC lhs part, FIC)
      const int k_base = nt * p.block_n;
      for (int cb = 0; cb < p.block_n; cb += 16) {
        uint32_t v[16];
        tmem_ld16(t_row + cb, v);
        tmem_ld_wait();
        int32_t a[16];
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          a[j] = static_cast<int32_t>(v[j]);
          const int k = k_base + cb + j;
          if (p.fault_key >= 0 && valid && k < p.K) {
            const int64_t key = (static_cast<int64_t>(n_img) * p.K + k) * PQ +
                                static_cast<int64_t>(pp) * p.Q + qq;
            if (key == p.fault_key) a[j] = static_cast<int32_t>(static_cast<uint32_t>(a[j]) ^ (1u << p.fault_bit));
          }
          if (!(valid && k < p.K)) a[j] = 0;
          row_sum += a[j];
        }
        if (p.check & CHECK_IC) {
          // per-channel column sums over the 32 rows of this warp, then one
          // atomic per channel per warp
#pragma unroll
          for (int j = 0; j < 16; ++j) {
            long long s = a[j];
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
            const int k = k_base + cb + j;
            if (lane == j && k < p.K && s != 0)
              atomicAdd(&p.ic_sum[k], static_cast<unsigned long long>(s));
          }
        }
        if (valid) {
          const int k0 = k_base + cb;
          switch (p.out_mode) {
            case OUT_I32_NCHW: {
              int32_t* o = static_cast<int32_t*>(p.out);
#pragma unroll
              for (int j = 0; j < 16; ++j)
                if (k0 + j < p.K)
                  o[(static_cast<int64_t>(n_img) * p.K + k0 + j) * PQ + static_cast<int64_t>(pp) * p.Q + qq] = a[j];
              break;
            }
            case OUT_I8_NCHW: {
              int8_t* o = static_cast<int8_t*>(p.out);
#pragma unroll
              for (int j = 0; j < 16; ++j)
                if (k0 + j < p.K)
                  o[(static_cast<int64_t>(n_img) * p.K + k0 + j) * PQ + static_cast<int64_t>(pp) * p.Q + qq] =
                      requant(a[j], p.scale, __ldg(p.bias + k0 + j), p.relu);
              break;
            }
            case OUT_F32_NCHW: {
              float* o = static_cast<float*>(p.out);
#pragma unroll
              for (int j = 0; j < 16; ++j)
                if (k0 + j < p.K) {
                  float f = __fmaf_rn(static_cast<float>(a[j]), p.scale, __ldg(p.bias + k0 + j));
                  if (p.relu && f < 0.0f) f = 0.0f;
                  o[(static_cast<int64_t>(n_img) * p.K + k0 + j) * PQ + static_cast<int64_t>(pp) * p.Q + qq] = f;
                }
              break;
            }
            case OUT_I8_PACKED:
            case OUT_I8_COMPARE: {
              uint32_t w4[4];
#pragma unroll
              for (int j4 = 0; j4 < 4; ++j4) {
                uint32_t word = 0;
#pragma unroll
                for (int b = 0; b < 4; ++b) {
                  const int j = j4 * 4 + b;
                  const int8_t y = (k0 + j < p.K) ? requant(a[j], p.scale, __ldg(p.bias + k0 + j), p.relu) : int8_t(0);
                  word |= static_cast<uint32_t>(static_cast<uint8_t>(y)) << (8 * b);
                }
                w4[j4] = word;
              }
              // output pixel (n, h=pp, w=qq) -> next layer's phase/sub-pixel
              const int hh = pp + p.o_ph, ww = qq + p.o_pw;
              const int a_ph = hh % p.o_sh, b_ph = ww % p.o_sw;
              const int ii = hh / p.o_sh, jj = ww / p.o_sw;
              const int phase_id = a_ph * p.o_nph_w + b_ph;
              const int64_t t = (static_cast<int64_t>(n_img) * p.o_Hl + ii) * p.o_Wl + jj;
              const int g = k0 >> 4;
              uint4* dst = reinterpret_cast<uint4*>(static_cast<int8_t*>(p.out) +
                                                    ((static_cast<int64_t>(phase_id) * p.o_c16 + g) * p.o_plane_len + t) * 16);
              const uint4 val = make_uint4(w4[0], w4[1], w4[2], w4[3]);
              if (p.out_mode == OUT_I8_PACKED) {
                *dst = val;
              } else {
                const uint4 ref = *dst;
                if (ref.x != val.x || ref.y != val.y || ref.z != val.z || ref.w != val.w)
                  atomicAdd(p.cmp_count, 1ull);
              }
              break;
            }
            default:
              break;
          }
        }
      }
      int64_t extra = 0;
      if (p.check & CHECK_FC) {
        uint32_t v[16];
        tmem_ld16(t_row + p.block_n, v);
        tmem_ld_wait();
        extra = static_cast<int64_t>(static_cast<int32_t>(v[0])) +
                (static_cast<int64_t>(static_cast<int32_t>(v[1])) << 8) +
                (static_cast<int64_t>(static_cast<int32_t>(v[2])) << 16);
        if (!valid) extra = 0;
      }
      // accumulator consumed: hand TMEM stage back to the MMA warp
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[as]);

      const int tile_id = nt * p.m_tiles + mt;
      if (p.check & CHECK_FC) {
        if (p.n_tiles > 1) {
          int64_t* part = p.fc_part + (static_cast<int64_t>(nt) * p.m_tiles * kBlockM + mt * kBlockM + row) * 2;
          part[0] = row_sum;
          part[1] = extra;
        } else {
          const bool bad = valid && (row_sum != extra);
          const unsigned ballot = __ballot_sync(0xffffffffu, bad);
          int64_t cnt = __popc(ballot);
          // first mismatching row of this warp (rows are in reference order)
          int64_t key = -1, lhs = 0, rhs = 0;
          if (ballot) {
            const int src = __ffs(ballot) - 1;
            key = __shfl_sync(0xffffffffu, ref_pix, src);
            lhs = __shfl_sync(0xffffffffu, row_sum, src);
            rhs = __shfl_sync(0xffffffffu, extra, src);
          }
          if (lane == 0) {
            red_s64[quarter][0] = cnt;
            red_s64[quarter][1] = key;
            red_s64[quarter][2] = lhs;
            red_s64[quarter][3] = rhs;
          }
          asm volatile("bar.sync 1, 128;" ::: "memory");
          if (ew == 0 && lane == 0) {
            int64_t c = 0, k = -1, l = 0, r = 0;
            for (int qd = 0; qd < 4; ++qd) {
              c += red_s64[qd][0];
              if (k < 0 && red_s64[qd][1] >= 0) {
                k = red_s64[qd][1];
                l = red_s64[qd][2];
                r = red_s64[qd][3];
              }
            }
            int64_t* rec = p.fc_rec + static_cast<int64_t>(tile_id) * 4;
            rec[0] = c;
            rec[1] = k;
            rec[2] = l;
            rec[3] = r;
          }
          asm volatile("bar.sync 1, 128;" ::: "memory");
        }
      }
      if (p.check & CHECK_FIC) {
        long long s = row_sum;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        if (lane == 0) red_s64[quarter][0] = s;
        asm volatile("bar.sync 1, 128;" ::: "memory");
        if (ew == 0 && lane == 0)
          p.fic_part[tile_id] = red_s64[0][0] + red_s64[1][0] + red_s64[2][0] + red_s64[3][0];
        asm volatile("bar.sync 1, 128;" ::: "memory");
      }
      if (++as == n_acc) {
        as = 0;
        aphase ^= 1u;
      }
    }
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

cudaError_t conv_tc_launch(const ConvTcParams& p, int num_sms, cudaStream_t stream) {
  const uint32_t smem = conv_tc_smem_bytes(p);
  static bool attr_done = false;
  if (!attr_done) {
    cudaError_t e = cudaFuncSetAttribute(abed_dev::conv_i8_tc_kernel,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, 232448 - 1024);
    if (e != cudaSuccess) return e;
    attr_done = true;
  }
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
  abed_dev::conv_i8_tc_kernel<<<grid, abed_dev::kThreads, smem, stream>>>(p);
  return cudaGetLastError();
}

}  // namespace abed_host
