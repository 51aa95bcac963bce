// tcgen05 implicit-GEMM INT8 convolution with fused ABED checks, verdicts and epilog.
//
// Replaces, on the device, the reference's int8 convolution
// (convolution.hpp:224 detail::conv_fast_i8 == :237 conv_direct) and, when a
// check is requested, the FC extra-fmap convolution + fc_verify
// (checksum.hpp:134-236), the FIC input checksum dot (gen_input_checksum +
// fic_dot, :248-285, the "FR" option: a second, independent read of the stored
// input), the FIC output reduction and verdict (:268, :287), and the IC
// per-channel reduction (:319-347), all inside one kernel, before the fused
// scale/bias/ReLU/requantise (convolution.hpp:353-387).
//
// CTA = 12 warps, one CTA per SM, persistent over (M tile, N tile) work units:
//   warp 0      producer: one elected lane issues 1-D bulk copies
//               (cp.async.bulk) of the activation strips and B blocks (or the
//               CTA's whole resident N tile of B once)
//   warp 1      TMEM allocator + tcgen05.mma issuer (warp-uniform loop)
//   warps 2..9  epilogue: thread = GEMM row (output pixel); the two warps of a
//               TMEM lane quarter split the tile's channels into halves;
//               checks, epilog and stores straight from tcgen05.ld registers;
//               double-buffered TMEM accumulators overlap the next unit's MMAs
//   warps 10,11 input checksum (FIC rhs = sum x.G over this CTA's share of the
//               stored input), when the plan computes it in-kernel
// The last CTA to finish reduces the per-CTA records and writes the FC and FIC
// abed_verify_outcome (checksum.hpp:30-51 VerifyOutcome) itself.
//
// The kernel opens with griddepcontrol (programmatic dependent launch): barrier
// init, TMEM allocation and the resident-filter prefetch overlap the previous
// kernel's tail; activations, outputs and accumulators are touched only after
// griddepcontrol.wait.
#pragma once
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <type_traits>

#include "abed_b200.h"
#include "conv_tc.cuh"
#include "ptx.cuh"

namespace abed_dev {

constexpr int kEpiWarps = 8;
constexpr int kEpiParts = kEpiWarps / 4;  // epilogue warps per TMEM lane quarter
constexpr int kMaxAcc = 2 * kEpiParts;     // TMEM accumulator stages (unit-interleaved epilogue)
// Timing-experiment flags (ConvTcParams::dbg, tools/epi_probe.py) exist only in a
// diagnostics build (-DABED_CONV_DEBUG=1): the product kernels carry none of their
// code (the epilogue's extra copies cost instruction-cache footprint)
#ifndef ABED_CONV_DEBUG
#define ABED_CONV_DEBUG 0
#endif
__device__ __forceinline__ int dbg_of(const ConvTcParams& p) { return ABED_CONV_DEBUG ? p.dbg : 0; }
constexpr int kEpiThreads = kEpiWarps * 32;
constexpr int kRhsWarps = 2;
constexpr int kConvThreads = 64 + kEpiThreads + kRhsWarps * 32;
static_assert(kConvThreads == kConvThreads_host, "host copy of the conv CTA size");
constexpr int kBiasSmem = 2048;
constexpr int kBarEpi = 1;       // named barrier: all epilogue warps
constexpr int kBarHalf0 = 2;     // named barrier: the four part-0 epilogue warps
constexpr int kBarQuarter0 = 4;  // named barriers 4..7: the epilogue warps of a TMEM lane quarter
constexpr int64_t kNoKey = 0x7fffffffffffffffll;

// compile-time output flavours
enum EpiKind : int { EPI_NONE = 0, EPI_NCHW = 1, EPI_PACKED = 2, EPI_COMPARE = 3 };

struct SmemLayout {
  uint32_t a_off, a_stage_bytes, b_off, bar_off, tab_off, fic_off, ic_off, total;
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
  off += 8 * (2 * kStages + 2 * kMaxAcc + 1) + 16;
  L.tab_off = off;  // per-stage MMA operand offset table (uint2 per MMA)
  off += 8u * p.ntaps * (p.gps / 2);
  off = (off + 15u) & ~15u;
  L.fic_off = off;  // FIC-SM class table + row / column classes, then its mbarrier
  off += p.fic_smem ? p.fic_smem + 16u : 0u;
  off = (off + 15u) & ~15u;
  L.ic_off = off;  // IC per-channel output sums of this CTA (flushed once at exit)
  off += p.ic_smem;
  L.total = off;
  return L;
}

__device__ __forceinline__ void decode_tile(const ConvTcParams& p, int tile_seq, int& mt, int& nt) {
  // b_resident with several N tiles: each CTA owns one N tile (blockIdx % n_tiles)
  if (p.b_resident) {
    nt = blockIdx.x % p.n_tiles;
    mt = blockIdx.x / p.n_tiles + tile_seq * (p.conv_grid / p.n_tiles);
  } else {
    const int t = blockIdx.x + tile_seq * p.conv_grid;
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

// requant_i8 with ReLU for two accumulators at once: one FFMA2 (fma.rn.f32x2 =
// two IEEE fmas, bit-identical to __fmaf_rn), one FADD2.RZ putting trunc(v) in
// the mantissa of 2^23 + v, and the clamp to [0, 127] done on the float's bit
// pattern with one DPX add-min-relu per value (positive floats order like their
// bits; v < 0 gives a pattern below 2^23's, v >= 127 one above 2^23 + 127, and
// every v in [0, 2^23) lands exactly on 2^23 + trunc(v)).
__device__ __forceinline__ void requant_relu_pair(int32_t a0, int32_t a1, float scale, float b0, float b1, int32_t& y0,
                                                  int32_t& y1) {
  const uint64_t v = (static_cast<uint64_t>(__float_as_uint(static_cast<float>(a1))) << 32) |
                     __float_as_uint(static_cast<float>(a0));
  const uint64_t sc = (static_cast<uint64_t>(__float_as_uint(scale)) << 32) | __float_as_uint(scale);
  const uint64_t bb = (static_cast<uint64_t>(__float_as_uint(b1)) << 32) | __float_as_uint(b0);
  uint64_t r;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(v), "l"(sc), "l"(bb));
  asm("add.rz.f32x2 %0, %1, %2;" : "=l"(r) : "l"(r), "l"(0x4B0000004B000000ull));
  y0 = __viaddmin_s32_relu(static_cast<int>(static_cast<uint32_t>(r)), -0x4B000000, 127);
  y1 = __viaddmin_s32_relu(static_cast<int>(static_cast<uint32_t>(r >> 32)), -0x4B000000, 127);
}

__device__ __forceinline__ uint32_t pack4(int32_t a, int32_t b, int32_t c, int32_t d) {
  const uint32_t lo = __byte_perm(static_cast<uint32_t>(a), static_cast<uint32_t>(b), 0x0040u);
  const uint32_t hi = __byte_perm(static_cast<uint32_t>(c), static_cast<uint32_t>(d), 0x0040u);
  return __byte_perm(lo, hi, 0x5410u);
}

// running FC record of one thread / warp / CTA: mismatch count and the first
// mismatching key (reference loop order) with its lhs / rhs
struct FcRec {
  int64_t cnt, key, lhs, rhs;
};
__device__ __forceinline__ void fc_note(FcRec& r, int64_t key, int64_t lhs, int64_t rhs) {
  ++r.cnt;
  if (key < r.key) {
    r.key = key;
    r.lhs = lhs;
    r.rhs = rhs;
  }
}
// exact (int64) or float-mode (f64) sums travel through int64 slots as bits
__device__ __forceinline__ int64_t acc_bits(int64_t v) { return v; }
__device__ __forceinline__ int64_t acc_bits(double v) { return __double_as_longlong(v); }
template <typename T>
__device__ __forceinline__ T bits_acc(int64_t b) {
  if constexpr (std::is_same_v<T, double>)
    return __longlong_as_double(b);
  else
    return b;
}
// fc_verify (exact, checksum.hpp:211-236) / fc_verify_f32 (|lhs - rhs| <= tau, :541-565)
template <int DT, typename T>
__device__ __forceinline__ bool fc_mismatch(T lhs, T rhs, double tau) {
  if constexpr (DT == DT_I8)
    return lhs != rhs;
  else
    return !(fabs(static_cast<double>(lhs) - static_cast<double>(rhs)) <= tau);
}
__device__ __forceinline__ FcRec fc_warp_reduce(FcRec r) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    FcRec t;
    t.cnt = __shfl_xor_sync(0xffffffffu, r.cnt, o);
    t.key = __shfl_xor_sync(0xffffffffu, r.key, o);
    t.lhs = __shfl_xor_sync(0xffffffffu, r.lhs, o);
    t.rhs = __shfl_xor_sync(0xffffffffu, r.rhs, o);
    r.cnt += t.cnt;
    if (t.key < r.key) {
      r.key = t.key;
      r.lhs = t.lhs;
      r.rhs = t.rhs;
    }
  }
  return r;
}
__device__ __forceinline__ long long warp_sum(long long s) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  return s;
}

__device__ __forceinline__ double warp_sum_d(double s) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  return s;
}

// two floats -> two 16-bit storage values (fp16 or bf16, round to nearest even)
template <int DT>
__device__ __forceinline__ uint32_t pack_h2(float a, float b) {
  if constexpr (DT == DT_BF16) {
    const __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
    return *reinterpret_cast<const uint32_t*>(&h);
  } else {
    const __half2 h = __floats2half2_rn(a, b);
    return *reinterpret_cast<const uint32_t*>(&h);
  }
}
// one 32-bit word of two 16-bit storage values -> two floats
template <int DT>
__device__ __forceinline__ float2 unpack_h2(uint32_t w) {
  if constexpr (DT == DT_BF16) {
    return make_float2(__uint_as_float(w << 16), __uint_as_float(w & 0xFFFF0000u));
  } else {
    __half2 h = *reinterpret_cast<const __half2*>(&w);
    return __half22float2(h);
  }
}

__device__ __forceinline__ void write_outcome_dev(abed_verify_outcome* o, int mismatch, int has_locus, int64_t l0,
                                                  int64_t l1, int64_t l2, int64_t lhs, int64_t rhs, int64_t count) {
  o->status = mismatch;
  o->has_locus = has_locus;
  o->locus[0] = l0;
  o->locus[1] = l1;
  o->locus[2] = l2;
  o->lhs = lhs;
  o->rhs = rhs;
  o->lhs_f = 0.0;
  o->rhs_f = 0.0;
  o->error_count = count;
}

// per-thread epilogue state of the current GEMM row
struct EpiCtx {
  int64_t PQ;
  const float* bias_smem;  // nullptr: bias read from global
  int8_t* pk_row;          // EPI_PACKED / EPI_COMPARE: this row's 16-byte pixel in plane 0
  int64_t nchw_row;        // EPI_NCHW: element (n, 0, p, q)
  int fk_k;                // ConvOut fault channel (or -1)
  bool chunk32, valid, fault_row;
  const uint4* af_row;     // FIC-AF: next layer's digit cell of this pixel, group 0 (nullptr: off)
  int64_t af_gstride;      // uint4 stride between channel groups of the digit planes
  unsigned long long* ic_acc;   // IC: the CTA's shared per-channel sums (nullptr: straight to global)
  unsigned long long* icb_lhs;  // ICBatch, real row: &icb_lhs[0][p][q] (nullptr: not a real row)
  int32_t* icb_dig;             // ICBatch, digit row j: &icb_dig[j][0][p][q] (nullptr: not a digit row)
};

// IC (ic_verify_k's lhs, checksum.hpp:319-347): per-channel sums of one chunk
// over the warp's 32 rows by a transpose-reduce butterfly -- xor 16 / 8 / 4 / 2
// halve the channels each lane carries (int32: 16 rows of |acc| < 2^27), xor 1
// adds the two 16-row halves in int64 -- 17 shuffles per 16 channels instead of
// 16 separate 64-bit warp reductions; each even lane then owns one channel's sum
// and adds it into the CTA's shared accumulator (flushed to global once per CTA:
// per-warp global reductions on the same K addresses serialised in L2).
__device__ __forceinline__ void ic_chunk_sums(const ConvTcParams& p, unsigned long long* ic_acc, bool valid,
                                              const int32_t (&a)[16], int k0) {
  const int lane = threadIdx.x & 31;
  int32_t v[16];
#pragma unroll
  for (int j = 0; j < 16; ++j) v[j] = valid ? a[j] : 0;
  int32_t w8[8], w4[4], w2[2];
  const bool b4 = lane & 16, b3 = lane & 8, b2 = lane & 4, b1 = lane & 2;
#pragma unroll
  for (int j = 0; j < 8; ++j) w8[j] = (b4 ? v[j + 8] : v[j]) + __shfl_xor_sync(0xffffffffu, b4 ? v[j] : v[j + 8], 16);
#pragma unroll
  for (int j = 0; j < 4; ++j) w4[j] = (b3 ? w8[j + 4] : w8[j]) + __shfl_xor_sync(0xffffffffu, b3 ? w8[j] : w8[j + 4], 8);
#pragma unroll
  for (int j = 0; j < 2; ++j) w2[j] = (b2 ? w4[j + 2] : w4[j]) + __shfl_xor_sync(0xffffffffu, b2 ? w4[j] : w4[j + 2], 4);
  const int32_t w1 = (b1 ? w2[1] : w2[0]) + __shfl_xor_sync(0xffffffffu, b1 ? w2[0] : w2[1], 2);
  const long long sum = static_cast<long long>(w1) + __shfl_xor_sync(0xffffffffu, static_cast<long long>(w1), 1);
  const int ch = (b4 ? 8 : 0) + (b3 ? 4 : 0) + (b2 ? 2 : 0) + (b1 ? 1 : 0);
  if (!(lane & 1) && k0 + ch < p.K && sum != 0) {
    if (ic_acc)
      atomicAdd(ic_acc + k0 + ch, static_cast<unsigned long long>(sum));
    else
      red_add_u64(&p.ic_sum[k0 + ch], static_cast<unsigned long long>(sum));
  }
}

// ICBatch (checksum.hpp:398-421): a real row adds its 16 outputs into the
// per-(k, p, q) batch sums; a row of digit image j stores conv(d_j) for the scan
template <bool TRIM>
__device__ __forceinline__ void icb_chunk(const ConvTcParams& p, const EpiCtx& e, const int32_t (&a)[16], int k0) {
  if (e.icb_lhs) {
    unsigned long long* q = e.icb_lhs + static_cast<int64_t>(k0) * e.PQ;
#pragma unroll
    for (int j = 0; j < 16; ++j)
      if (!TRIM || k0 + j < p.K) red_add_u64(q + j * e.PQ, static_cast<unsigned long long>(static_cast<long long>(a[j])));
  } else if (e.icb_dig) {
    int32_t* q = e.icb_dig + static_cast<int64_t>(k0) * e.PQ;
#pragma unroll
    for (int j = 0; j < 16; ++j)
      if (!TRIM || k0 + j < p.K) q[j * e.PQ] = a[j];
  }
}

// One 16-channel chunk of one row: (slow path only: fault hook, filler trim),
// row sum, IC / ICBatch extras (XTRA 1 / 2 on the fast path; by plan on the slow
// path), requantise + store (or compare).  Returns the chunk's
// contribution to the row sum.  b = the chunk's 16 biases.
template <int EPI, bool RELU, bool SUMS, bool SLOW, bool C32 = false, int XTRA = 0>
__device__ __forceinline__ int64_t epi_chunk(const ConvTcParams& p, const EpiCtx& e, int32_t (&a)[16],
                                             const float (&b)[16], int k0, long long& af_out) {
  if (SLOW) {
    if (e.fault_row && e.fk_k >= k0 && e.fk_k < k0 + 16) {
#pragma unroll
      for (int j = 0; j < 16; ++j)
        if (k0 + j == e.fk_k) a[j] = static_cast<int32_t>(static_cast<uint32_t>(a[j]) ^ (1u << p.fault_bit));
    }
#pragma unroll
    for (int j = 0; j < 16; ++j)
      if (k0 + j >= p.K) a[j] = 0;
  }
  int64_t sum = 0;
  if (SUMS) {
    // C32 (compile time, chosen per layer from e.chunk32): the 16-value chunk sum
    // in int32 (exact when CRS < 8192) -- a runtime flag here made the compiler
    // evaluate both the int32 and the sign-extended int64 chains (~2.7 instr/value)
    if constexpr (C32) {
      int32_t s = 0;
#pragma unroll
      for (int j = 0; j < 16; ++j) s += a[j];
      sum = s;
    } else {
#pragma unroll
      for (int j = 0; j < 16; ++j) sum += a[j];
    }
  }
  if (XTRA == 1) ic_chunk_sums(p, e.ic_acc, e.valid, a, k0);
  if (XTRA == 2) icb_chunk<SLOW>(p, e, a, k0);
  // the slow path (fault hook, filler channels) is one copy with the activation
  // read at run time; the fast path has one copy per activation
  const bool relu = SLOW ? p.relu != 0 : RELU;
  if (EPI == EPI_PACKED || EPI == EPI_COMPARE) {
    int32_t y[16];
    if (dbg_of(p) & 16) {  // timing experiment: skip the requantise math
#pragma unroll
      for (int j = 0; j < 16; ++j) y[j] = a[j];
    } else if (relu) {
#pragma unroll
      for (int j = 0; j < 16; j += 2) requant_relu_pair(a[j], a[j + 1], p.scale, b[j], b[j + 1], y[j], y[j + 1]);
    } else {
#pragma unroll
      for (int j = 0; j < 16; ++j) y[j] = requant_i8(a[j], p.scale, b[j], 0);
    }
    if (SLOW) {
#pragma unroll
      for (int j = 0; j < 16; ++j)
        if (k0 + j >= p.K) y[j] = 0;
    }
    const uint4 val = make_uint4(pack4(y[0], y[1], y[2], y[3]), pack4(y[4], y[5], y[6], y[7]),
                                 pack4(y[8], y[9], y[10], y[11]), pack4(y[12], y[13], y[14], y[15]));
    uint4* dst = reinterpret_cast<uint4*>(e.pk_row + static_cast<int64_t>(k0 >> 4) * p.o_plane_len * 16);
    if (EPI == EPI_PACKED) {
      if (e.valid) {
        *dst = val;
        if (XTRA != 0 && e.af_row) {  // FIC-AF: the next layer's rhs from the stored values (12 dp4a)
          const uint4* gd = e.af_row + static_cast<int64_t>(k0 >> 4) * e.af_gstride;
          const uint4 g0 = __ldg(gd), g1 = __ldg(gd + 1), g2 = __ldg(gd + 2);
          int32_t d0 = 0, d1 = 0, d2 = 0;
          d0 = __dp4a(static_cast<int>(val.x), static_cast<int>(g0.x), d0);
          d0 = __dp4a(static_cast<int>(val.y), static_cast<int>(g0.y), d0);
          d0 = __dp4a(static_cast<int>(val.z), static_cast<int>(g0.z), d0);
          d0 = __dp4a(static_cast<int>(val.w), static_cast<int>(g0.w), d0);
          d1 = __dp4a(static_cast<int>(val.x), static_cast<int>(g1.x), d1);
          d1 = __dp4a(static_cast<int>(val.y), static_cast<int>(g1.y), d1);
          d1 = __dp4a(static_cast<int>(val.z), static_cast<int>(g1.z), d1);
          d1 = __dp4a(static_cast<int>(val.w), static_cast<int>(g1.w), d1);
          d2 = __dp4a(static_cast<int>(val.x), static_cast<int>(g2.x), d2);
          d2 = __dp4a(static_cast<int>(val.y), static_cast<int>(g2.y), d2);
          d2 = __dp4a(static_cast<int>(val.z), static_cast<int>(g2.z), d2);
          d2 = __dp4a(static_cast<int>(val.w), static_cast<int>(g2.w), d2);
          af_out += static_cast<long long>(d0) + (static_cast<long long>(d1) << 8) + (static_cast<long long>(d2) << 16);
        }
      }
    } else if (e.valid) {
      const uint4 ref = *dst;
      if (ref.x != val.x || ref.y != val.y || ref.z != val.z || ref.w != val.w) atomicAdd(p.cmp_count, 1ull);
    }
  } else if (EPI == EPI_NCHW) {
    if (e.valid) {
      const int64_t base = e.nchw_row + static_cast<int64_t>(k0) * e.PQ;
      if (p.out_mode == OUT_I32_NCHW) {
        int32_t* o = static_cast<int32_t*>(p.out) + base;
        for (int j = 0; j < 16; ++j)
          if (k0 + j < p.K) o[j * e.PQ] = a[j];
      } else if (p.out_mode == OUT_I8_NCHW) {
        int8_t* o = static_cast<int8_t*>(p.out) + base;
        for (int j = 0; j < 16; ++j)
          if (k0 + j < p.K) o[j * e.PQ] = static_cast<int8_t>(requant_i8(a[j], p.scale, b[j], relu ? 1 : 0));
      } else {  // OUT_F32_NCHW
        float* o = static_cast<float*>(p.out) + base;
        for (int j = 0; j < 16; ++j)
          if (k0 + j < p.K) {
            float f = __fmaf_rn(static_cast<float>(a[j]), p.scale, b[j]);
            if (relu && f < 0.0f) f = 0.0f;
            o[j * e.PQ] = f;
          }
      }
    }
  }
  return sum;
}

// Float mode (fp16 / bf16 operands): one 16-channel chunk of f32 accumulators.
// Row sum in f64 (checksum.hpp:524 reduce_all_f64 / :541 fc_verify_f32 reduce
// in double); epilog v = fma(acc, scale, bias), ReLU, then f32 NCHW or 16-bit
// packed output (8 channels per 16-byte pixel).
template <int DT, int EPI, bool RELU, bool SUMS, bool SLOW>
__device__ __forceinline__ double epi_chunk_h(const ConvTcParams& p, const EpiCtx& e, uint32_t (&v)[16],
                                              const float (&b)[16], int k0) {
  if (SLOW) {
    if (e.fault_row && e.fk_k >= k0 && e.fk_k < k0 + 16) {
#pragma unroll
      for (int j = 0; j < 16; ++j)
        if (k0 + j == e.fk_k) v[j] ^= 1u << p.fault_bit;
    }
#pragma unroll
    for (int j = 0; j < 16; ++j)
      if (k0 + j >= p.K) v[j] = 0u;
  }
  float a[16];
#pragma unroll
  for (int j = 0; j < 16; ++j) a[j] = __uint_as_float(v[j]);
  double sum = 0.0;
  if (SUMS) {
    // f32 pairwise tree over the chunk, one conversion, f64 across chunks: 16
    // F2F.F64 + 16 DADD per chunk cost VGG-16 conv1_2 ~75 us.  The tree adds at
    // most 4 * 2^-24 * sum|out| to the lhs error, inside the thresholds' slack
    // ((CRS + 32) * 2^-22 per output, bench.py / DESIGN.md)
    float t8[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) t8[j] = a[2 * j] + a[2 * j + 1];
#pragma unroll
    for (int j = 0; j < 4; ++j) t8[j] = t8[2 * j] + t8[2 * j + 1];
    sum = static_cast<double>((t8[0] + t8[1]) + (t8[2] + t8[3]));
  }
  if (EPI == EPI_PACKED || EPI == EPI_COMPARE) {
    float y[16];
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      y[j] = __fmaf_rn(a[j], p.scale, b[j]);
      if (RELU) y[j] = fmaxf(y[j], 0.0f);
      if (SLOW && k0 + j >= p.K) y[j] = 0.0f;
    }
    const uint4 lo = make_uint4(pack_h2<DT>(y[0], y[1]), pack_h2<DT>(y[2], y[3]), pack_h2<DT>(y[4], y[5]),
                                pack_h2<DT>(y[6], y[7]));
    const uint4 hi = make_uint4(pack_h2<DT>(y[8], y[9]), pack_h2<DT>(y[10], y[11]), pack_h2<DT>(y[12], y[13]),
                                pack_h2<DT>(y[14], y[15]));
    const int64_t plane_bytes = p.o_plane_len * 16;
    uint4* dst0 = reinterpret_cast<uint4*>(e.pk_row + static_cast<int64_t>(k0 >> 3) * plane_bytes);
    uint4* dst1 = reinterpret_cast<uint4*>(e.pk_row + static_cast<int64_t>((k0 >> 3) + 1) * plane_bytes);
    if (EPI == EPI_PACKED) {
      if (e.valid) {
        *dst0 = lo;
        *dst1 = hi;
      }
    } else if (e.valid) {
      const uint4 r0 = *dst0, r1 = *dst1;
      const bool same = r0.x == lo.x && r0.y == lo.y && r0.z == lo.z && r0.w == lo.w && r1.x == hi.x &&
                        r1.y == hi.y && r1.z == hi.z && r1.w == hi.w;
      if (!same) atomicAdd(p.cmp_count, 1ull);
    }
  } else if (EPI == EPI_NCHW) {
    if (e.valid) {
      float* o = static_cast<float*>(p.out) + e.nchw_row + static_cast<int64_t>(k0) * e.PQ;
      for (int j = 0; j < 16; ++j)
        if (k0 + j < p.K) {
          float f = __fmaf_rn(a[j], p.scale, b[j]);
          if (RELU && f < 0.0f) f = 0.0f;
          o[j * e.PQ] = f;
        }
    }
  }
  return sum;
}

__device__ __forceinline__ void load_bias16(const ConvTcParams& p, const EpiCtx& e, int k0, float (&b)[16]) {
  if (e.bias_smem) {
    const float4* b4 = reinterpret_cast<const float4*>(e.bias_smem + k0);
#pragma unroll
    for (int j4 = 0; j4 < 4; ++j4) {
      const float4 bb = b4[j4];
      b[4 * j4] = bb.x;
      b[4 * j4 + 1] = bb.y;
      b[4 * j4 + 2] = bb.z;
      b[4 * j4 + 3] = bb.w;
    }
  } else {
#pragma unroll
    for (int j = 0; j < 16; ++j) b[j] = k0 + j < p.K ? __ldg(p.bias + k0 + j) : 0.0f;
  }
}

// Chunks [c_lo, c_hi) of one row, 32 columns per step.  TMEM loads are software
// pipelined (the next step's tcgen05.ld is in flight while this one is
// processed) and the biases are read before the wait.  The loop body is not
// unrolled across steps, so the epilogue stays resident in the instruction cache.
// An odd trailing chunk is loaded as a 16-column step.
template <int DT, int EPI, bool RELU, bool SUMS, bool SLOW, bool C32 = false, int XTRA = 0>
__device__ __forceinline__ std::conditional_t<DT == DT_I8, int64_t, double> epi_columns(
    const ConvTcParams& p, const EpiCtx& e, uint32_t t_row, int k_base, int c_lo, int c_hi, long long& af_out) {
  std::conditional_t<DT == DT_I8, int64_t, double> row_sum = 0;
  auto chunk = [&](uint32_t (&v)[16], const float (&b)[16], int k0) {
    if constexpr (DT == DT_I8) {
      int32_t a[16];
#pragma unroll
      for (int j = 0; j < 16; ++j) a[j] = static_cast<int32_t>(v[j]);
      row_sum += epi_chunk<EPI, RELU, SUMS, SLOW, C32, XTRA>(p, e, a, b, k0, af_out);
    } else {
      row_sum += epi_chunk_h<DT, EPI, RELU, SUMS, SLOW>(p, e, v, b, k0);
    }
  };
  const int pairs_end = c_lo + ((c_hi - c_lo) & ~1);
  if (c_lo < pairs_end) {
    uint32_t v[32];
    tmem_ld32(t_row + c_lo * 16, v);
#pragma unroll 1
    for (int c = c_lo; c < pairs_end; c += 2) {
      float b[16];
      load_bias16(p, e, k_base + c * 16, b);
      tmem_ld_wait();
      uint32_t a0[16], a1[16];
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        a0[j] = v[j];
        a1[j] = v[16 + j];
      }
      if (c + 2 < pairs_end) tmem_ld32(t_row + (c + 2) * 16, v);
      chunk(a0, b, k_base + c * 16);
      load_bias16(p, e, k_base + (c + 1) * 16, b);
      chunk(a1, b, k_base + (c + 1) * 16);
    }
  }
  if (pairs_end < c_hi) {
    uint32_t v[16];
    tmem_ld16(t_row + pairs_end * 16, v);
    float b[16];
    load_bias16(p, e, k_base + pairs_end * 16, b);
    tmem_ld_wait();
    chunk(v, b, k_base + pairs_end * 16);
  }
  return row_sum;
}

// ---------------------------------------------------------------- MMA issue
// Everything the MMA warp needs, set up once by the kernel.
struct MmaEnv {
  uint8_t* sA;
  uint8_t* sB;
  uint32_t a_stage_bytes;
  uint64_t* full;
  uint64_t* empty;
  uint64_t* tfull;
  uint64_t* tempty;
  uint64_t* bres;
  uint32_t tmem_base;
  int acc_cols, n_acc, n_units, lane;
  int64_t* trace;
  long long t_entry;
};

template <int DT>
__device__ __forceinline__ void issue_one(uint32_t d_tmem, uint32_t a_hi, uint32_t b_hi, uint32_t ao, uint32_t bo,
                                          uint32_t idesc, uint32_t accum) {
  const uint64_t ad = (static_cast<uint64_t>(a_hi) << 32) | ao, bd = (static_cast<uint64_t>(b_hi) << 32) | bo;
  if constexpr (DT == DT_I8)
    mma_i8_w(d_tmem, ad, bd, idesc, accum);  // K = 32 int8, s32 accumulate
  else
    mma_f16_w(d_tmem, ad, bd, idesc, accum);  // K = 16 fp16/bf16, f32 accumulate
}

// The MMA warp.  Per stage: every tap (r, s) x channel-group pair g; tap (r, s)
// reads stride phase (r % SH, s % SW) of the A strips at pixel shift
// (r / SH) * Wl + s / SW, and B advances one block_n_tot x 16-byte block per
// channel group.  For the common patterns (R > 0) the loop is unrolled at
// compile time and every per-MMA operand offset is computed once, before the
// unit loop, so issuing one tcgen05.mma is two uniform adds: measured on B200
// a loop that recomputes offsets from runtime geometry costs 85-128 cycles of
// issue per MMA (tools/mma_microbench3.cu), more than the MMA itself.
// R == 0: generic runtime loop (any filter size / stride).
template <int DT, int R, int S, int SH, int SW, int GPS>
__device__ __forceinline__ void mma_warp_run(const ConvTcParams& p, const MmaEnv& v) {
  constexpr int NM = R > 0 ? R * S * (GPS / 2) : 1;
  const uint32_t strip16 = p.strip_pix;  // channel-group stride of the A strips (16-B units)
  const uint32_t blbo16 = p.block_n_tot;
  // the planner keeps block_n_tot <= 256: one MMA spans the N tile
  const uint32_t idesc = DT == DT_I8 ? make_idesc_i8(static_cast<uint32_t>(p.block_n_tot))
                                     : make_idesc_f16(static_cast<uint32_t>(p.block_n_tot), DT == DT_BF16);
  uint32_t aoff[NM], boff[NM];
  if (R > 0) {
    constexpr int NPH_W = S < SW ? S : SW;
#pragma unroll
    for (int r = 0; r < (R > 0 ? R : 1); ++r)
#pragma unroll
      for (int s = 0; s < (R > 0 ? S : 1); ++s)
#pragma unroll
        for (int g = 0; g < (R > 0 ? GPS : 2); g += 2) {
          const int i = (r * S + s) * (GPS / 2) + g / 2;
          aoff[i] = static_cast<uint32_t>(((r % SH) * NPH_W + (s % SW)) * GPS + g) * strip16 +
                    static_cast<uint32_t>(r / SH) * static_cast<uint32_t>(p.Wl) + static_cast<uint32_t>(s / SW);
          boff[i] = static_cast<uint32_t>((r * S + s) * GPS + g) * blbo16;
        }
  }
  long long tr_first = 0, tr_last = 0, tr_full = 0, tr_empty = 0;  // diagnostics (registers)
  if (v.n_units > 0) {
    if (p.b_resident) mbar_wait(v.bres, 0);
    int stage = 0;
    uint32_t phase = 0;
    for (int u = 0; u < v.n_units; ++u) {
      const int as = u % v.n_acc;
      const uint32_t aphase = static_cast<uint32_t>(u / v.n_acc) & 1u;
      if (dbg_of(p) & 8) {
      } else if (v.trace) {
        const long long w0 = clock64();
        mbar_wait(&v.tempty[as], aphase ^ 1u);
        tr_empty += clock64() - w0;
      } else {
        mbar_wait(&v.tempty[as], aphase ^ 1u);
      }
      tc_fence_after();
      const uint32_t d_tmem = v.tmem_base + as * v.acc_cols;
      for (int ks = 0; ks < p.k_stages; ++ks) {
        if (v.trace) {
          const long long w0 = clock64();
          mbar_wait(&v.full[stage], phase);
          const long long w1 = clock64();
          if (u == 0 && ks == 0) {
            tr_first = w1 - v.t_entry;
            uint64_t gt_;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(gt_));
            if (v.lane == 0) v.trace[17] = static_cast<int64_t>(gt_);
          }
          tr_full += w1 - w0;
        } else {
          mbar_wait(&v.full[stage], phase);
        }
        tc_fence_after();
        const uint64_t a0 = make_sdesc(smem_u32(v.sA + stage * v.a_stage_bytes), strip16 * 16u, 128u);
        const uint64_t b0 = make_sdesc(
            smem_u32(p.b_resident ? v.sB + ks * p.b_stage_bytes : v.sB + stage * p.b_stage_bytes), blbo16 * 16u, 128u);
        // the 14-bit start-address field never carries out of the low word
        const uint32_t a_lo = static_cast<uint32_t>(a0), a_hi = static_cast<uint32_t>(a0 >> 32);
        const uint32_t b_lo = static_cast<uint32_t>(b0), b_hi = static_cast<uint32_t>(b0 >> 32);
        uint32_t accum = ks > 0 ? 1u : 0u;
        if (R > 0) {
#pragma unroll
          for (int i = 0; i < NM; ++i)
            issue_one<DT>(d_tmem, a_hi, b_hi, a_lo + aoff[i], b_lo + boff[i], idesc, i > 0 ? 1u : accum);
        } else {
          const uint32_t ph_row = static_cast<uint32_t>(p.nph_w * p.gps) * strip16;
          const uint32_t ph_col = static_cast<uint32_t>(p.gps) * strip16;
          uint32_t bo = b_lo;
          uint32_t r_ph = 0, r_q = 0;
          for (int r = 0; r < p.R; ++r) {
            const uint32_t roff = a_lo + r_ph * ph_row + r_q * static_cast<uint32_t>(p.Wl);
            uint32_t s_ph = 0, s_q = 0;
            for (int sc = 0; sc < p.S; ++sc) {
              const uint32_t ao = roff + s_ph * ph_col + s_q;
              for (int g = 0; g < p.gps; g += 2) {
                issue_one<DT>(d_tmem, a_hi, b_hi, ao + g * strip16, bo + g * blbo16, idesc, accum);
                accum = 1u;
              }
              bo += static_cast<uint32_t>(p.gps) * blbo16;
              if (++s_ph == static_cast<uint32_t>(p.sw)) {
                s_ph = 0;
                ++s_q;
              }
            }
            if (++r_ph == static_cast<uint32_t>(p.sh)) {
              r_ph = 0;
              ++r_q;
            }
          }
        }
        mma_commit_w(&v.empty[stage]);
        if (++stage == p.n_stages) {
          stage = 0;
          phase ^= 1u;
        }
      }
      if (!(dbg_of(p) & 8) || u >= v.n_units - 2) mma_commit_w(&v.tfull[as]);
      if (v.trace && u == v.n_units - 1) {
        tr_last = clock64() - v.t_entry;
        uint64_t gt_;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(gt_));
        if (v.lane == 0) v.trace[18] = static_cast<int64_t>(gt_);
      }
    }
  }
  if (v.trace && v.lane == 0) {
    v.trace[3] = tr_first;
    v.trace[4] = tr_last;
    v.trace[9] = tr_full;
    v.trace[13] = tr_empty;
  }
}

// int8 FR pass body: items first, first + stride, ... of (plane, pixel, image
// split); per item the NDIG balanced base-256 digit planes of G for the pixel are
// loaded once and dotted (dp4a) with the pixel's 16 channels of every image of
// the split, DEPTH image loads in flight.  NDIG = 2 when every third digit of the
// plan's G is zero (8 instead of 12 dp4a per 16-byte chunk; exact either way).
template <int DEPTH, int NDIG>
__device__ __forceinline__ void fic_rhs_fr_i8(const ConvTcParams& p, int64_t first, int64_t stride, long long& acc) {
  const int64_t HlWl = static_cast<int64_t>(p.Hl) * p.Wl;
  const int nsplit = p.rhs_nsplit;
  const int64_t total = static_cast<int64_t>(p.n_phase) * p.c16 * HlWl * nsplit;
  for (int64_t idx = first; idx < total; idx += stride) {
    const int64_t pix = idx % HlWl;
    const int64_t rest = idx / HlWl;
    const int split = static_cast<int>(rest % nsplit);
    const int64_t plane = rest / nsplit;
    const uint4* gw = reinterpret_cast<const uint4*>(p.ficw8) + (plane * HlWl + pix) * 3;
    const uint4 g0 = __ldg(gw), g1 = __ldg(gw + 1);
    const uint4 g2 = NDIG == 3 ? __ldg(gw + 2) : make_uint4(0u, 0u, 0u, 0u);
    const uint4* src = reinterpret_cast<const uint4*>(p.act) + plane * p.plane_len + pix;
    const int n0 = static_cast<int>(static_cast<int64_t>(p.N) * split / nsplit);
    const int n1 = static_cast<int>(static_cast<int64_t>(p.N) * (split + 1) / nsplit);
    int32_t d0 = 0, d1 = 0, d2 = 0;  // |sum| <= 32 images * 16 * 128 * 128 < 2^31
    for (int n = n0; n < n1; n += DEPTH) {  // DEPTH image loads in flight
      uint4 x[DEPTH];
#pragma unroll
      for (int j = 0; j < DEPTH; ++j)
        x[j] = n + j < n1 ? __ldcg(src + static_cast<int64_t>(n + j) * HlWl) : make_uint4(0u, 0u, 0u, 0u);
#pragma unroll
      for (int j = 0; j < DEPTH; ++j) {
        d0 = __dp4a(static_cast<int>(x[j].x), static_cast<int>(g0.x), d0);
        d0 = __dp4a(static_cast<int>(x[j].y), static_cast<int>(g0.y), d0);
        d0 = __dp4a(static_cast<int>(x[j].z), static_cast<int>(g0.z), d0);
        d0 = __dp4a(static_cast<int>(x[j].w), static_cast<int>(g0.w), d0);
        d1 = __dp4a(static_cast<int>(x[j].x), static_cast<int>(g1.x), d1);
        d1 = __dp4a(static_cast<int>(x[j].y), static_cast<int>(g1.y), d1);
        d1 = __dp4a(static_cast<int>(x[j].z), static_cast<int>(g1.z), d1);
        d1 = __dp4a(static_cast<int>(x[j].w), static_cast<int>(g1.w), d1);
        if (NDIG == 3) {
          d2 = __dp4a(static_cast<int>(x[j].x), static_cast<int>(g2.x), d2);
          d2 = __dp4a(static_cast<int>(x[j].y), static_cast<int>(g2.y), d2);
          d2 = __dp4a(static_cast<int>(x[j].z), static_cast<int>(g2.z), d2);
          d2 = __dp4a(static_cast<int>(x[j].w), static_cast<int>(g2.w), d2);
        }
      }
      if (((n - n0) & 31) == 32 - DEPTH) {  // keep the digit sums inside int32
        acc += static_cast<long long>(d0) + (static_cast<long long>(d1) << 8) + (static_cast<long long>(d2) << 16);
        d0 = d1 = d2 = 0;
      }
    }
    acc += static_cast<long long>(d0) + (static_cast<long long>(d1) << 8) + (static_cast<long long>(d2) << 16);
  }
}

// FIC rhs, FR option: sum over the stored input of x * G (checksum.hpp:248-285
// gen_input_checksum + fic_dot restated as one pass), work items
// first, first + stride, ... of (plane, pixel, image split).  int8: G as three
// balanced base-256 digit planes, 12 dp4a per 16-byte chunk, every image load of
// an item issued before use.  float mode: G in f32, f32 FMAs per item, f64 across
// items (input_checksum_f64 / fic_dot_f64, checksum.hpp:496-535).  Run by the conv
// CTAs' input-checksum warps, or by all warps of the extra input-checksum CTAs
// that fill the SMs a small conv grid leaves idle.
template <int DT, int DEPTH = 8>
__device__ __forceinline__ void fic_rhs_fr(const ConvTcParams& p, int64_t first, int64_t stride, long long& acc,
                                           double& facc_rhs) {
  if constexpr (DT != DT_I8) {
    const int64_t HlWl = static_cast<int64_t>(p.Hl) * p.Wl;
    const int nsplit = p.rhs_nsplit;
    const int64_t total = static_cast<int64_t>(p.n_phase) * p.c16 * HlWl * nsplit;
    for (int64_t idx = first; idx < total; idx += stride) {
      const int64_t pix = idx % HlWl;
      const int64_t rest = idx / HlWl;
      const int split = static_cast<int>(rest % nsplit);
      const int64_t plane = rest / nsplit;
      const float4* gw = reinterpret_cast<const float4*>(p.ficwf) + (plane * HlWl + pix) * 2;
      const float4 ga = __ldg(gw), gb = __ldg(gw + 1);
      const uint4* src = reinterpret_cast<const uint4*>(p.act) + plane * p.plane_len + pix;
      const int n0 = static_cast<int>(static_cast<int64_t>(p.N) * split / nsplit);
      const int n1 = static_cast<int>(static_cast<int64_t>(p.N) * (split + 1) / nsplit);
      // DEPTH image loads in flight and four independent FMA chains: with one
      // chain and four loads the two input-checksum warps of a busy SM moved
      // ~1.6 TB/s machine-wide (VGG-16 conv1_2: the re-read took longer than the conv)
      constexpr int kD = DEPTH < 8 ? 8 : DEPTH;
      float acc4[4] = {0.0f, 0.0f, 0.0f, 0.0f};
      for (int n = n0; n < n1; n += kD) {
        uint4 x[kD];
#pragma unroll
        for (int j = 0; j < kD; ++j)
          x[j] = n + j < n1 ? __ldcg(src + static_cast<int64_t>(n + j) * HlWl) : make_uint4(0u, 0u, 0u, 0u);
#pragma unroll
        for (int j = 0; j < kD; ++j) {
          const float2 x0 = unpack_h2<DT>(x[j].x), x1 = unpack_h2<DT>(x[j].y), x2 = unpack_h2<DT>(x[j].z),
                       x3 = unpack_h2<DT>(x[j].w);
          float& a = acc4[j & 3];
          a = __fmaf_rn(x0.x, ga.x, a);
          a = __fmaf_rn(x0.y, ga.y, a);
          a = __fmaf_rn(x1.x, ga.z, a);
          a = __fmaf_rn(x1.y, ga.w, a);
          a = __fmaf_rn(x2.x, gb.x, a);
          a = __fmaf_rn(x2.y, gb.y, a);
          a = __fmaf_rn(x3.x, gb.z, a);
          a = __fmaf_rn(x3.y, gb.w, a);
        }
      }
      const float item = (acc4[0] + acc4[1]) + (acc4[2] + acc4[3]);
      facc_rhs += static_cast<double>(item);
    }
  } else {
    if (p.g_ndig == 2)
      fic_rhs_fr_i8<DEPTH, 2>(p, first, stride, acc);
    else
      fic_rhs_fr_i8<DEPTH, 3>(p, first, stride, acc);
  }
}

// FR input-checksum items of this CTA (the same set fic_rhs_fr's static stride
// gives its two input-checksum warps), claimed 32 at a time from a shared-memory
// counter, so warps that have finished their own role -- producer, MMA issuer,
// epilogue after its last unit -- take over part of the input-checksum tail.
template <int DT>
__device__ __forceinline__ void fr_claim_loop(const ConvTcParams& p, int* s_claim, int lane, long long& acc,
                                              double& facc) {
  const int64_t HlWl = static_cast<int64_t>(p.Hl) * p.Wl;
  const int64_t total = static_cast<int64_t>(p.n_phase) * p.c16 * HlWl * p.rhs_nsplit;
  const int64_t stride = static_cast<int64_t>(p.conv_grid) * (kRhsWarps * 32);
  const int64_t base0 = static_cast<int64_t>(blockIdx.x) * (kRhsWarps * 32);
  for (;;) {
    int c = 0;
    if (lane == 0) c = atomicAdd(s_claim, 1);
    c = __shfl_sync(0xffffffffu, c, 0);
    const int64_t idx0 = base0 + (c & 1) * 32 + static_cast<int64_t>(c >> 1) * stride;
    if (idx0 >= total) break;
    if (DT != DT_I8 || p.rhs_deep)
      fic_rhs_fr<DT, 16>(p, idx0 + lane, int64_t(1) << 62, acc, facc);
    else
      fic_rhs_fr<DT, 8>(p, idx0 + lane, int64_t(1) << 62, acc, facc);
  }
}

// ICBatch writer (ic_batch_checksum, checksum.hpp:350-362, fused): cells
// first, first + stride, ... of (plane, pixel) of the packed input; per cell the
// 16 channel bytes are summed over the N images (x ^ 0x80 = x + 128 as unsigned
// bytes, even / odd bytes in 16-bit lanes, flushed every 128 images) and the sum
// s in [-128 N, 127 N] is stored as icb_d balanced base-256 digit images after
// the real ones (digit image j at M-space image N + j), so the tensor-core conv of
// those rows gives conv(d_j) exactly and sum_j 256^j conv(d_j) = conv_batch_checksum.
// Then one release increment of icb_ready per warp (the producers of tiles that
// reach the digit images wait for every writer warp).
__device__ __forceinline__ void icb_write_digits(const ConvTcParams& p, int64_t first, int64_t stride) {
  const int64_t HlWl = static_cast<int64_t>(p.Hl) * p.Wl;
  const int64_t cells = static_cast<int64_t>(p.n_phase) * p.c16 * HlWl;
  for (int64_t idx = first; idx < cells; idx += stride) {
    const int64_t plane = idx / HlWl, pix = idx - plane * HlWl;
    const uint4* src = reinterpret_cast<const uint4*>(p.act) + plane * p.plane_len + pix;
    int32_t s[16];
#pragma unroll
    for (int e = 0; e < 16; ++e) s[e] = 0;
    for (int n0 = 0; n0 < p.N; n0 += 128) {
      const int n1 = n0 + 128 < p.N ? n0 + 128 : p.N;
      uint32_t lo[4] = {0u, 0u, 0u, 0u}, hi[4] = {0u, 0u, 0u, 0u};
      for (int n = n0; n < n1; n += 8) {
        uint4 x[8];
#pragma unroll
        for (int j = 0; j < 8; ++j)
          x[j] = n + j < n1 ? __ldcg(src + static_cast<int64_t>(n + j) * HlWl) : make_uint4(0x80808080u, 0x80808080u,
                                                                                             0x80808080u, 0x80808080u);
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const uint32_t w[4] = {x[j].x ^ 0x80808080u, x[j].y ^ 0x80808080u, x[j].z ^ 0x80808080u,
                                 x[j].w ^ 0x80808080u};
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            lo[q] += w[q] & 0x00FF00FFu;
            hi[q] += (w[q] >> 8) & 0x00FF00FFu;
          }
        }
      }
      // padded slots added 0x80 ^ 0x80 = 0; real ones x + 128
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        s[4 * q + 0] += static_cast<int32_t>(lo[q] & 0xFFFFu);
        s[4 * q + 2] += static_cast<int32_t>(lo[q] >> 16);
        s[4 * q + 1] += static_cast<int32_t>(hi[q] & 0xFFFFu);
        s[4 * q + 3] += static_cast<int32_t>(hi[q] >> 16);
      }
    }
    uint32_t dw[3][4];
#pragma unroll
    for (int q = 0; q < 4; ++q) dw[0][q] = dw[1][q] = dw[2][q] = 0u;
#pragma unroll
    for (int e = 0; e < 16; ++e) {
      int32_t v = s[e] - 128 * p.N;
#pragma unroll
      for (int d = 0; d < 3; ++d) {
        const int32_t dg = d < 2 ? ((v + 128) & 0xFF) - 128 : v;  // the last digit takes the rest (|v| <= 128)
        v = (v - dg) >> 8;                                         // exact: v - dg is a multiple of 256
        dw[d][e >> 2] |= (static_cast<uint32_t>(dg) & 0xFFu) << (8 * (e & 3));
      }
    }
    uint4* dst = reinterpret_cast<uint4*>(const_cast<int8_t*>(p.act)) + plane * p.plane_len +
                 static_cast<int64_t>(p.N) * HlWl + pix;
#pragma unroll
    for (int d = 0; d < 3; ++d)
      if (d < p.icb_d) dst[static_cast<int64_t>(d) * HlWl] = make_uint4(dw[d][0], dw[d][1], dw[d][2], dw[d][3]);
  }
  __threadfence();
  __syncwarp();
  if ((threadIdx.x & 31) == 0) red_release_gpu_add(p.icb_ready, 1u);
}

// IC input checksum, FR option (rhs_mode 4): items first, first + stride, ... of
// (plane, pixel, image split); per item the 16 channel bytes summed over the
// split's images (biased bytes in 16-bit lanes, flushed every 128 images), added
// into the class sums ic_S[phase][row class][column class][channel] (integer
// reductions: deterministic).  A plane pixel's position class fixes which taps
// (r, s) it feeds, so gen_input_checksum's ic[c,r,s] (checksum.hpp:248-266) is a
// sum of class sums (ic_from_classes_kernel, at the verdict).
__device__ __forceinline__ void ic_class_sums_fr(const ConvTcParams& p, int64_t first, int64_t stride) {
  const int64_t HlWl = static_cast<int64_t>(p.Hl) * p.Wl;
  const int nsplit = p.rhs_nsplit;
  const int64_t total = static_cast<int64_t>(p.n_phase) * p.c16 * HlWl * nsplit;
  const int c256 = p.c16 * 16;
  // warp-uniform loop (the aggregation below shuffles): lanes past the end idle
  for (int64_t base = first - (threadIdx.x & 31); base < total; base += stride) {
    const int64_t idx = base + (threadIdx.x & 31);
    const bool ok = idx < total;
    const int64_t it = ok ? idx : 0;
    const int64_t pix = it % HlWl;
    const int64_t rest = it / HlWl;
    const int split = static_cast<int>(rest % nsplit);
    const int64_t plane = rest / nsplit;
    const int phase = static_cast<int>(plane / p.c16), grp = static_cast<int>(plane % p.c16);
    const int i = static_cast<int>(pix / p.Wl), j = static_cast<int>(pix % p.Wl);
    const int a = phase / p.nph_w, b = phase - (phase / p.nph_w) * p.nph_w;
    const int cell = (phase * p.ic_nrc + p.ic_rowcls[a * p.Hl + i]) * p.ic_ncc + p.ic_colcls[b * p.Wl + j];
    const uint4* src = reinterpret_cast<const uint4*>(p.act) + plane * p.plane_len + pix;
    const int n0 = ok ? static_cast<int>(static_cast<int64_t>(p.N) * split / nsplit) : 0;
    const int n1 = ok ? static_cast<int>(static_cast<int64_t>(p.N) * (split + 1) / nsplit) : 0;
    int32_t s[16];
#pragma unroll
    for (int e = 0; e < 16; ++e) s[e] = 0;
    for (int m0 = n0; m0 < n1; m0 += 128) {
      const int m1 = m0 + 128 < n1 ? m0 + 128 : n1;
      uint32_t lo[4] = {0u, 0u, 0u, 0u}, hi[4] = {0u, 0u, 0u, 0u};
      for (int n = m0; n < m1; n += 8) {
        uint4 x[8];
#pragma unroll
        for (int q = 0; q < 8; ++q)
          x[q] = n + q < m1 ? __ldcg(src + static_cast<int64_t>(n + q) * HlWl)
                            : make_uint4(0x80808080u, 0x80808080u, 0x80808080u, 0x80808080u);
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          const uint32_t w[4] = {x[q].x ^ 0x80808080u, x[q].y ^ 0x80808080u, x[q].z ^ 0x80808080u,
                                 x[q].w ^ 0x80808080u};
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            lo[u] += w[u] & 0x00FF00FFu;
            hi[u] += (w[u] >> 8) & 0x00FF00FFu;
          }
        }
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        s[4 * u + 0] += static_cast<int32_t>(lo[u] & 0xFFFFu);
        s[4 * u + 2] += static_cast<int32_t>(lo[u] >> 16);
        s[4 * u + 1] += static_cast<int32_t>(hi[u] & 0xFFFFu);
        s[4 * u + 3] += static_cast<int32_t>(hi[u] >> 16);
      }
    }
    // warp aggregation: interior pixels share one class, so per-lane L2
    // reductions on the same addresses serialise.  The warp's lanes are split
    // into groups of equal (class, channel group) -- a row edge gives 2-4 groups
    // -- and each group's 16 channel sums are reduced across the warp (int32
    // transpose-reduce, |sum| <= 32 * 128 * N) into one reduction per channel.
    const int lane = threadIdx.x & 31;
    const int key = ok ? cell * 4096 + grp : -1;
    unsigned long long* dst = reinterpret_cast<unsigned long long*>(p.ic_S) +
                              static_cast<int64_t>(ok ? cell : 0) * c256 + (ok ? grp : 0) * 16;
    int32_t v[16];
#pragma unroll
    for (int e = 0; e < 16; ++e) v[e] = ok ? s[e] - 128 * (n1 - n0) : 0;
    const bool b4 = lane & 16, b3 = lane & 8, b2 = lane & 4, b1 = lane & 2;
    const int ch = (b4 ? 8 : 0) + (b3 ? 4 : 0) + (b2 ? 2 : 0) + (b1 ? 1 : 0);
    unsigned remaining = __ballot_sync(0xffffffffu, ok);
    while (remaining) {
      const int leader = __ffs(remaining) - 1;
      const int lkey = __shfl_sync(0xffffffffu, key, leader);
      const bool mine = ok && key == lkey;
      remaining &= ~__ballot_sync(0xffffffffu, mine);
      int32_t w8[8], w4[4], w2[2];
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        const int32_t lo = mine ? v[e] : 0, hi = mine ? v[e + 8] : 0;
        w8[e] = (b4 ? hi : lo) + __shfl_xor_sync(0xffffffffu, b4 ? lo : hi, 16);
      }
#pragma unroll
      for (int e = 0; e < 4; ++e) w4[e] = (b3 ? w8[e + 4] : w8[e]) + __shfl_xor_sync(0xffffffffu, b3 ? w8[e] : w8[e + 4], 8);
#pragma unroll
      for (int e = 0; e < 2; ++e) w2[e] = (b2 ? w4[e + 2] : w4[e]) + __shfl_xor_sync(0xffffffffu, b2 ? w4[e] : w4[e + 2], 4);
      int32_t w1 = (b1 ? w2[1] : w2[0]) + __shfl_xor_sync(0xffffffffu, b1 ? w2[0] : w2[1], 2);
      w1 += __shfl_xor_sync(0xffffffffu, w1, 1);
      unsigned long long* d0 =
          reinterpret_cast<unsigned long long*>(__shfl_sync(0xffffffffu, reinterpret_cast<uintptr_t>(dst), leader));
      if (!(lane & 1) && w1 != 0) red_add_u64(d0 + ch, static_cast<unsigned long long>(static_cast<long long>(w1)));
    }
  }
}

// producer side: every digit writer warp of the grid has released its stores
__device__ __forceinline__ void icb_wait_ready(const ConvTcParams& p) {
  while (ld_acquire_gpu(p.icb_ready) < p.icb_writers) __nanosleep(64);
  fence_proxy_async_global();  // the bulk copies (async proxy) now see them
}

// pattern ids (host: mma_pattern_of in plan.cu)
enum MmaPattern : int {
  PAT_GENERIC = 0,
  PAT_3x3_S1_G4 = 1, PAT_3x3_S1_G2 = 2, PAT_3x3_S2_G4 = 3, PAT_3x3_S2_G2 = 4,
  PAT_1x1_S1_G4 = 5, PAT_1x1_S1_G2 = 6, PAT_1x1_S2_G4 = 7, PAT_1x1_S2_G2 = 8,
};

template <int DT, int EPI, bool FC, bool FIC, int XT>
__global__ void __launch_bounds__(kConvThreads, 1) conv_i8_tc_kernel(const __grid_constant__ ConvTcParams p) {
  using Acc = std::conditional_t<DT == DT_I8, int64_t, double>;  // exact int / f64 float-mode sums
  extern __shared__ __align__(128) uint8_t smem[];
  const SmemLayout L = smem_layout(p);
  uint8_t* sA = smem + L.a_off;
  uint8_t* sB = smem + L.b_off;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L.bar_off);
  uint64_t* full = bars;
  uint64_t* empty = bars + kStages;
  uint64_t* tfull = bars + 2 * kStages;
  uint64_t* tempty = bars + 2 * kStages + kMaxAcc;
  uint64_t* bres = bars + 2 * kStages + 2 * kMaxAcc;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * kStages + 2 * kMaxAcc + 1);
  __shared__ __align__(16) float s_bias[kBiasSmem];
  __shared__ FcRec s_fc[kEpiWarps];
  __shared__ long long s_lhs[kEpiWarps];
  __shared__ int64_t s_rowsum[kEpiParts - 1][kBlockM];
  __shared__ int s_tile_last;

  // warp index through a shuffle: provably warp-uniform, so ptxas keeps the
  // role branches convergent and the MMA descriptors in uniform registers
  const int warp = __shfl_sync(0xffffffffu, static_cast<int>(threadIdx.x >> 5), 0);
  const int lane = threadIdx.x & 31;

  if (static_cast<int>(blockIdx.x) >= p.conv_grid) {
    // ------------------------------------------------ input-checksum CTA
    // an SM the conv grid leaves idle: every warp works on the FR input checksum
    pdl_launch_dependents();
    long long acc = 0;
    double facc_rhs = 0.0;
    pdl_wait();
    if (DT == DT_I8 && XT == 2 && p.icb_d) {
      const int64_t writers = static_cast<int64_t>(p.conv_grid) * (kRhsWarps * 32) +
                              static_cast<int64_t>(p.ic_ctas) * kConvThreads;
      icb_write_digits(p, static_cast<int64_t>(p.conv_grid) * (kRhsWarps * 32) +
                              static_cast<int64_t>(blockIdx.x - p.conv_grid) * kConvThreads + threadIdx.x, writers);
    }
    if (DT == DT_I8 && XT == 1 && p.rhs_mode == 4)
      ic_class_sums_fr(p, static_cast<int64_t>(blockIdx.x - p.conv_grid) * kConvThreads + threadIdx.x,
                       static_cast<int64_t>(p.ic_ctas) * kConvThreads);
    if (FIC && p.rhs_mode == 1)
      fic_rhs_fr<DT, 16>(p, static_cast<int64_t>(blockIdx.x - p.conv_grid) * kConvThreads + threadIdx.x,
                     static_cast<int64_t>(p.ic_ctas) * kConvThreads, acc, facc_rhs);
    __shared__ long long s_ic[kConvThreads / 32];
    if (FIC) {
      const long long w = DT == DT_I8 ? warp_sum(acc) : __double_as_longlong(warp_sum_d(facc_rhs));
      if (lane == 0) s_ic[warp] = w;
    }
    __syncthreads();
    if ((FC || FIC) && threadIdx.x == 0) {
      int64_t* rec = p.cta_rec + static_cast<int64_t>(blockIdx.x) * kCtaRec;
      rec[0] = 0;       // no FC rows here
      rec[1] = kNoKey;
      rec[2] = rec[3] = 0;
      long long r = 0;
      double rf = 0.0;
      for (int w = 0; w < kConvThreads / 32; ++w) {
        r += s_ic[w];
        rf += __longlong_as_double(s_ic[w]);
      }
      rec[4] = DT == DT_I8 ? 0ll : __double_as_longlong(0.0);
      rec[5] = DT == DT_I8 ? r : __double_as_longlong(rf);
    }
    return;
  }
  int64_t* const trace = p.trace ? p.trace + static_cast<int64_t>(blockIdx.x) * kTraceSlots : nullptr;
  const long long t_entry = clock64();
  if (trace && threadIdx.x == 0) {
    uint64_t gt;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(gt));
    trace[0] = static_cast<int64_t>(gt);
    trace[1] = t_entry;
  }

  // accumulator stages: columns per stage (multiple of 32), 2 stages when they fit.
  // Narrow int8 tiles (<= 64 output channels: ResNet-50 layer1 class) interleave
  // units across the epilogue warps of a lane quarter instead of splitting the
  // columns: each warp drains whole units (all channels of its 32 rows), the
  // kEpiParts warps of a quarter take alternate units, so two units' tcgen05.ld
  // latency and requantise overlap; kEpiParts + 1 .. 2 * kEpiParts stages keep
  // the MMA warp fed.
  // (Splitting 64 columns over 2 warps left each warp one 32-column load per unit
  // with its latency fully exposed: the epilogue set the pace at ~2.1K cycles/unit;
  // layer1 b1024 FIC 244 -> 182 us, b32 12.5 -> 11.1 us.  For 128-column tiles the
  // interleave measured no gain at b1024 and a loss at b32, so they keep the split.)
  const int acc_cols = (p.block_n_tot + 31) & ~31;
  const bool alt = DT == DT_I8 && p.block_n <= 64 && (kEpiParts + 1) * acc_cols <= 512 && !(dbg_of(p) & 512);
  const int n_acc = alt ? min(kMaxAcc, 512 / acc_cols) : (2 * acc_cols <= 512) ? 2 : 1;
  uint32_t tmem_cols = 32;
  while (tmem_cols < static_cast<uint32_t>(n_acc * acc_cols)) tmem_cols <<= 1;

  // FIC-SM: the input-checksum warps read every A stage too, so a stage is free
  // once the MMA commit and each of them have arrived
  const bool rhs_staged = DT == DT_I8 && FIC && XT == 4 && p.rhs_mode == 3;
  if (threadIdx.x == 0) {
    for (int i = 0; i < kStages; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], rhs_staged ? 1 + kRhsWarps : 1);
    }
    for (int i = 0; i < n_acc; ++i) {
      mbar_init(&tfull[i], 1);
      mbar_init(&tempty[i], alt ? 4 : kEpiWarps);  // alt: one warp per lane quarter drains a unit
    }
    mbar_init(bres, 1);
    if (rhs_staged) mbar_init(reinterpret_cast<uint64_t*>(smem + L.fic_off + p.fic_smem), 1);
    fence_mbar_init();
  }
  __shared__ int s_fr_claim;
  __shared__ long long s_rhs_all[kConvThreads / 32];
  unsigned long long* const s_ic = (XT == 1 && p.ic_smem) ? reinterpret_cast<unsigned long long*>(smem + L.ic_off) : nullptr;
  if (s_ic)
    for (int i = threadIdx.x; i < p.K; i += kConvThreads) s_ic[i] = 0ull;
  if (threadIdx.x == 0) s_fr_claim = 0;
  if (threadIdx.x < kConvThreads / 32) s_rhs_all[threadIdx.x] = 0;
  if (warp == 1) tmem_alloc(tmem_slot, tmem_cols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  // FR input checksum shared by every warp that has finished its role (dbg 256: off)
  // float mode only: on int8 layers the claims of the producer / MMA warps slowed the
  // epilogue-bound CTAs (ResNet-50 layer1 FIC 12.3 -> 13.4 us); VGG-16 FP16 FIC 18% -> 11%
  const bool fr_share = DT != DT_I8 && FIC && p.rhs_mode == 1 && p.ic_ctas == 0 && !(dbg_of(p) & 256);
  long long fr_acc = 0;
  double fr_facc = 0.0;
  if (trace && threadIdx.x == 0) trace[2] = clock64() - t_entry;
  pdl_launch_dependents();

  // number of work units for this CTA
  int n_units;
  if (p.b_resident) {
    const int per = p.conv_grid / p.n_tiles;
    const int mt0 = blockIdx.x / p.n_tiles;
    n_units = (static_cast<int>(blockIdx.x) < per * p.n_tiles && mt0 < p.m_tiles) ? (p.m_tiles - mt0 + per - 1) / per : 0;
  } else {
    const int total = p.m_tiles * p.n_tiles;
    n_units = static_cast<int>(blockIdx.x) < total ? (total - blockIdx.x + p.conv_grid - 1) / p.conv_grid : 0;
  }

  if (warp == 0) {
    // ------------------------------------------------------------ producer
    // warp-uniform loop; one elected lane issues each copy (ptx.cuh *_w)
    if (n_units > 0) {
      const uint64_t pol_b = policy_evict_last();
      if (p.b_resident) {
        // filters are plan-owned and immutable: prefetch before the PDL wait
        const int nt = blockIdx.x % p.n_tiles;
        const uint32_t bytes = p.b_stage_bytes * p.k_stages;
        mbar_arrive_expect_tx_w(bres, bytes);
        const int8_t* src = p.wpk + static_cast<int64_t>(nt) * p.k_stages * p.b_stage_bytes;
        for (uint32_t o = 0; o < bytes; o += 65536u) {
          const uint32_t sz = (bytes - o) < 65536u ? (bytes - o) : 65536u;
          bulk_g2s_evict_last_w(sB + o, src + o, sz, bres, pol_b);
        }
      }
      const uint32_t strip_bytes = p.strip_pix * 16u;
      const uint32_t bytes = L.a_stage_bytes + (p.b_resident ? 0u : p.b_stage_bytes);
      // streamed filters: the first ring fill's B blocks do not depend on the
      // previous kernel either, so they are requested before the PDL wait too
      const int total_stages = n_units * p.k_stages;
      const int pre = p.b_resident ? 0 : (total_stages < p.n_stages ? total_stages : p.n_stages);
      for (int i = 0; i < pre; ++i) {
        int mt, nt;
        decode_tile(p, i / p.k_stages, mt, nt);
        const int ks = i % p.k_stages;
        mbar_arrive_expect_tx_w(&full[i], bytes);
        const int8_t* src = p.wpk + (static_cast<int64_t>(nt) * p.k_stages + ks) * p.b_stage_bytes;
        bulk_g2s_evict_last_w(sB + i * p.b_stage_bytes, src, p.b_stage_bytes, &full[i], pol_b);
      }
      pdl_wait();
      int stage = 0;
      uint32_t phase = 0;
      if (trace && lane == 0) {
        trace[8] = clock64() - t_entry;
        uint64_t gt_;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(gt_));
        trace[16] = static_cast<int64_t>(gt_);
      }
      bool icb_seen = false;
      for (int u = 0; u < n_units; ++u) {
        int mt, nt;
        decode_tile(p, u, mt, nt);
        const int64_t m0 = static_cast<int64_t>(mt) * kBlockM;
        if (DT == DT_I8 && XT == 2 && p.icb_d && !icb_seen && m0 + p.strip_pix > p.m_real) {
          icb_wait_ready(p);  // this tile's strips reach the ICBatch digit images
          icb_seen = true;
        }
        for (int ks = 0; ks < p.k_stages; ++ks) {
          const bool prefetched = u * p.k_stages + ks < pre;
          if (!prefetched) {
            mbar_wait(&empty[stage], phase ^ 1u);
            mbar_arrive_expect_tx_w(&full[stage], bytes);
          }
          uint8_t* dstA = sA + stage * L.a_stage_bytes;
          for (int ph = 0; ph < p.n_phase; ++ph) {
            for (int g = 0; g < p.gps; ++g) {
              const int64_t plane = static_cast<int64_t>(ph) * p.c16 + ks * p.gps + g;
              const int8_t* src = p.act + (plane * p.plane_len + m0) * 16;
              bulk_g2s_w(dstA + (ph * p.gps + g) * strip_bytes, src, strip_bytes, &full[stage]);
            }
          }
          if (!p.b_resident && !prefetched) {
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
    } else {
      pdl_wait();
    }
    if (fr_share) fr_claim_loop<DT>(p, &s_fr_claim, lane, fr_acc, fr_facc);
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    pdl_wait();
    MmaEnv v;
    v.sA = sA;
    v.sB = sB;
    v.a_stage_bytes = L.a_stage_bytes;
    v.full = full;
    v.empty = empty;
    v.tfull = tfull;
    v.tempty = tempty;
    v.bres = bres;
    v.tmem_base = tmem_base;
    v.acc_cols = acc_cols;
    v.n_acc = n_acc;
    v.n_units = n_units;
    v.lane = lane;
    v.trace = trace;
    v.t_entry = t_entry;
    switch (p.mma_pattern) {
      case PAT_3x3_S1_G4: mma_warp_run<DT, 3, 3, 1, 1, 4>(p, v); break;
      case PAT_3x3_S1_G2: mma_warp_run<DT, 3, 3, 1, 1, 2>(p, v); break;
      case PAT_3x3_S2_G4: mma_warp_run<DT, 3, 3, 2, 2, 4>(p, v); break;
      case PAT_3x3_S2_G2: mma_warp_run<DT, 3, 3, 2, 2, 2>(p, v); break;
      case PAT_1x1_S1_G4: mma_warp_run<DT, 1, 1, 1, 1, 4>(p, v); break;
      case PAT_1x1_S1_G2: mma_warp_run<DT, 1, 1, 1, 1, 2>(p, v); break;
      case PAT_1x1_S2_G4: mma_warp_run<DT, 1, 1, 2, 2, 4>(p, v); break;
      case PAT_1x1_S2_G2: mma_warp_run<DT, 1, 1, 2, 2, 2>(p, v); break;
      default: mma_warp_run<DT, 0, 0, 1, 1, 2>(p, v); break;
    }
    if (fr_share) fr_claim_loop<DT>(p, &s_fr_claim, lane, fr_acc, fr_facc);
  } else if (warp < 2 + kEpiWarps) {
    // ------------------------------------------------------------ epilogue
    // kEpiParts warps per TMEM lane quarter split the tile's 16-column chunks
    // into contiguous parts; every epilogue warp drains every unit.  Several
    // warps per SM sub-partition keep tcgen05.ld latency hidden behind the
    // requantise math of the others.
    const int ew = warp - 2;        // 0 .. kEpiWarps-1
    const int part = ew >> 2;       // which part of the chunks
    const int quarter = warp & 3;   // TMEM lane quarter this warp may access
    const int row = quarter * 32 + lane;
    pdl_wait();
    if (EPI != EPI_NONE && p.K <= kBiasSmem) {
      for (int i = ew * 32 + lane; i < p.K; i += kEpiThreads) s_bias[i] = p.bias[i];
    }
    named_bar(kBarEpi, kEpiThreads);
    EpiCtx e;
    e.PQ = static_cast<int64_t>(p.P) * p.Q;
    e.bias_smem = p.K <= kBiasSmem ? s_bias : nullptr;
    e.ic_acc = s_ic;
    // chunk-sum in int32 is exact when 16 * max|acc| < 2^31 (CRS < 8192)
    e.chunk32 = p.ntaps * p.c16 * 16 < 8192;
    // ConvOut fault hook target (faults.hpp:230-233), decoded once
    int64_t fk_n = -1, fk_pq = -1;
    e.fk_k = -1;
    if (p.fault_key >= 0) {
      fk_n = p.fault_key / (static_cast<int64_t>(p.K) * e.PQ);
      e.fk_k = static_cast<int>((p.fault_key / e.PQ) % p.K);
      fk_pq = p.fault_key % e.PQ;
    }
    const uint32_t HlWl = static_cast<uint32_t>(p.Hl) * p.Wl;
    FcRec fc{0, kNoKey, 0, 0};
    Acc fic_sum = 0;
    long long af_sum = 0;  // FIC-AF: this thread's share of the next layer's rhs
    e.af_row = nullptr;
    e.af_gstride = p.af_HlWl * 3;
    long long tr_wait = 0, tr_acc = 0, tr_proc = 0;  // diagnostics (registers)
    const int nch = p.block_n >> 4;  // 16-column chunks of real output channels
    // alt: this warp drains units part, part + kEpiParts, ... with all the chunks
    const int c_lo = alt ? 0 : (nch * part) / kEpiParts, c_hi = alt ? nch : (nch * (part + 1)) / kEpiParts;
    const int u_first = alt ? part : 0, u_step = alt ? kEpiParts : 1;
    // per-unit coordinates without integer division: exact float-reciprocal
    // quotients (every operand < 2^24), shifts for the 1/2-strided consumer
    const float rcp_hlwl = 1.0f / static_cast<float>(HlWl), rcp_wl = 1.0f / static_cast<float>(p.Wl);
    auto fdiv = [](uint32_t a, uint32_t d, float rcp) {
      uint32_t q = __float2uint_rz(__fmul_rz(__uint2float_rz(a), rcp));
      if (q * d > a) --q;
      else if ((q + 1u) * d <= a) ++q;
      return q;
    };
    const bool o_pow2 = (p.o_sh == 1 || p.o_sh == 2) && (p.o_sw == 1 || p.o_sw == 2);
    const int o_shh = p.o_sh == 2 ? 1 : 0, o_shw = p.o_sw == 2 ? 1 : 0;
    for (int u = u_first; u < n_units; u += u_step) {
      int mt, nt;
      decode_tile(p, u, mt, nt);
      const uint32_t m = static_cast<uint32_t>(mt) * kBlockM + row;
      uint32_t n_img = 0, pp = 0, qq = 0;
      bool valid = m < static_cast<uint64_t>(p.m_total);
      if (valid) {
        n_img = fdiv(m, HlWl, rcp_hlwl);
        const uint32_t rem = m - n_img * HlWl;
        pp = fdiv(rem, static_cast<uint32_t>(p.Wl), rcp_wl);
        qq = rem - pp * p.Wl;
        valid = pp < static_cast<uint32_t>(p.P) && qq < static_cast<uint32_t>(p.Q);
      }
      e.icb_lhs = nullptr;
      e.icb_dig = nullptr;
      if (DT == DT_I8 && XT == 2 && p.icb_d && valid) {
        const int64_t kq = static_cast<int64_t>(pp) * p.Q + qq;
        if (n_img >= static_cast<uint32_t>(p.N)) {  // ICBatch digit row: no output, no FC / FIC
          e.icb_dig = p.icb_dig + static_cast<int64_t>(n_img - p.N) * p.K * e.PQ + kq;
          valid = false;
        } else {
          e.icb_lhs = p.icb_lhs + kq;
        }
      }
      e.valid = valid;
      const int64_t key = static_cast<int64_t>(n_img) * e.PQ + static_cast<int64_t>(pp) * p.Q + qq;
      e.fault_row = valid && p.fault_key >= 0 && n_img == fk_n && (key - static_cast<int64_t>(n_img) * e.PQ) == fk_pq;
      if (EPI == EPI_PACKED || EPI == EPI_COMPARE) {
        const int hh = pp + p.o_ph, ww = qq + p.o_pw;
        int a_ph, b_ph, hq, wq;
        if (o_pow2) {
          a_ph = hh & o_shh;
          b_ph = ww & o_shw;
          hq = hh >> o_shh;
          wq = ww >> o_shw;
        } else {
          a_ph = hh % p.o_sh;
          b_ph = ww % p.o_sw;
          hq = hh / p.o_sh;
          wq = ww / p.o_sw;
        }
        const int64_t t = (static_cast<int64_t>(n_img) * p.o_Hl + hq) * p.o_Wl + wq;
        e.pk_row = static_cast<int8_t*>(p.out) +
                   (static_cast<int64_t>(a_ph * p.o_nph_w + b_ph) * p.o_c16 * p.o_plane_len + t) * 16;
        if (EPI == EPI_PACKED && DT == DT_I8 && XT != 0 && p.af_ficw8)
          e.af_row = reinterpret_cast<const uint4*>(p.af_ficw8) +
                     (static_cast<int64_t>(a_ph * p.o_nph_w + b_ph) * p.o_c16 * p.af_HlWl +
                      static_cast<int64_t>(hq) * p.o_Wl + wq) * 3;
      } else if (EPI == EPI_NCHW) {
        e.nchw_row = static_cast<int64_t>(n_img) * p.K * e.PQ + static_cast<int64_t>(pp) * p.Q + qq;
      }

      const int as = u % n_acc;
      const uint32_t uphase = static_cast<uint32_t>(u / n_acc) & 1u;
      if ((dbg_of(p) & 8) && u < n_units - 2) continue;
      long long t_proc = 0;
      if (trace) {
        const long long w0 = clock64();
        mbar_wait(&tfull[as], uphase);
        t_proc = clock64();
        tr_wait += t_proc - w0;
        tr_acc = t_proc - t_entry;
      } else {
        mbar_wait(&tfull[as], uphase);
      }
      tc_fence_after();
      const uint32_t t_row = tmem_base + (static_cast<uint32_t>(quarter * 32) << 16) + as * acc_cols;
      const int k_base = nt * p.block_n;
      // FC checksum digits ride in the 16 columns after the tile's channels
      uint32_t dig[4] = {0u, 0u, 0u, 0u};
      if (FC && (alt || part == 0)) tmem_ld4(t_row + p.block_n, dig);
      // fast path: no fault hook, no filler channels, no IC column sums (warp-uniform)
      const bool slow = p.fault_key >= 0 || k_base + c_hi * 16 > p.K;
      // IC column sums / ICBatch batch sums on the fast path (int8 plans only)
      constexpr int xtra = DT != DT_I8 ? 0 : XT;
      Acc row_sum = 0;
      if constexpr (xtra != 0) {
        // IC / ICBatch plans (their own kernel instances)
        if (!slow)
          row_sum = p.relu ? epi_columns<DT, EPI, true, FC || FIC, false, false, xtra>(p, e, t_row, k_base, c_lo, c_hi, af_sum)
                           : epi_columns<DT, EPI, false, FC || FIC, false, false, xtra>(p, e, t_row, k_base, c_lo, c_hi, af_sum);
        else
          row_sum = epi_columns<DT, EPI, false, FC || FIC, true, false, xtra>(p, e, t_row, k_base, c_lo, c_hi, af_sum);
      } else if (dbg_of(p) & 1) {
      } else if (dbg_of(p) & 64) {
        row_sum = epi_columns<DT, EPI, true, false, false>(p, e, t_row, k_base, c_lo, c_hi, af_sum);
      } else if (!slow && !(DT == DT_I8 && (FC || FIC) && !e.chunk32)) {
        // ONE fast copy of the drain loop per activation (int8 checked plans: int32
        // chunk sums, exact for CRS < 8192; larger CRS take the general path) --
        // every extra copy of this loop in the kernel cost instruction-cache misses
        constexpr bool kC32 = DT == DT_I8 && (FC || FIC);
        row_sum = p.relu ? epi_columns<DT, EPI, true, FC || FIC, false, kC32>(p, e, t_row, k_base, c_lo, c_hi, af_sum)
                         : epi_columns<DT, EPI, false, FC || FIC, false, kC32>(p, e, t_row, k_base, c_lo, c_hi, af_sum);
      } else if constexpr (DT == DT_I8) {
        row_sum = epi_columns<DT, EPI, false, FC || FIC, true>(p, e, t_row, k_base, c_lo, c_hi, af_sum);
      } else {
        row_sum = p.relu ? epi_columns<DT, EPI, true, FC || FIC, true>(p, e, t_row, k_base, c_lo, c_hi, af_sum)
                         : epi_columns<DT, EPI, false, FC || FIC, true>(p, e, t_row, k_base, c_lo, c_hi, af_sum);
      }
      // accumulator consumed: hand the TMEM stage back to the MMA warp
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[as]);
      if (trace) tr_proc += clock64() - t_proc;
      if (!valid) row_sum = 0;
      if (FIC) fic_sum += row_sum;
      if (FC) {
        // combine the two column halves of each row (alt: this warp has the whole row)
        if (!alt) {
          if (part > 0) s_rowsum[part - 1][row] = acc_bits(row_sum);
          named_bar(kBarQuarter0 + quarter, 32 * kEpiParts);
        }
        if (alt || part == 0) {
          if (!alt) {
#pragma unroll
            for (int q = 0; q < kEpiParts - 1; ++q) row_sum += bits_acc<Acc>(s_rowsum[q][row]);
          }
          Acc extra = 0;
          if (valid) {
            if constexpr (DT == DT_I8) {
              // checksum.hpp:179-196 recombination of the (balanced) digit columns
              extra = static_cast<int64_t>(static_cast<int32_t>(dig[0])) +
                      (static_cast<int64_t>(static_cast<int32_t>(dig[1])) << 8) +
                      (static_cast<int64_t>(static_cast<int32_t>(dig[2])) << 16);
            } else {
              // float mode: the filter checksum rides as hi + lo + lo2 split rows
              extra = static_cast<double>(__uint_as_float(dig[0])) + static_cast<double>(__uint_as_float(dig[1])) +
                      static_cast<double>(__uint_as_float(dig[2]));
            }
          }
          if (p.n_tiles == 1) {
            if (valid && fc_mismatch<DT>(row_sum, extra, p.tau_fc)) fc_note(fc, key, acc_bits(row_sum), acc_bits(extra));
          } else {
            // row partial of this N tile.  No cross-CTA hand-off: the tile's own
            // checksum rows (its share of the filter checksum) give an exact
            // per-tile check; a tile whose rows all pass cannot fail the
            // full-channel check (fc_verify, :211-236), so the CTA only raises the
            // M tile's flag, and the verdict kernel -- after the whole grid --
            // recomputes the full-channel sums of flagged tiles from these
            // partials, with the reference's semantics and loop order.
            int64_t* part = p.fc_part + (static_cast<int64_t>(nt) * p.m_tiles * kBlockM + m) * 2;
            part[0] = acc_bits(row_sum);
            part[1] = acc_bits(extra);
            if constexpr (DT == DT_I8) {
              // every (N tile, M tile, lane quarter) flag is overwritten by every
              // run, so a replayed graph never sees a stale flag
              const bool bad = valid && row_sum != extra;
              const unsigned any = __any_sync(0xffffffffu, bad) ? 1u : 0u;
              if (lane == 0) p.tile_sem[(static_cast<int64_t>(nt) * p.m_tiles + mt) * 4 + quarter] = any;
            } else {
              // float mode: per-tile differences may add up across tiles, so the
              // full-channel check stays in-kernel -- the CTA completing the M
              // tile's last N tile sums every tile's partials (fc_verify_f32,
              // :541-565); tile_sem counts tiles here
              __threadfence();
              named_bar(kBarHalf0, 128);
              if (row == 0) {
                const unsigned prev = atomicAdd(&p.tile_sem[mt], 1u);
                s_tile_last = prev == static_cast<unsigned>(p.n_tiles - 1);
              }
              named_bar(kBarHalf0, 128);
              if (s_tile_last) {
                __threadfence();
                if (valid) {
                  Acc l = 0, r = 0;
                  for (int t = 0; t < p.n_tiles; ++t) {
                    const int64_t* q = p.fc_part + (static_cast<int64_t>(t) * p.m_tiles * kBlockM + m) * 2;
                    l += bits_acc<Acc>(__ldcg(q));
                    r += bits_acc<Acc>(__ldcg(q + 1));
                  }
                  if (fc_mismatch<DT>(l, r, p.tau_fc)) fc_note(fc, key, acc_bits(l), acc_bits(r));
                }
                if (row == 0) p.tile_sem[mt] = 0u;  // ready for the next run
              }
            }
          }
        }
        // s_rowsum reuse guard for the next unit
        if (!alt) named_bar(kBarQuarter0 + quarter, 32 * kEpiParts);
      }
    }
    if (EPI == EPI_PACKED && DT == DT_I8 && XT != 0 && p.af_ficw8) {
      // FIC-AF partial of this warp straight into the next layer's accumulator
      // (fire-and-forget reduction; the next layer's verdict reads and resets it)
      const long long w = warp_sum(af_sum);
      if (lane == 0 && w != 0) atomicAdd(p.af_acc, static_cast<unsigned long long>(w));
    }
    if (trace && warp == 2 && lane == 0) {
      trace[10] = tr_wait;
      trace[11] = tr_acc;
      trace[12] = tr_proc;
    }
    if (fr_share) fr_claim_loop<DT>(p, &s_fr_claim, lane, fr_acc, fr_facc);
    // CTA-level partials of the epilogue warps
    if (FC) {
      const FcRec w = fc_warp_reduce(fc);
      if (lane == 0) s_fc[ew] = w;
    }
    if (FIC) {
      if constexpr (DT == DT_I8) {
        const long long w = warp_sum(fic_sum);
        if (lane == 0) s_lhs[ew] = w;
      } else {
        const double w = warp_sum_d(fic_sum);
        if (lane == 0) s_lhs[ew] = __double_as_longlong(w);
      }
    }
  } else {
    // ------------------------------------------------------------ input checksum
    // FIC rhs (FR option): sum over the stored input of x * G, G[plane][pix][16]
    // the offline position weights (checksum.hpp:248-285 restated as one pass).
    // G is held as three balanced base-256 digit planes, so one 16-byte input
    // chunk costs 12 dp4a; every image load of a work item is issued before use.
    const int rw = warp - (2 + kEpiWarps);
    long long acc = 0;
    double facc_rhs = 0.0;
    if (DT == DT_I8 && XT == 2 && p.icb_d) {
      // ICBatch digit images first: the producers of the last tiles wait for them
      pdl_wait();
      icb_write_digits(p, static_cast<int64_t>(blockIdx.x) * (kRhsWarps * 32) + rw * 32 + lane,
                       static_cast<int64_t>(p.conv_grid) * (kRhsWarps * 32) +
                           static_cast<int64_t>(p.ic_ctas) * kConvThreads);
    }
    if (DT != DT_I8 && FIC && p.rhs_mode == 1 && p.ic_ctas == 0) {
      pdl_wait();
      if (fr_share) {
        fr_claim_loop<DT>(p, &s_fr_claim, lane, acc, facc_rhs);
      } else {
        const int64_t first = static_cast<int64_t>(blockIdx.x) * (kRhsWarps * 32) + rw * 32 + lane;
        const int64_t stride = static_cast<int64_t>(p.conv_grid) * (kRhsWarps * 32);
        fic_rhs_fr<DT, 16>(p, first, stride, acc, facc_rhs);
      }
    } else if (rhs_staged) {
      // FIC-SM: the same sum x * G, with x taken from the A stages the producer
      // staged for the MMAs.  M tile mt owns plane pixels [m0, m0 + 128) of every
      // (phase, channel group) strip; the M tiles partition the planes, so with
      // the N-tile-0 units doing the work every stored pixel is counted once.
      // G comes from the class table (a few KB, L1 resident).
      constexpr int kIcThreads = kRhsWarps * 32;
      constexpr int kPx = kBlockM / kIcThreads;  // pixels per thread
      const int it = rw * 32 + lane;
      const uint32_t HlWl = static_cast<uint32_t>(p.Hl) * p.Wl;
      const float rcp_hlwl = 1.0f / static_cast<float>(HlWl), rcp_wl = 1.0f / static_cast<float>(p.Wl);
      const int nph_h = p.n_phase / p.nph_w;
      const int ncell = p.n_phase * p.nrc * p.ncc + 1;  // table: [group][digit][cell][16 B]; last cell = 0
      // the plan-owned class table and class arrays -> shared memory (before the
      // PDL wait: they do not depend on the previous kernel)
      uint8_t* sF = smem + L.fic_off;
      const uint4* T = reinterpret_cast<const uint4*>(sF);
      const uint8_t* sRow = sF + p.fic_tab_bytes;
      const uint8_t* sCol = sRow + ((nph_h * p.Hl + 15) & ~15);
      uint64_t* fbar = reinterpret_cast<uint64_t*>(sF + p.fic_smem);
      if (rw == 0) {
        mbar_arrive_expect_tx_w(fbar, p.fic_smem);
        bulk_g2s_w(sF, p.ficc8, p.fic_smem, fbar);
      }
      mbar_wait(fbar, 0);
      pdl_wait();
      int stage = 0;
      uint32_t sphase = 0;
      for (int u = 0; u < n_units; ++u) {
        int mt, nt;
        decode_tile(p, u, mt, nt);
        const bool own = nt == 0;
        int cell[kPx][4];  // class-table cell of each pixel per stride phase
        bool ok[kPx];
#pragma unroll
        for (int x = 0; x < kPx; ++x) {
          const uint32_t t = static_cast<uint32_t>(mt) * kBlockM + it + x * kIcThreads;
          ok[x] = own && t < static_cast<uint64_t>(p.m_real);  // real images only
          uint32_t i = 0, j = 0;
          if (ok[x]) {
            uint32_t n_img = __float2uint_rz(__fmul_rz(__uint2float_rz(t), rcp_hlwl));
            if (n_img * HlWl > t) --n_img;
            else if ((n_img + 1u) * HlWl <= t) ++n_img;
            const uint32_t rem = t - n_img * HlWl;
            i = __float2uint_rz(__fmul_rz(__uint2float_rz(rem), rcp_wl));
            if (i * p.Wl > rem) --i;
            else if ((i + 1u) * p.Wl <= rem) ++i;
            j = rem - i * p.Wl;
          }
#pragma unroll
          for (int ph = 0; ph < 4; ++ph) {
            cell[x][ph] = ncell - 1;  // zero cell: pixel outside the images (or not this CTA's)
            if (ok[x] && ph < p.n_phase) {
              const int a = ph / p.nph_w, b = ph - (ph / p.nph_w) * p.nph_w;
              const int rc = sRow[a * p.Hl + i], cc = sCol[b * p.Wl + j];
              cell[x][ph] = (ph * p.nrc + rc) * p.ncc + cc;
            }
          }
        }
        for (int ks = 0; ks < p.k_stages; ++ks) {
          mbar_wait(&full[stage], sphase);
          if (own && !(dbg_of(p) & 128)) {  // dbg bit 7: timing experiment, stages released unread
            const uint8_t* sa = sA + stage * L.a_stage_bytes;
            int32_t d0 = 0, d1 = 0, d2 = 0;  // <= 4 phases * 4 groups * kPx chunks: |d| < 2^27
#pragma unroll
            for (int ph = 0; ph < 4; ++ph) {
              if (ph >= p.n_phase) break;
#pragma unroll
              for (int g = 0; g < 4; ++g) {
                if (g >= p.gps) break;
                const int cg = ks * p.gps + g;
                const uint4* xs = reinterpret_cast<const uint4*>(sa) + (ph * p.gps + g) * p.strip_pix + it;
                uint4 xv[kPx], g0[kPx], g1[kPx], g2[kPx];
#pragma unroll
                for (int x = 0; x < kPx; ++x) {
                  xv[x] = xs[x * kIcThreads];
                  const uint4* gd = T + cg * 3 * ncell + cell[x][ph];
                  g0[x] = gd[0];
                  g1[x] = gd[ncell];
                  g2[x] = gd[2 * ncell];
                }
#pragma unroll
                for (int x = 0; x < kPx; ++x) {
                  d0 = __dp4a(static_cast<int>(xv[x].x), static_cast<int>(g0[x].x), d0);
                  d0 = __dp4a(static_cast<int>(xv[x].y), static_cast<int>(g0[x].y), d0);
                  d0 = __dp4a(static_cast<int>(xv[x].z), static_cast<int>(g0[x].z), d0);
                  d0 = __dp4a(static_cast<int>(xv[x].w), static_cast<int>(g0[x].w), d0);
                  d1 = __dp4a(static_cast<int>(xv[x].x), static_cast<int>(g1[x].x), d1);
                  d1 = __dp4a(static_cast<int>(xv[x].y), static_cast<int>(g1[x].y), d1);
                  d1 = __dp4a(static_cast<int>(xv[x].z), static_cast<int>(g1[x].z), d1);
                  d1 = __dp4a(static_cast<int>(xv[x].w), static_cast<int>(g1[x].w), d1);
                  d2 = __dp4a(static_cast<int>(xv[x].x), static_cast<int>(g2[x].x), d2);
                  d2 = __dp4a(static_cast<int>(xv[x].y), static_cast<int>(g2[x].y), d2);
                  d2 = __dp4a(static_cast<int>(xv[x].z), static_cast<int>(g2[x].z), d2);
                  d2 = __dp4a(static_cast<int>(xv[x].w), static_cast<int>(g2[x].w), d2);
                }
              }
            }
            acc += static_cast<long long>(d0) + (static_cast<long long>(d1) << 8) + (static_cast<long long>(d2) << 16);
          }
          // stage consumed (the loads above have returned): release it
          __syncwarp();
          if (lane == 0) mbar_arrive(&empty[stage]);
          if (++stage == p.n_stages) {
            stage = 0;
            sphase ^= 1u;
          }
        }
      }
    } else if (DT == DT_I8 && XT == 1 && p.rhs_mode == 4 && p.ic_ctas == 0) {
      // IC input checksum (class sums) by the two input-checksum warps
      pdl_wait();
      ic_class_sums_fr(p, static_cast<int64_t>(blockIdx.x) * (kRhsWarps * 32) + rw * 32 + lane,
                       static_cast<int64_t>(p.conv_grid) * (kRhsWarps * 32));
    } else if (DT == DT_I8 && FIC && p.rhs_mode == 1 && p.ic_ctas == 0) {
      pdl_wait();
      if (fr_share) {
        fr_claim_loop<DT>(p, &s_fr_claim, lane, acc, facc_rhs);
      } else {
        const int64_t first = static_cast<int64_t>(blockIdx.x) * (kRhsWarps * 32) + rw * 32 + lane;
        const int64_t stride = static_cast<int64_t>(p.conv_grid) * (kRhsWarps * 32);
        // large inputs (HBM-bound 1x1 layers with C >> K): more image loads in
        // flight; measured slower on the small 3x3 inputs, so chosen per plan
        if (p.rhs_deep)
          fic_rhs_fr<DT, 16>(p, first, stride, acc, facc_rhs);
        else
          fic_rhs_fr<DT, 8>(p, first, stride, acc, facc_rhs);
      }
    } else {
      pdl_wait();
    }
    fr_acc += acc;
    fr_facc += facc_rhs;
  }
  // every warp's share of the FIC rhs (input-checksum warps, and the others when
  // they took part through fr_claim_loop)
  if (FIC && (DT != DT_I8 || warp >= 2 + kEpiWarps)) {  // int8: only the input-checksum warps hold a share
    const long long w = DT == DT_I8 ? warp_sum(fr_acc) : __double_as_longlong(warp_sum_d(fr_facc));
    if (lane == 0) s_rhs_all[warp] = w;
  }

  if (trace && warp == 2 && lane == 0) {
    trace[5] = clock64() - t_entry;
    trace[6] = n_units;
    uint64_t gt_;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(gt_));
    trace[19] = static_cast<int64_t>(gt_);
  }
  if (trace && warp == 2 + kEpiWarps && lane == 0) trace[15] = clock64() - t_entry;  // input-checksum warps done
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem_base, tmem_cols);
  }
  if (s_ic)  // IC: this CTA's per-channel output sums, one reduction per channel
    for (int i = threadIdx.x; i < p.K; i += kConvThreads)
      if (s_ic[i]) red_add_u64(&p.ic_sum[i], s_ic[i]);

  // ---------------------------------------------------------------- verdict records
  // Each CTA stores its partials in its own record and exits; verdict_kernel
  // (one small launch per plan, or per pass of many layers) reduces them.  A
  // last-CTA reduction in this kernel would hold every CTA at exit for a ticket
  // atomic round trip (measured: ~2.5 us per layer on the critical path).
  if ((FC || FIC) && !(dbg_of(p) & 32) && threadIdx.x == 0) {
    int64_t* rec = p.cta_rec + static_cast<int64_t>(blockIdx.x) * kCtaRec;
    if (FC) {
      FcRec r{0, kNoKey, 0, 0};
      for (int w = 0; w < kEpiWarps; ++w) {
        r.cnt += s_fc[w].cnt;
        if (s_fc[w].key < r.key) {
          r.key = s_fc[w].key;
          r.lhs = s_fc[w].lhs;
          r.rhs = s_fc[w].rhs;
        }
      }
      rec[0] = r.cnt;
      rec[1] = r.key;
      rec[2] = r.lhs;
      rec[3] = r.rhs;
    }
    if (FIC) {
      if constexpr (DT == DT_I8) {
        long long l = 0;
        for (int w = 0; w < kEpiWarps; ++w) l += s_lhs[w];
        rec[4] = l;
        long long r = 0;
        for (int w = 0; w < kConvThreads / 32; ++w) r += s_rhs_all[w];
        rec[5] = r;
      } else {
        double l = 0.0;
        for (int w = 0; w < kEpiWarps; ++w) l += __longlong_as_double(s_lhs[w]);
        rec[4] = __double_as_longlong(l);
        double r = 0.0;
        for (int w = 0; w < kConvThreads / 32; ++w) r += __longlong_as_double(s_rhs_all[w]);
        rec[5] = __double_as_longlong(r);
      }
    }
  }
  if (trace && threadIdx.x == 0) {
    uint64_t gt;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(gt));
    trace[14] = static_cast<int64_t>(gt);
  }
}

}  // namespace abed_dev

// host-side launch templates: instantiated per (dtype, output flavour) in
// conv_inst_*.cu so the 48 kernel variants compile in parallel
namespace abed_host {
using abed_dev::ConvTcParams;
inline uint32_t conv_tc_smem_bytes_inl(const ConvTcParams& p) { return abed_dev::smem_layout(p).total; }
template <int DT, int EPI, bool FC, bool FIC, int XT>
cudaError_t launch_variant(const ConvTcParams& p, int grid, bool pdl, cudaStream_t stream) {
  // the smem opt-in is per device: one flag per ordinal
  static bool attr_done[64] = {};
  auto kern = abed_dev::conv_i8_tc_kernel<DT, EPI, FC, FIC, XT>;
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64 || !attr_done[dev]) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, abed_dev::kConvDynSmemMax);
    if (e != cudaSuccess) return e;
    if (dev >= 0 && dev < 64) attr_done[dev] = true;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(abed_dev::kConvThreads);
  cfg.dynamicSmemBytes = conv_tc_smem_bytes_inl(p);
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kern, p);
}

// XT: 0 = no per-channel extras, 1 = IC column sums, 2 = ICBatch batch sums,
// 3 = FIC-AF producer (the next layer's rhs dotted from the stored outputs),
// 4 = FIC with the staged input-checksum source (FIC-SM)
// (int8 only; separate kernel instances so the FC / FIC / unprotected kernels
// carry none of their code or registers: instruction-cache footprint is time)
template <int DT, int EPI, int XT>
cudaError_t launch_epi(const ConvTcParams& p, int grid, bool pdl, cudaStream_t st) {
  const bool fc = (p.check & abed_dev::CHECK_FC) != 0, fic = (p.check & abed_dev::CHECK_FIC) != 0;
  if constexpr (XT == 4) {  // FIC with the staged input-checksum source
    if (fc) return launch_variant<DT, EPI, true, true, XT>(p, grid, pdl, st);
    return launch_variant<DT, EPI, false, true, XT>(p, grid, pdl, st);
  }
  if (fc && fic) return launch_variant<DT, EPI, true, true, XT>(p, grid, pdl, st);
  if (fc) return launch_variant<DT, EPI, true, false, XT>(p, grid, pdl, st);
  if (fic) return launch_variant<DT, EPI, false, true, XT>(p, grid, pdl, st);
  return launch_variant<DT, EPI, false, false, XT>(p, grid, pdl, st);
}

}  // namespace abed_host
