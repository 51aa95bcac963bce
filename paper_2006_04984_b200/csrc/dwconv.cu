// Depthwise INT8 convolution with the FIC check (MobileNetV2, BASELINE configs[3]).
//
// No reference counterpart (LayerShape has no groups; "MobileNetV2
// depthwise ... parity unpinned"): the oracle restates conv_reference
// (convolution.hpp:78-111) with one filter per channel, and the ABED identity is
// the reference's FIC by linearity -- sum of all outputs = sum_{c,r,s}
// f[c,r,s] * ic[c,r,s] with ic = gen_input_checksum (checksum.hpp:248-266),
// i.e. fic_dot with the depthwise filter as the filter checksum.  (FC has no
// cheaper form for depthwise: the channel-sum checksum filter IS the
// computation, so the plan offers FIC only.)
//
// Layout: the same strip planes as the tensor-core conv (16 channels per
// 16-byte pixel, stride phases, shared zero halo), so a pointwise conv can write
// a depthwise layer's input directly and vice versa.  One thread = one output
// pixel x 16 channels: the nine tap vectors are loaded as 16-byte pixels, four
// taps x four channels are byte-transposed with PRMT so one dp4a accumulates
// four taps of one channel, then the epilog (bias, ReLU, requantise) writes the
// next layer's packed pixel.  HBM / issue bound: ~16 B in and out per 16
// outputs x 9 MACs.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <vector>

#include "abed_internal.h"

namespace abed_dev {

struct DwParams {
  const int8_t* act;
  int64_t plane_len, m_total;
  int n_phase, c16, ntaps, quads, Hl, Wl, P, Q, N, C;
  int tap_phase[kMaxTaps];
  int tap_shift[kMaxTaps];
  const uint32_t* fpk;  // [c16][16 channels][quads] words of four taps (int8), zero padded
  // epilogue
  int out_mode;
  void* out;
  const float* bias;
  float scale;
  int relu;
  int64_t o_plane_len;
  int o_Hl, o_Wl, o_ph, o_pw, o_sh, o_sw, o_nph_w, o_c16;
  // FIC lhs records ([grid][kCtaRec], slot 4), ConvOut fault hook
  int fic;
  int64_t* cta_rec;
  unsigned long long* cmp_count;
  int64_t fault_key;
  int fault_bit;
  // FIC-AF producer side (see ConvTcParams::af_*)
  const int8_t* af_ficw8;
  unsigned long long* af_acc;
  int64_t af_HlWl;
  // FIC rhs in-kernel (FR): this plan's G digit planes [phase][c16][Hl*Wl][3][16 B]
  // and the image split of the (plane, pixel) items; nullptr = off
  const int8_t* ficw8;
  int rhs_nsplit;
};

// FIC rhs (FR option) over the stored input, x . G with G as three balanced
// base-256 digit planes: item = (plane, pixel position, image split), its G
// digits loaded once, 8 image loads in flight, 12 dp4a per 16-byte chunk; the
// digit partials are flushed every 32 images (exact in int32).  Same sum as
// checksum.hpp:248-285 (gen_input_checksum + fic_dot) regrouped by input pixel.
__device__ __forceinline__ long long dw_fic_rhs(const DwParams& p, int64_t first, int64_t stride) {
  constexpr int DEPTH = 8;
  const int64_t HlWl = static_cast<int64_t>(p.Hl) * p.Wl;
  const int nsplit = p.rhs_nsplit;
  const int64_t total = static_cast<int64_t>(p.n_phase) * p.c16 * HlWl * nsplit;
  long long acc = 0;
  for (int64_t idx = first; idx < total; idx += stride) {
    const int64_t pix = idx % HlWl;
    const int64_t rest = idx / HlWl;
    const int split = static_cast<int>(rest % nsplit);
    const int64_t plane = rest / nsplit;
    const uint4* gw = reinterpret_cast<const uint4*>(p.ficw8) + (plane * HlWl + pix) * 3;
    const uint4 g0 = __ldg(gw), g1 = __ldg(gw + 1), g2 = __ldg(gw + 2);
    const uint4* src = reinterpret_cast<const uint4*>(p.act) + plane * p.plane_len + pix;
    const int n0 = static_cast<int>(static_cast<int64_t>(p.N) * split / nsplit);
    const int n1 = static_cast<int>(static_cast<int64_t>(p.N) * (split + 1) / nsplit);
    int32_t d0 = 0, d1 = 0, d2 = 0;
    for (int n = n0; n < n1; n += DEPTH) {
      uint4 x[DEPTH];
#pragma unroll
      for (int j = 0; j < DEPTH; ++j)
        x[j] = n + j < n1 ? __ldcs(src + static_cast<int64_t>(n + j) * HlWl) : make_uint4(0u, 0u, 0u, 0u);
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
        d2 = __dp4a(static_cast<int>(x[j].x), static_cast<int>(g2.x), d2);
        d2 = __dp4a(static_cast<int>(x[j].y), static_cast<int>(g2.y), d2);
        d2 = __dp4a(static_cast<int>(x[j].z), static_cast<int>(g2.z), d2);
        d2 = __dp4a(static_cast<int>(x[j].w), static_cast<int>(g2.w), d2);
      }
      if (((n - n0) & 31) == 32 - DEPTH) {
        acc += static_cast<long long>(d0) + (static_cast<long long>(d1) << 8) + (static_cast<long long>(d2) << 16);
        d0 = d1 = d2 = 0;
      }
    }
    acc += static_cast<long long>(d0) + (static_cast<long long>(d1) << 8) + (static_cast<long long>(d2) << 16);
  }
  return acc;
}

// 4x4 byte transpose of four taps (a, b, c, d: one byte per channel) so that
// y[i] = {a.i, b.i, c.i, d.i} holds four taps of channel i for one dp4a
__device__ __forceinline__ void transpose4(uint32_t a, uint32_t b, uint32_t c, uint32_t d, uint32_t (&y)[4]) {
  const uint32_t t0 = __byte_perm(a, b, 0x5140), t1 = __byte_perm(a, b, 0x7362);
  const uint32_t t2 = __byte_perm(c, d, 0x5140), t3 = __byte_perm(c, d, 0x7362);
  y[0] = __byte_perm(t0, t2, 0x5410);
  y[1] = __byte_perm(t0, t2, 0x7632);
  y[2] = __byte_perm(t1, t3, 0x5410);
  y[3] = __byte_perm(t1, t3, 0x7632);
}

__device__ __forceinline__ int32_t dw_requant(int32_t acc, float scale, float bias, int relu) {
  float v = __fmaf_rn(static_cast<float>(acc), scale, bias);  // convolution.hpp:374-381 (FMA)
  v = relu ? fminf(fmaxf(v, 0.0f), 127.0f) : fminf(127.0f, fmaxf(-128.0f, v));
  return __float2int_rz(v);
}

template <int EPI>  // 0 none, 1 NCHW (int8 / int32 / f32 per out_mode), 2 packed, 3 compare
__global__ void __launch_bounds__(256) dwconv_i8_kernel(const __grid_constant__ DwParams p) {
  __shared__ long long s_red[8];
  long long af = 0;
  const uint32_t HlWl = static_cast<uint32_t>(p.Hl) * p.Wl;
  const int64_t PQ = static_cast<int64_t>(p.P) * p.Q;
  long long fic = 0;
  const int64_t total = static_cast<int64_t>(p.c16) * p.m_total;
  for (int64_t idx = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; idx < total;
       idx += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int g = static_cast<int>(idx / p.m_total);
    const int64_t m = idx - static_cast<int64_t>(g) * p.m_total;
    const uint32_t n_img = static_cast<uint32_t>(m / HlWl);
    const uint32_t rem = static_cast<uint32_t>(m - static_cast<int64_t>(n_img) * HlWl);
    const uint32_t pp = rem / p.Wl, qq = rem - pp * p.Wl;
    if (pp >= static_cast<uint32_t>(p.P) || qq >= static_cast<uint32_t>(p.Q)) continue;  // halo row
    int32_t acc[16];
#pragma unroll
    for (int c = 0; c < 16; ++c) acc[c] = 0;
    const uint32_t* fw = p.fpk + static_cast<int64_t>(g) * 16 * p.quads;
    for (int q = 0; q < p.quads; ++q) {
      uint4 X[4];
#pragma unroll
      for (int t4 = 0; t4 < 4; ++t4) {
        const int tap = 4 * q + t4;
        if (tap < p.ntaps) {
          const int64_t plane = static_cast<int64_t>(p.tap_phase[tap]) * p.c16 + g;
          X[t4] = __ldg(reinterpret_cast<const uint4*>(p.act) + plane * p.plane_len + m + p.tap_shift[tap]);
        } else {
          X[t4] = make_uint4(0u, 0u, 0u, 0u);
        }
      }
      const uint32_t xw[4][4] = {{X[0].x, X[0].y, X[0].z, X[0].w},
                                 {X[1].x, X[1].y, X[1].z, X[1].w},
                                 {X[2].x, X[2].y, X[2].z, X[2].w},
                                 {X[3].x, X[3].y, X[3].z, X[3].w}};
#pragma unroll
      for (int wq = 0; wq < 4; ++wq) {  // channels 4*wq .. 4*wq+3
        uint32_t y[4];
        transpose4(xw[0][wq], xw[1][wq], xw[2][wq], xw[3][wq], y);
#pragma unroll
        for (int b = 0; b < 4; ++b) {
          const int c = 4 * wq + b;
          acc[c] = __dp4a(static_cast<int>(y[b]), static_cast<int>(__ldg(fw + c * p.quads + q)), acc[c]);
        }
      }
    }
    const int k0 = g * 16;
    if (p.fault_key >= 0) {  // ConvOut fault hook (faults.hpp:230-233)
      const int64_t key0 = (static_cast<int64_t>(n_img) * p.C + k0) * PQ + static_cast<int64_t>(pp) * p.Q + qq;
#pragma unroll
      for (int c = 0; c < 16; ++c)
        if (key0 + c * PQ == p.fault_key) acc[c] = static_cast<int32_t>(static_cast<uint32_t>(acc[c]) ^ (1u << p.fault_bit));
    }
#pragma unroll
    for (int c = 0; c < 16; ++c)
      if (k0 + c >= p.C) acc[c] = 0;
    if (p.fic) {
      int32_t s = 0;  // |acc| <= 9 * 128 * 128 * 16 < 2^31 per pixel group for R*S <= 64
#pragma unroll
      for (int c = 0; c < 16; ++c) s += acc[c];
      fic += s;
    }
    if (EPI == 2 || EPI == 3) {
      uint32_t w[4] = {0u, 0u, 0u, 0u};
#pragma unroll
      for (int c = 0; c < 16; ++c) {
        const int32_t y = k0 + c < p.C ? dw_requant(acc[c], p.scale, __ldg(p.bias + k0 + c), p.relu) : 0;
        w[c >> 2] |= (static_cast<uint32_t>(y) & 0xFFu) << (8 * (c & 3));
      }
      const int hh = pp + p.o_ph, ww = qq + p.o_pw;
      const int64_t t = (static_cast<int64_t>(n_img) * p.o_Hl + hh / p.o_sh) * p.o_Wl + ww / p.o_sw;
      uint4* dst = reinterpret_cast<uint4*>(static_cast<int8_t*>(p.out)) +
                   (static_cast<int64_t>((hh % p.o_sh) * p.o_nph_w + (ww % p.o_sw)) * p.o_c16 + g) * p.o_plane_len + t;
      const uint4 val = make_uint4(w[0], w[1], w[2], w[3]);
      if (EPI == 2) {
        *dst = val;
        if (p.af_ficw8) {  // FIC-AF: the next layer's rhs from the stored values
          const uint4* gd = reinterpret_cast<const uint4*>(p.af_ficw8) +
                            ((static_cast<int64_t>((hh % p.o_sh) * p.o_nph_w + (ww % p.o_sw)) * p.o_c16 + g) * p.af_HlWl +
                             static_cast<int64_t>(hh / p.o_sh) * p.o_Wl + ww / p.o_sw) * 3;
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
          af += static_cast<long long>(d0) + (static_cast<long long>(d1) << 8) + (static_cast<long long>(d2) << 16);
        }
      } else {
        const uint4 r = *dst;
        if (r.x != val.x || r.y != val.y || r.z != val.z || r.w != val.w) atomicAdd(p.cmp_count, 1ull);
      }
    } else if (EPI == 1) {
      const int64_t base = static_cast<int64_t>(n_img) * p.C * PQ + static_cast<int64_t>(k0) * PQ +
                           static_cast<int64_t>(pp) * p.Q + qq;
      for (int c = 0; c < 16 && k0 + c < p.C; ++c) {
        if (p.out_mode == OUT_I32_NCHW) {
          static_cast<int32_t*>(p.out)[base + c * PQ] = acc[c];
        } else if (p.out_mode == OUT_I8_NCHW) {
          static_cast<int8_t*>(p.out)[base + c * PQ] =
              static_cast<int8_t>(dw_requant(acc[c], p.scale, __ldg(p.bias + k0 + c), p.relu));
        } else {
          float f = __fmaf_rn(static_cast<float>(acc[c]), p.scale, __ldg(p.bias + k0 + c));
          if (p.relu && f < 0.0f) f = 0.0f;
          static_cast<float*>(p.out)[base + c * PQ] = f;
        }
      }
    }
  }
  if (EPI == 2 && p.af_ficw8) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) af += __shfl_xor_sync(0xffffffffu, af, o);
    if ((threadIdx.x & 31) == 0 && af != 0) atomicAdd(p.af_acc, static_cast<unsigned long long>(af));
  }
  if (p.fic) {
    // this block's share of the FIC rhs (FR), after its conv work
    long long rhs = p.ficw8 ? dw_fic_rhs(p, static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x,
                                         static_cast<int64_t>(gridDim.x) * blockDim.x)
                            : 0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      fic += __shfl_xor_sync(0xffffffffu, fic, o);
      rhs += __shfl_xor_sync(0xffffffffu, rhs, o);
    }
    __shared__ long long s_rhs[8];
    if ((threadIdx.x & 31) == 0) {
      s_red[threadIdx.x >> 5] = fic;
      s_rhs[threadIdx.x >> 5] = rhs;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      long long t = 0, r = 0;
      for (int w = 0; w < static_cast<int>(blockDim.x >> 5); ++w) {
        t += s_red[w];
        r += s_rhs[w];
      }
      int64_t* rec = p.cta_rec + static_cast<int64_t>(blockIdx.x) * kCtaRec;
      rec[4] = t;
      rec[5] = r;
    }
  }
}

}  // namespace abed_dev

namespace abed_host {

using abed_dev::ActGeom;

namespace {

// [c16][16][quads] words of four taps of one channel's filter (int8, (r,s) order)
__global__ void pack_dw_filters_kernel(const int8_t* __restrict__ f, int C, int ntaps, int quads, int c16,
                                       uint32_t* __restrict__ out) {
  const int total = c16 * 16 * quads;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += gridDim.x * blockDim.x) {
    const int q = i % quads, c = i / quads;
    uint32_t w = 0;
    for (int t4 = 0; t4 < 4; ++t4) {
      const int tap = 4 * q + t4;
      const int8_t v = (c < C && tap < ntaps) ? f[(int64_t)c * ntaps + tap] : (int8_t)0;
      w |= (uint32_t)(uint8_t)v << (8 * t4);
    }
    out[i] = w;
  }
}

// the depthwise filter is its own filter checksum: fsum[c,r,s] = f[c,0,r,s]
__global__ void dw_fsum_kernel(const int8_t* __restrict__ f, int64_t n, int32_t* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = f[i];
}

constexpr int kDwBlocksPerSm = 4;

}  // namespace

int dw_grid() { return num_sms() * kDwBlocksPerSm; }

abed_conv_plan* plan_create_dw(const abed_layer_shape& shape, const int8_t* filters, int checks) {
  require_device();
  validate_shape(shape);
  if (shape.k != shape.c) throw_invalid("depthwise conv: K must equal C (one filter per channel)");
  if (checks & ~ABED_CHECK_FIC) throw_invalid("depthwise conv: only the FIC scheme applies");
  if (shape.r * shape.s > abed_dev::kMaxTaps) throw_invalid("conv: filters with more than 64 taps are not supported");
  auto* pl = new abed_conv_plan();
  try {
    pl->dw = 1;
    pl->shape = shape;
    pl->checks = checks;
    pl->g = make_geom(shape, 16);
    const ActGeom& g = pl->g;
    const int ntaps = g.r * g.s, quads = (ntaps + 3) / 4;
    cuda_check(cudaMalloc(&pl->d_dwf, (size_t)g.c16 * 16 * quads * 4), "cudaMalloc(dwf)");
    pack_dw_filters_kernel<<<grid_for(g.c16 * 16 * quads, 256), 256>>>(filters, g.c, ntaps, quads, g.c16, pl->d_dwf);
    cuda_check(cudaGetLastError(), "pack_dw_filters");
    const int64_t crs = shape.c * ntaps;
    cuda_check(cudaMalloc(&pl->d_filters, (size_t)crs), "cudaMalloc(filters)");
    cuda_check(cudaMemcpy(pl->d_filters, filters, (size_t)crs, cudaMemcpyDeviceToDevice), "copy filters");
    cuda_check(cudaMalloc(&pl->d_fsum, crs * 4), "cudaMalloc(fsum)");
    dw_fsum_kernel<<<grid_for(crs, 256), 256>>>(filters, crs, pl->d_fsum);
    cuda_check(cudaMalloc(&pl->d_cta_rec, (size_t)dw_grid() * abed_dev::kCtaRec * 8), "cudaMalloc(cta_rec)");
    cuda_check(cudaMemset(pl->d_cta_rec, 0, (size_t)dw_grid() * abed_dev::kCtaRec * 8), "memset cta_rec");
    cuda_check(cudaMalloc(&pl->d_acc, (4 + shape.k) * 8), "cudaMalloc(acc)");
    cuda_check(cudaMemset(pl->d_acc, 0, (4 + shape.k) * 8), "memset acc");
    cuda_check(cudaMalloc(&pl->d_zero_bias, shape.k * 4), "cudaMalloc(bias)");
    cuda_check(cudaMemset(pl->d_zero_bias, 0, shape.k * 4), "memset bias");
    if (checks & ABED_CHECK_FIC) {
      const int64_t nw = (int64_t)g.n_phase * g.c16 * 16 * g.Hl * g.Wl;
      cuda_check(cudaMalloc(&pl->d_ficw, nw * 4), "cudaMalloc(ficw)");
      fic_weight_kernel<<<grid_for(nw, 256), 256>>>(pl->d_fsum, g, pl->d_ficw);
      cuda_check(cudaGetLastError(), "fic_weight");
      cuda_check(cudaMalloc(&pl->d_ficw8, nw * 3), "cudaMalloc(ficw8)");
      int* d_big = nullptr;
      cuda_check(cudaMalloc(&d_big, 4), "cudaMalloc(flag)");
      cuda_check(cudaMemset(d_big, 0, 4), "memset flag");
      fic_weight_digits_kernel<<<grid_for(nw, 256), 256>>>(pl->d_ficw, nw / 16, pl->d_ficw8, d_big);
      int big = 0;
      cuda_check(cudaMemcpy(&big, d_big, 4, cudaMemcpyDeviceToHost), "flag d2h");
      cudaFree(d_big);
      pl->ficw8_ok = (big & 1) ? 0 : 1;  // bit 1: a third digit is needed (unused here)
    }
    cuda_check(cudaMalloc(&pl->d_af_acc, 8), "cudaMalloc(af_acc)");
    cuda_check(cudaMemset(pl->d_af_acc, 0, 8), "memset af_acc");
    cuda_check(cudaDeviceSynchronize(), "plan_create_dw sync");
  } catch (...) {
    abed_conv_plan_destroy(pl);
    throw;
  }
  return pl;
}

void plan_run_dw(abed_conv_plan* pl, const int8_t* packed, const abed_epilog_params* ep, int out_mode, void* out,
                 const abed_conv_plan* next, int64_t fault_key, int fault_bit, cudaStream_t st) {
  const ActGeom& g = pl->g;
  abed_dev::DwParams p;
  std::memset(&p, 0, sizeof(p));
  p.act = packed;
  p.plane_len = g.plane_len;
  p.m_total = g.m_total;
  p.n_phase = g.n_phase;
  p.c16 = g.c16;
  p.ntaps = g.r * g.s;
  p.quads = (p.ntaps + 3) / 4;
  p.Hl = g.Hl; p.Wl = g.Wl; p.P = g.p; p.Q = g.q; p.N = g.n; p.C = g.c;
  for (int r = 0; r < g.r; ++r)
    for (int s = 0; s < g.s; ++s) {
      const int t = r * g.s + s;
      p.tap_phase[t] = (r % g.sh) * g.nph_w + (s % g.sw);
      p.tap_shift[t] = (r / g.sh) * g.Wl + (s / g.sw);
    }
  p.fpk = pl->d_dwf;
  p.out_mode = out_mode;
  p.out = out;
  if (ep) {
    if (!std::isfinite(ep->scale)) throw_invalid("epilog: non-finite scale");
    if (ep->bias && ep->bias_len != pl->shape.k) throw_invalid("epilog: bias length must equal the channel count");
    p.scale = ep->scale;
    p.bias = ep->bias ? ep->bias : pl->d_zero_bias;
    p.relu = ep->activation == ABED_RELU ? 1 : 0;
  } else {
    p.scale = 1.0f;
    p.bias = pl->d_zero_bias;
    p.relu = 0;
  }
  if (out_mode == ABED_OUT_H_PACKED || out_mode == ABED_OUT_H_COMPARE)
    throw_invalid("depthwise conv: int8 plan, 16-bit output modes do not apply");
  if (out_mode == ABED_OUT_I8_PACKED || out_mode == ABED_OUT_I8_COMPARE) {
    ActGeom o;
    if (next) {
      o = next->g;
      if (o.c != g.k || o.h != g.p || o.w != g.q || o.n != g.n || o.cpg != g.cpg)
        throw_invalid("conv plan: next layer input does not match this layer's output");
    } else {
      abed_layer_shape s1{g.n, g.k, g.p, g.q, 1, 1, 1, 1, 1, 0, 0, g.p, g.q};
      o = make_geom(s1, g.cpg);
    }
    p.o_plane_len = o.plane_len; p.o_Hl = o.Hl; p.o_Wl = o.Wl; p.o_ph = o.ph; p.o_pw = o.pw;
    p.o_sh = o.sh; p.o_sw = o.sw; p.o_nph_w = o.nph_w; p.o_c16 = o.c16;
    if (next && out_mode == ABED_OUT_I8_PACKED && next->af_input && (next->checks & ABED_CHECK_FIC)) {
      p.af_ficw8 = next->d_ficw8;
      p.af_acc = next->d_af_acc;
      p.af_HlWl = (int64_t)o.Hl * o.Wl;
    }
    if (out_mode == ABED_OUT_I8_COMPARE) cuda_check(cudaMemsetAsync(pl->d_acc + 1, 0, 8, st), "memset cmp");
  }
  p.fic = (pl->checks & ABED_CHECK_FIC) ? 1 : 0;
  p.cta_rec = pl->d_cta_rec;
  p.cmp_count = pl->d_acc + 1;
  p.fault_key = fault_key;
  p.fault_bit = fault_bit;
  const bool af_in = p.fic && pl->af_input && !pl->reuse_input_checksum;
  bool fr_in_kernel = false;
  if (p.fic && !pl->reuse_input_checksum && !af_in) {
    const int64_t cells = (int64_t)g.n_phase * g.c16 * g.Hl * g.Wl;
    if (pl->ficw8_ok) {
      // FR inside the depthwise kernel: every block dots its share of the stored
      // input after its conv work; the rhs rides in the per-block records (slot 5)
      const int64_t threads = (int64_t)dw_grid() * 256;
      p.ficw8 = pl->d_ficw8;
      p.rhs_nsplit = (int)std::max<int64_t>(1, std::min<int64_t>(std::max(1, g.n / 8), (threads + cells - 1) / cells));
      fr_in_kernel = true;
    } else {
      // |G| too large for the 3-digit map: one separate pass ahead of the conv
      cuda_check(cudaMemsetAsync(pl->d_acc, 0, 8, st), "memset rhs");
      const int nsplit = g.n >= 8 ? 8 : g.n;
      fic_rhs_kernel<<<grid_for(cells * nsplit, 256), 256, 0, st>>>(packed, g, pl->d_ficw, nsplit, pl->d_acc);
      cuda_check(cudaGetLastError(), "fic_rhs");
    }
  }
  // AF accumulator, FR rhs from the block records, or the rhs kept in d_acc[0]
  pl->last_rhs_mode = af_in ? 2 : fr_in_kernel ? 1 : 0;
  const int grid = dw_grid();
  switch (out_mode) {
    case ABED_OUT_NONE: abed_dev::dwconv_i8_kernel<0><<<grid, 256, 0, st>>>(p); break;
    case ABED_OUT_I8_PACKED: abed_dev::dwconv_i8_kernel<2><<<grid, 256, 0, st>>>(p); break;
    case ABED_OUT_I8_COMPARE: abed_dev::dwconv_i8_kernel<3><<<grid, 256, 0, st>>>(p); break;
    default: abed_dev::dwconv_i8_kernel<1><<<grid, 256, 0, st>>>(p); break;
  }
  cuda_check(cudaGetLastError(), "dwconv launch");
}

}  // namespace abed_host

using namespace abed_host;

extern "C" {

int abed_conv_plan_create_dw(const abed_layer_shape* shape, const int8_t* filters, int32_t checks,
                             abed_conv_plan** plan) {
  return guarded([&] { *plan = plan_create_dw(*shape, filters, checks); });
}

}  // extern "C"
