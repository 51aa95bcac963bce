// Float mode on tensor cores: fp16 / bf16 operands, f32 accumulation.
//
// The reference's float mode (checksum.hpp:471-595) runs f32 operands with f64
// checksum reductions and absolute-threshold comparisons (float_verify).  Here
// the operands are stored as fp16 or bf16 (rounded to nearest even from the
// caller's f32 tensors), the convolution runs as tcgen05 kind::f16 MMAs with f32
// accumulators in TMEM (the same conv_tc kernel as INT8: a 16-byte pixel holds 8
// channels instead of 16, one MMA consumes K = 16 elements = 32 bytes, so every
// descriptor is unchanged), and the FC / FIC checks keep the reference's float
// semantics: f64 sums, |lhs - rhs| <= tau.
//
//   FC  filter checksum column: fsum_tile[c,r,s] = sum_k f (f64, rounded
//       filters) rides in three B rows as hi + lo + lo2 16-bit splits, so the
//       extra fmap carries ~24-33 significant bits.
//   FIC rhs = sum x * G computed by the kernel's input-checksum warps (G in f32
//       from the f64 filter checksum), lhs = f64 sum of the outputs.
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>

#include "abed_internal.h"

namespace abed_host {

using abed_dev::ActGeom;
using abed_dev::ConvTcParams;

namespace {

template <int DT>
__device__ __forceinline__ uint16_t to_h(float v) {
  if constexpr (DT == abed_dev::DT_BF16) {
    const __nv_bfloat16 h = __float2bfloat16_rn(v);
    return *reinterpret_cast<const uint16_t*>(&h);
  } else {
    const __half h = __float2half_rn(v);
    return *reinterpret_cast<const uint16_t*>(&h);
  }
}
template <int DT>
__device__ __forceinline__ float from_h(uint16_t b) {
  if constexpr (DT == abed_dev::DT_BF16) {
    return __uint_as_float(static_cast<uint32_t>(b) << 16);
  } else {
    __half h = *reinterpret_cast<const __half*>(&b);
    return __half2float(h);
  }
}
template <int DT>
__device__ __forceinline__ float round_h(float v) {
  return from_h<DT>(to_h<DT>(v));
}

// NCHW f32 -> strip planes of 16-bit values, 8 channels per 16-byte pixel
// (the INT8 pack_input_kernel with cpg = 8)
template <int DT>
__global__ void pack_input_h_kernel(const float* __restrict__ x, ActGeom g, int8_t* __restrict__ out) {
  const int64_t total = (int64_t)g.n_phase * g.c16 * g.plane_len;
  const int64_t HlWl = (int64_t)g.Hl * g.Wl;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t t = idx % g.plane_len;
    const int64_t plane = idx / g.plane_len;
    const int grp = (int)(plane % g.c16);
    const int phase = (int)(plane / g.c16);
    uint32_t w4[4] = {0, 0, 0, 0};
    if (t < g.m_total) {
      const int n = (int)(t / HlWl);
      const int64_t rem = t - n * HlWl;
      const int i = (int)(rem / g.Wl), j = (int)(rem % g.Wl);
      const int a = phase / g.nph_w, b = phase % g.nph_w;
      const int hh = i * g.sh + a - g.ph, ww = j * g.sw + b - g.pw;
      if (hh >= 0 && hh < g.h && ww >= 0 && ww < g.w) {
        for (int e = 0; e < 8; ++e) {
          const int c = grp * 8 + e;
          if (c < g.c) {
            const uint16_t v = to_h<DT>(x[(((int64_t)n * g.c + c) * g.h + hh) * g.w + ww]);
            w4[e >> 1] |= (uint32_t)v << (16 * (e & 1));
          }
        }
      }
    }
    reinterpret_cast<uint4*>(out)[idx] = make_uint4(w4[0], w4[1], w4[2], w4[3]);
  }
}

// B blocks [nt][ks][tap][gl][row][16 B] of 16-bit filters (8 channels per
// row); rows block_n .. block_n+2 hold the per-N-tile filter checksum as
// hi / lo / lo2 splits of its f64 value (rounded filters).
template <int DT>
__global__ void pack_filters_h_kernel(const float* __restrict__ f, ActGeom g, int block_n, int block_n_tot,
                                      int n_tiles, int gps, int k_stages, int fc, int8_t* __restrict__ out) {
  const int ntaps = g.r * g.s;
  const int64_t rows_total = (int64_t)n_tiles * k_stages * ntaps * gps * block_n_tot;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < rows_total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    int64_t rem = idx;
    const int row = (int)(rem % block_n_tot); rem /= block_n_tot;
    const int gl = (int)(rem % gps); rem /= gps;
    const int tap = (int)(rem % ntaps); rem /= ntaps;
    const int ks = (int)(rem % k_stages); rem /= k_stages;
    const int nt = (int)rem;
    const int r = tap / g.s, s = tap % g.s;
    const int cbase = (ks * gps + gl) * 8;
    uint16_t vals[8];
    for (int e = 0; e < 8; ++e) {
      const int c = cbase + e;
      float v = 0.0f;
      if (row < block_n) {
        const int k = nt * block_n + row;
        if (k < g.k && c < g.c) v = f[(((int64_t)k * g.c + c) * g.r + r) * g.s + s];
      } else {
        const int digit = row - block_n;
        if (fc && digit < 3 && c < g.c) {
          const int k_end = min(g.k, (nt + 1) * block_n);
          double sum = 0.0;
          for (int k = nt * block_n; k < k_end; ++k) sum += round_h<DT>(f[(((int64_t)k * g.c + c) * g.r + r) * g.s + s]);
          const float hi = round_h<DT>((float)sum);
          const float lo = round_h<DT>((float)(sum - hi));
          const float lo2 = round_h<DT>((float)(sum - hi - lo));
          v = digit == 0 ? hi : digit == 1 ? lo : lo2;
        }
      }
      vals[e] = to_h<DT>(v);
    }
    uint32_t w4[4];
    for (int q = 0; q < 4; ++q) w4[q] = (uint32_t)vals[2 * q] | ((uint32_t)vals[2 * q + 1] << 16);
    reinterpret_cast<uint4*>(out)[idx] = make_uint4(w4[0], w4[1], w4[2], w4[3]);
  }
}

// filter_checksum_f64 (checksum.hpp:483-494) of the rounded filters, (c,r,s) order
template <int DT>
__global__ void filter_sum_h_kernel(const float* __restrict__ f, int64_t K, int64_t crs, double* __restrict__ sums) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < crs; i += (int64_t)gridDim.x * blockDim.x) {
    double acc = 0.0;
    for (int64_t k = 0; k < K; ++k) acc += round_h<DT>(f[k * crs + i]);
    sums[i] = acc;
  }
}

// G[phase][grp][pix][8] = sum of fsum[c,r,s] over the taps whose window at this
// input position is a valid output (the INT8 fic_weight_kernel, f64 -> f32)
__global__ void fic_weight_h_kernel(const double* __restrict__ fsum, ActGeom g, float* __restrict__ G) {
  const int64_t HlWl = (int64_t)g.Hl * g.Wl;
  const int64_t total = (int64_t)g.n_phase * g.c16 * 8 * HlWl;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total; idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t pix = idx % HlWl;
    const int64_t ce = idx / HlWl;
    const int c = (int)(ce % (g.c16 * 8));
    const int phase = (int)(ce / (g.c16 * 8));
    const int i = (int)(pix / g.Wl), j = (int)(pix % g.Wl);
    double acc = 0.0;
    if (c < g.c) {
      for (int r = 0; r < g.r; ++r)
        for (int s = 0; s < g.s; ++s) {
          if ((r % g.sh) * g.nph_w + (s % g.sw) != phase) continue;
          const int p = i - r / g.sh, q = j - s / g.sw;
          if (p >= 0 && p < g.p && q >= 0 && q < g.q) acc += fsum[((int64_t)c * g.r + r) * g.s + s];
        }
    }
    const int grp = c >> 3, e = c & 7;
    G[(((int64_t)phase * g.c16 + grp) * HlWl + pix) * 8 + e] = (float)acc;
  }
}

int dt_of(int elem_kind) {
  if (elem_kind == ABED_F16) return abed_dev::DT_F16;
  if (elem_kind == ABED_BF16) return abed_dev::DT_BF16;
  throw_invalid("float-mode plan: element kind must be ABED_F16 or ABED_BF16");
  return 0;
}

template <int DT>
void build_h_plan(abed_conv_plan* pl, const float* filters) {
  const ActGeom& g = pl->g;
  const ConvTcParams& p = pl->base;
  const abed_layer_shape& shape = pl->shape;
  const int64_t crs = shape.c * shape.r * shape.s;
  cuda_check(cudaMalloc(&pl->d_wpk, (size_t)p.n_tiles * p.k_stages * p.b_stage_bytes), "cudaMalloc(wpk)");
  const int64_t rows = (int64_t)p.n_tiles * p.k_stages * p.ntaps * p.gps * p.block_n_tot;
  pack_filters_h_kernel<DT><<<grid_for(rows, 256), 256>>>(filters, g, p.block_n, p.block_n_tot, p.n_tiles, p.gps,
                                                     p.k_stages, (pl->checks & ABED_CHECK_FC) ? 1 : 0, pl->d_wpk);
  cuda_check(cudaGetLastError(), "pack_filters_h");
  cuda_check(cudaMalloc(&pl->d_fsum_f, crs * 8), "cudaMalloc(fsum_f)");
  filter_sum_h_kernel<DT><<<grid_for(crs, 256), 256>>>(filters, shape.k, crs, pl->d_fsum_f);
  cuda_check(cudaGetLastError(), "filter_sum_h");
  cuda_check(cudaMalloc(&pl->d_facc, 2 * 8), "cudaMalloc(facc)");
  cuda_check(cudaMemset(pl->d_facc, 0, 2 * 8), "memset facc");
  cuda_check(cudaMalloc(&pl->d_rhs_f, 8), "cudaMalloc(rhs_f)");
  cuda_check(cudaMemset(pl->d_rhs_f, 0, 8), "memset rhs_f");
  if (pl->checks & ABED_CHECK_FIC) {
    const int64_t nw = (int64_t)g.n_phase * g.c16 * 8 * g.Hl * g.Wl;
    cuda_check(cudaMalloc(&pl->d_ficwf, nw * 4), "cudaMalloc(ficwf)");
    fic_weight_h_kernel<<<grid_for(nw, 256), 256>>>(pl->d_fsum_f, g, pl->d_ficwf);
    cuda_check(cudaGetLastError(), "fic_weight_h");
  }
  cuda_check(cudaDeviceSynchronize(), "plan_create_h sync");
}

}  // namespace

abed_conv_plan* plan_create_h(const abed_layer_shape& shape, const float* filters, int elem_kind, int checks,
                              double tau_fc, double tau_fic, int force_bn) {
  require_device();
  validate_shape(shape);
  const int dt = dt_of(elem_kind);
  if (checks & ABED_CHECK_IC) throw_invalid("float-mode plan: the IC scheme is not supported on tensor cores");
  if (!(tau_fc >= 0.0) || !(tau_fic >= 0.0)) throw_invalid("float_verify: tau must be >= 0");
  if (shape.r * shape.s > abed_dev::kMaxTaps) throw_invalid("conv: filters with more than 64 taps are not supported");
  auto* pl = new abed_conv_plan();
  try {
    plan_init_common(pl, shape, checks, force_bn, 8);
    pl->dtype = dt;
    pl->tau_fc = tau_fc;
    pl->tau_fic = tau_fic;
    if (dt == abed_dev::DT_BF16)
      build_h_plan<abed_dev::DT_BF16>(pl, filters);
    else
      build_h_plan<abed_dev::DT_F16>(pl, filters);
  } catch (...) {
    abed_conv_plan_destroy(pl);
    throw;
  }
  return pl;
}

}  // namespace abed_host

using namespace abed_host;

extern "C" {

int abed_conv_plan_create_h(const abed_layer_shape* shape, const float* filters, int32_t elem_kind, int32_t checks,
                            double tau_fc, double tau_fic, int32_t force_block_n, abed_conv_plan** plan) {
  return guarded([&] { *plan = plan_create_h(*shape, filters, elem_kind, checks, tau_fc, tau_fic, force_block_n); });
}

int abed_pack_input_h(const abed_conv_plan* pl, const float* input, void* packed, void* stream) {
  return guarded([&] {
    if (pl->dtype == abed_dev::DT_I8) throw_invalid("pack_input_h: not a float-mode plan");
    const int64_t n16 = geom_packed_bytes(pl->g) / 16;
    if (pl->dtype == abed_dev::DT_BF16)
      pack_input_h_kernel<abed_dev::DT_BF16><<<grid_for(n16, 256), 256, 0, (cudaStream_t)stream>>>(
          input, pl->g, static_cast<int8_t*>(packed));
    else
      pack_input_h_kernel<abed_dev::DT_F16><<<grid_for(n16, 256), 256, 0, (cudaStream_t)stream>>>(
          input, pl->g, static_cast<int8_t*>(packed));
    cuda_check(cudaGetLastError(), "pack_input_h");
  });
}

int abed_conv_plan_set_tau(abed_conv_plan* pl, double tau_fc, double tau_fic) {
  return guarded([&] {
    if (!(tau_fc >= 0.0) || !(tau_fic >= 0.0)) throw_invalid("float_verify: tau must be >= 0");
    pl->tau_fc = tau_fc;
    pl->tau_fic = tau_fic;
  });
}

}  // extern "C"
