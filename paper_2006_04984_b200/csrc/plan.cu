// Layer planning and the HBM-bound helper kernels of the protected int8 conv:
//   * geometry of the packed strip-plane activation layout (conv_tc.cuh)
//   * pack_input:   reference NCHW int8  -> strip planes       (boundary, once per call)
//   * pack_filters: reference KCRS int8  -> UMMA B blocks + FC checksum-digit rows
//                   (checksum.hpp:75 gen_filter_checksum, :108 decompose, offline)
//   * batch_sum / box_sum_dot: input checksum and FIC right-hand side
//                   (checksum.hpp:248 gen_input_checksum, :275 fic_dot, :350 ic_batch_checksum)
//   * finalize kernels turning per-tile records into a reference VerifyOutcome
//                   (checksum.hpp:211-236 fc_verify, :287-294 fic_verify, :319-347 ic_verify_k)
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstring>
#include <stdexcept>
#include <string>

#include "abed_internal.h"

namespace abed_host {

using abed_dev::ActGeom;
using abed_dev::ConvTcParams;

static inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

ActGeom make_geom(const abed_layer_shape& s, int cpg, int n_extra) {
  ActGeom g{};
  g.n = (int)s.n; g.c = (int)s.c; g.h = (int)s.h; g.w = (int)s.w;
  g.k = (int)s.k; g.r = (int)s.r; g.s = (int)s.s;
  g.sh = (int)s.stride_h; g.sw = (int)s.stride_w; g.ph = (int)s.pad_h; g.pw = (int)s.pad_w;
  g.p = (int)s.p; g.q = (int)s.q;
  g.nph_h = std::min(g.sh, g.r);
  g.nph_w = std::min(g.sw, g.s);
  g.n_phase = g.nph_h * g.nph_w;
  g.cpg = cpg;
  g.c16 = (int)ceil_div(g.c, cpg);
  if (g.c16 & 1) g.c16 += 1;  // one MMA consumes two 16-byte channel groups (32 bytes of K)
  auto extent = [](int P, int H, int R, int st, int pad, int nph) {
    auto zero_lead = [&](int a) { return pad > a ? (int)ceil_div(pad - a, st) : 0; };
    int L = P;
    for (int a = 0; a < nph; ++a)
      if (pad + H - 1 - a >= 0) L = std::max(L, 1 + (pad + H - 1 - a) / st);
    for (int r = 0; r < R; ++r) L = std::max(L, P + r / st - zero_lead(r % st));
    return L;
  };
  g.Hl = extent(g.p, g.h, g.r, g.sh, g.ph, g.nph_h);
  g.Wl = extent(g.q, g.w, g.s, g.sw, g.pw, g.nph_w);
  g.max_shift = ((g.r - 1) / g.sh) * g.Wl + (g.s - 1) / g.sw;
  g.n_extra = n_extra;
  g.m_total = (int64_t)(g.n + n_extra) * g.Hl * g.Wl;
  g.m_tiles = (int)ceil_div(g.m_total, abed_dev::kBlockM);
  const int strip = (int)((abed_dev::kBlockM + g.max_shift + 7) / 8 * 8);
  g.plane_len = (int64_t)(g.m_tiles - 1) * abed_dev::kBlockM + strip;
  return g;
}

int geom_strip_pix(const ActGeom& g) { return (abed_dev::kBlockM + g.max_shift + 7) / 8 * 8; }

int64_t geom_packed_bytes(const ActGeom& g) {
  return (int64_t)g.n_phase * g.c16 * g.plane_len * 16;
}

// ---------------------------------------------------------------------------
// pack_input: one thread per (plane, pixel t); 16 channel bytes gathered from
// NCHW, zero outside the image (padding halo) and beyond the last image.
// ---------------------------------------------------------------------------
__global__ void pack_input_kernel(const int8_t* __restrict__ x, ActGeom g, int8_t* __restrict__ out) {
  const int64_t total = (int64_t)g.n_phase * g.c16 * g.plane_len;
  const int64_t HlWl = (int64_t)g.Hl * g.Wl;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t t = idx % g.plane_len;
    const int64_t plane = idx / g.plane_len;
    const int grp = (int)(plane % g.c16);
    const int phase = (int)(plane / g.c16);
    uint32_t w4[4] = {0, 0, 0, 0};
    if (t < (int64_t)g.n * HlWl) {
      const int n = (int)(t / HlWl);
      const int64_t rem = t - n * HlWl;
      const int i = (int)(rem / g.Wl), j = (int)(rem % g.Wl);
      const int a = phase / g.nph_w, b = phase % g.nph_w;
      const int hh = i * g.sh + a - g.ph, ww = j * g.sw + b - g.pw;
      if (hh >= 0 && hh < g.h && ww >= 0 && ww < g.w) {
        for (int e = 0; e < 16; ++e) {
          const int c = grp * 16 + e;
          if (c < g.c) {
            const uint8_t v = (uint8_t)x[(((int64_t)n * g.c + c) * g.h + hh) * g.w + ww];
            w4[e >> 2] |= (uint32_t)v << (8 * (e & 3));
          }
        }
      }
    }
    reinterpret_cast<uint4*>(out)[idx] = make_uint4(w4[0], w4[1], w4[2], w4[3]);
  }
}

// ---------------------------------------------------------------------------
// pack_input, vectorised: one thread per four consecutive pixels of ONE M-space
// row of one plane (quads are aligned to row starts, so no quad crosses a row).
// For a unit-stride phase each channel's four source bytes are contiguous in the
// NCHW row: two aligned 32-bit loads + a funnel shift fetch them, halo / edge
// pixels are masked arithmetically (no divergent per-pixel path), and a 4x4 byte
// transpose (__byte_perm) turns the 16 channel words into four 16-byte pixels:
// 32 loads per 64 output bytes instead of 64 byte loads.  Strided phases gather
// bytes.  Pixels past the last image (plane tail) are zero-filled.
// ---------------------------------------------------------------------------
__device__ __forceinline__ void transpose_store4(const uint32_t (&cw)[16], uint4* dst, int n_pix) {
  uint32_t o[4][4];  // [pixel][channel word q]
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const uint32_t a0 = __byte_perm(cw[4 * q], cw[4 * q + 1], 0x5140);      // c0p0 c1p0 c0p1 c1p1
    const uint32_t a1 = __byte_perm(cw[4 * q], cw[4 * q + 1], 0x7362);      // c0p2 c1p2 c0p3 c1p3
    const uint32_t b0 = __byte_perm(cw[4 * q + 2], cw[4 * q + 3], 0x5140);  // c2p0 c3p0 c2p1 c3p1
    const uint32_t b1 = __byte_perm(cw[4 * q + 2], cw[4 * q + 3], 0x7362);  // c2p2 c3p2 c2p3 c3p3
    o[0][q] = __byte_perm(a0, b0, 0x5410);
    o[1][q] = __byte_perm(a0, b0, 0x7632);
    o[2][q] = __byte_perm(a1, b1, 0x5410);
    o[3][q] = __byte_perm(a1, b1, 0x7632);
  }
#pragma unroll
  for (int u = 0; u < 4; ++u)
    if (u < n_pix) dst[u] = make_uint4(o[u][0], o[u][1], o[u][2], o[u][3]);
}

__global__ void __launch_bounds__(256) pack_input_v4_kernel(const int8_t* __restrict__ x, ActGeom g, int64_t x_bytes,
                                                            int vec_ok, int8_t* __restrict__ out) {
  // blockIdx.y = plane (phase, channel group); 32-bit index math inside a plane
  // (64-bit divisions per quad made this kernel issue-bound)
  const int plane = blockIdx.y;
  const int grp = plane % g.c16;
  const int phase = plane / g.c16;
  const int a = phase / g.nph_w, b = phase % g.nph_w;
  const uint32_t qpr = (uint32_t)((g.Wl + 3) >> 2);  // quads per M-space row
  const uint32_t rows = (uint32_t)g.n * (uint32_t)g.Hl;
  const uint32_t body = rows * qpr;
  const uint32_t tail_q = (uint32_t)((g.plane_len - g.m_total + 3) >> 2);  // zero quads after the last image
  const uint32_t total = body + tail_q;
  const int64_t HW = (int64_t)g.h * g.w;
  uint4* const pbase = reinterpret_cast<uint4*>(out) + (int64_t)plane * g.plane_len;
  for (uint32_t idx = blockIdx.x * blockDim.x + threadIdx.x; idx < total; idx += gridDim.x * blockDim.x) {
    if (idx >= body) {
      const int64_t t0 = g.m_total + (int64_t)(idx - body) * 4;
      uint4* dst = pbase + t0;
      const int np = (int)(g.plane_len - t0 < 4 ? g.plane_len - t0 : 4);
      for (int u = 0; u < np; ++u) dst[u] = make_uint4(0, 0, 0, 0);
      continue;
    }
    const uint32_t row = idx / qpr;  // n * Hl + i
    const uint32_t qi = idx - row * qpr;
    const uint32_t n = row / (uint32_t)g.Hl;
    const int i = (int)(row - n * (uint32_t)g.Hl);
    const int j0 = (int)qi * 4;
    const int n_pix = min(4, g.Wl - j0);
    uint4* dst = pbase + (int64_t)row * g.Wl + j0;
    const int hh = i * g.sh + a - g.ph;
    const int ww0 = j0 * g.sw + b - g.pw;
    uint32_t cw[16];
    if (hh < 0 || hh >= g.h || grp * 16 >= g.c) {
#pragma unroll
      for (int e = 0; e < 16; ++e) cw[e] = 0;
    } else {
      // byte mask of the pixels whose source column lies inside the image
      uint32_t keep = 0;
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int ww = ww0 + u * g.sw;
        if (u < n_pix && ww >= 0 && ww < g.w) keep |= 0xFFu << (8 * u);
      }
      const int64_t row0 = ((int64_t)n * g.c + grp * 16) * HW + (int64_t)hh * g.w;
      if (g.sw == 1 && vec_ok && x_bytes >= 4) {
        // all 32 aligned words first (clamped addresses, no branches), then the
        // funnel shifts: with load -> use per channel only two loads were in flight
        uint32_t lo[16], hi[16];
        int64_t al[16];
#pragma unroll
        for (int e = 0; e < 16; ++e) {
          const int ce = min(grp * 16 + e, g.c - 1);
          al[e] = ((int64_t)n * g.c + ce) * HW + (int64_t)hh * g.w + ww0;
          // clamp into the aligned words that overlap [0, x_bytes): an aligned word
          // holding a valid byte never crosses a page, and the bytes past the end
          // are masked by `keep`
          const int64_t a = al[e] & ~int64_t(3);
          const int64_t lim = (x_bytes - 1) & ~int64_t(3);
          const int64_t a0 = a < 0 ? 0 : (a > lim ? lim : a);
          const int64_t a1 = a + 4 > lim ? lim : (a + 4 < 0 ? 0 : a + 4);
          lo[e] = __ldg(reinterpret_cast<const uint32_t*>(x + a0));
          hi[e] = __ldg(reinterpret_cast<const uint32_t*>(x + a1));
        }
#pragma unroll
        for (int e = 0; e < 16; ++e) {
          const int64_t a = al[e] & ~int64_t(3);
          const uint32_t l = (a >= 0 && a < x_bytes) ? lo[e] : 0u, h = a + 4 < x_bytes ? hi[e] : 0u;
          const uint32_t v = __funnelshift_r(l, h, (uint32_t)(al[e] & 3) * 8) & keep;
          cw[e] = grp * 16 + e < g.c ? v : 0u;
        }
      } else {
#pragma unroll
        for (int e = 0; e < 16; ++e) {
          uint32_t v = 0;
          if (grp * 16 + e < g.c) {
            const int8_t* src = x + row0 + (int64_t)e * HW;
#pragma unroll
            for (int u = 0; u < 4; ++u)
              if ((keep >> (8 * u)) & 1u) v |= (uint32_t)(uint8_t)__ldg(src + ww0 + u * g.sw) << (8 * u);
          }
          cw[e] = v;
        }
      }
    }
    transpose_store4(cw, dst, n_pix);
  }
}

// Shared-memory staged transpose (NCHW -> strip planes): block = (plane, band of
// rb M-space rows, group of ipb images); smem holds one image's band in the
// OUTPUT layout (two buffers, alternating over the images): rows of wp 16-byte
// pixel slots, output pixel j of band row ii at slot ii * wp + pad0 + j, slot s
// stored at s ^ ((s >> 3) & 7) (an XOR swizzle inside each 8-slot group).
// Phase 1: work item = (band row, channel quad, input word of WB bytes = WB
// columns): 4 coalesced WB-byte loads (the quad's channels), WB/4 4 x 4 byte
// transposes (__byte_perm) and one 32-bit smem store per column.  Lanes of a warp
// cover (channel quad, word) pairs of one row; the swizzle spreads a store
// instruction over distinct banks.  With stride 1, pad0 aligns every input word
// to a slot group, so the stores need no bounds checks (slots outside the output
// row are never read) and their addresses are one XOR apart.  Phase 2 writes the
// band out with 16-byte stores; halo pixels (rows / columns outside the input)
// and filler channel quads are written as zeros there, so there is no zeroing
// pass.  When every thread has at most one item (the common case) its source
// offset, smem address and copy-out slots are computed once per block and pinned
// in registers, and the next image's words are loaded before the current image's
// barrier and copy-out.  Every input byte read once per stride phase, every output
// byte written once.  WB = 2 for rows of an even width (ResNet's 14-wide stages:
// 12.6 -> 6.1 us per b32 layer, stride 2: 34.7 -> 12.4 us).  WB = 0: odd widths
// (or an odd base address) use byte loads.  The zero tail of each plane (after
// the last image) is written
// by one extra block per plane.
#ifndef ABED_PACK_MINB
#define ABED_PACK_MINB 6  // resident 256-thread blocks per SM the register budget allows (40 regs; 5: 48 regs, 0.68 vs 0.71 of HBM)
#endif
__device__ __forceinline__ int pack_slot(int s) { return s ^ ((s >> 3) & 7); }

// n / d for 0 <= n < 2^31 with a multiply-high (the divisor fixed per launch)
struct PackDiv {
  uint32_t m, l, d;
  __device__ __forceinline__ int div(int n) const { return (int)((__umulhi((uint32_t)n, m) + (uint32_t)n) >> l); }
};
static PackDiv pack_div(uint32_t d) {
  uint32_t l = 0;
  while ((1ull << l) < d) ++l;
  return PackDiv{(uint32_t)(((1ull << 32) * ((1ull << l) - d)) / d + 1), l, d};
}

// one (band row, channel quad, input word) item of phase 1: load (pack_load),
// transpose and store to the staging rows (pack_store)
template <int WB>
__device__ __forceinline__ void pack_load(const int8_t* src, int HW, uint32_t lm, uint32_t (&v)[4][WB >= 4 ? WB / 4 : 1]) {
  constexpr int NW = WB >= 4 ? WB / 4 : 1;  // 32-bit words per load
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    if ((lm >> e) & 1u) {  // channel 4cq + e exists
      if (NW == 2) {
        const uint2 t = __ldg(reinterpret_cast<const uint2*>(src + e * HW));
        v[e][0] = t.x;
        v[e][NW - 1] = t.y;
      } else if (WB == 2) {
        v[e][0] = __ldg(reinterpret_cast<const uint16_t*>(src + e * HW));
      } else {
        v[e][0] = __ldg(reinterpret_cast<const uint32_t*>(src + e * HW));
      }
    } else {
#pragma unroll
      for (int h = 0; h < NW; ++h) v[e][h] = 0u;
    }
  }
}

template <int SW, int WB>
__device__ __forceinline__ void pack_store(const uint32_t (&v)[4][WB >= 4 ? WB / 4 : 1], int cq, uint8_t* buf, int q,
                                           int ii, int wp, int pad0, int off, int sw, int Wl, int fixed_base) {
  constexpr int NW = WB >= 4 ? WB / 4 : 1;  // 32-bit words per load
  constexpr int NP = WB >= 2 ? WB : 1;      // columns per word (WB = 2: the low two of a transpose)
  // 4 x 4 byte transposes: pw[4h + t] = channels 4cq..4cq+3 of column WB*q + 4h + t
  uint32_t pw[4 * NW];
#pragma unroll
  for (int h = 0; h < NW; ++h) {
    const uint32_t t01lo = __byte_perm(v[0][h], v[1][h], 0x5140), t01hi = __byte_perm(v[0][h], v[1][h], 0x7362);
    const uint32_t t23lo = __byte_perm(v[2][h], v[3][h], 0x5140), t23hi = __byte_perm(v[2][h], v[3][h], 0x7362);
    pw[4 * h + 0] = __byte_perm(t01lo, t23lo, 0x5410);
    pw[4 * h + 1] = __byte_perm(t01lo, t23lo, 0x7632);
    pw[4 * h + 2] = __byte_perm(t01hi, t23hi, 0x5410);
    pw[4 * h + 3] = __byte_perm(t01hi, t23hi, 0x7632);
  }
  if (SW == 1) {
    // slots s0 .. s0 + NP - 1 (s0 a multiple of NP): the swizzled byte address of
    // column t is base ^ (t << 4)
    const uint32_t base = fixed_base >= 0 ? (uint32_t)fixed_base
                                          : (uint32_t)pack_slot(ii * wp + pad0 + off + q * NP) * 16u + cq * 4u;
#pragma unroll
    for (int t = 0; t < NP; ++t) *reinterpret_cast<uint32_t*>(buf + (base ^ (t << 4))) = pw[t];
  } else {
#pragma unroll
    for (int t = 0; t < NP; ++t) {
      const int jj = q * NP + t + off;  // = j * sw
      int j;
      if (SW == 2) {
        if (jj & 1) continue;
        j = jj >> 1;
      } else {
        if (jj % sw) continue;
        j = jj / sw;
      }
      if (jj < 0 || j >= Wl) continue;
      *reinterpret_cast<uint32_t*>(buf + pack_slot(ii * wp + pad0 + j) * 16 + cq * 4) = pw[t];
    }
  }
}

template <int SW, int WB>  // SW: horizontal stride 1 or 2 (0: any); WB: 8, 4 or 0 (bytes)
__global__ void __launch_bounds__(256, ABED_PACK_MINB) pack_input_smem_kernel(const int8_t* __restrict__ x, ActGeom g, int lrb,
                                                                 PackDiv div_bands, int ipb, int pad0, int wp,
                                                                 int8_t* __restrict__ out) {
  extern __shared__ __align__(128) uint8_t tile[];  // 2 x [rb][wp][16]
  const int rb = 1 << lrb;
  const int grp = blockIdx.y, phase = blockIdx.z;
  const int plane = phase * g.c16 + grp;
  int a = phase, b = 0;
  if (SW == 2 && g.nph_w == 2) a = phase >> 1, b = phase & 1;
  if (SW == 0) a = phase / g.nph_w, b = phase - a * g.nph_w;
  uint4* const pbase = reinterpret_cast<uint4*>(out) + (int64_t)plane * g.plane_len;
  if (blockIdx.x == gridDim.x - 1) {  // zero tail of this plane
    for (int64_t t = g.m_total + threadIdx.x; t < g.plane_len; t += blockDim.x) pbase[t] = make_uint4(0, 0, 0, 0);
    return;
  }
  const int ng = div_bands.div(blockIdx.x);
  const int i0 = (blockIdx.x - ng * (int)div_bands.d) * rb;
  const int rows = min(rb, g.Hl - i0);
  const int nch = max(0, min(16, g.c - grp * 16));  // 0: a filler group (c16 is even)
  const int nq = (nch + 3) >> 2;
  const int npix = rows * g.Wl;
  const int HW = g.h * g.w;
  const int off = g.pw - b;  // output column j holds input column j * sw - off
  const int sw = SW ? SW : g.sw;
  // valid output columns [jlo, jhi): 0 <= j * sw - off < w
  int jlo, jhi;
  if (SW == 1) {
    jlo = max(off, 0);
    jhi = min(g.Wl, g.w + off);
  } else {
    jlo = off <= 0 ? 0 : (off + sw - 1) / sw;
    jhi = min(g.Wl, g.w - 1 + off < 0 ? 0 : (g.w - 1 + off) / sw + 1);
  }
  // valid band rows [ilo, ihi): 0 <= r0 + ii * sh < h
  const int r0 = i0 * g.sh + a - g.ph;
  int ilo = 0, ihi = rows;
  while (ilo < rows && r0 + ilo * g.sh < 0) ++ilo;
  while (ihi > ilo && r0 + (ihi - 1) * g.sh >= g.h) --ihi;
  // phase-1 lane roles (fixed for the block): lanes split into groups of lpr lanes
  // (lane -> input word q of a row); a group is one (row, channel quad) pair
  // rp = 4 * ii + cq; warps and groups walk the pairs
  const int wq = WB ? g.w / WB : 0;
  const int lpr = wq <= 4 ? 4 : wq <= 8 ? 8 : wq <= 16 ? 16 : 32;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int sub = lane / lpr, ql = lane - sub * lpr;
  const int gpw = 32 / lpr;
  const int npairs = ihi << 2;
  const int rp0 = ilo * 4 + warp * gpw + sub;
  // common case: every thread has at most one item; its source offset and smem
  // address are fixed for all images of the block
  const bool one = WB != 0 && (ihi - ilo) * 4 <= 8 * gpw && wq <= lpr;
  // (pinned in registers: the compiler would otherwise recompute them per image)
  uint32_t lm0 = 0;
  if (one && rp0 < npairs && ql < wq) lm0 = (1u << max(0, min(4, nch - 4 * (rp0 & 3)))) - 1u;
  int src0 = (rp0 & 3) * 4 * HW + (r0 + (rp0 >> 2) * g.sh) * g.w + ql * WB;
  int base0 = SW == 1 ? pack_slot((rp0 >> 2) * wp + pad0 + off + ql * WB) * 16 + (rp0 & 3) * 4
                      : -1;
  asm volatile("" : "+r"(lm0), "+r"(src0), "+r"(base0));
  // phase 2: the (up to 4) pixels of this thread and their smem slots, packed
  // two per register (0xffff: halo, stored as zeros; 0xfffe: no pixel)
  const bool p2fast = npix <= 4 * 256 && nq == 4;
  uint32_t slots[2] = {0xfffefffeu, 0xfffefffeu};
  if (p2fast) {
    const float rwl = 1.0f / (float)g.Wl;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int i = threadIdx.x + 256 * k;
      const int ii = __float2int_rz(((float)i + 0.5f) * rwl);
      const int j = i - ii * g.Wl;
      uint32_t sl = 0xfffeu;
      if (i < npix)
        sl = (ii >= ilo && ii < ihi && j >= jlo && j < jhi) ? (uint32_t)pack_slot(ii * wp + pad0 + j) : 0xffffu;
      slots[k >> 1] = (slots[k >> 1] & ~(0xffffu << (16 * (k & 1)))) | (sl << (16 * (k & 1)));
    }
    asm volatile("" : "+r"(slots[0]), "+r"(slots[1]));
  }
  const int n_end = min(g.n, (ng + 1) * ipb);
  // per-image pointers advance by one image: this thread's item source, the band's output
  const int64_t xstep = (int64_t)g.c * HW, dstep = (int64_t)g.Hl * g.Wl;
  const int8_t* xg = x + ((int64_t)ng * ipb * g.c + grp * 16) * HW;
  uint4* dst = pbase + ((int64_t)ng * ipb * g.Hl + i0) * g.Wl;
  constexpr int NW = WB >= 4 ? WB / 4 : 1;
  uint32_t v[4][NW];  // common case: the next image's item, loaded before this image's phase 2
  if (WB != 0 && one && lm0) pack_load<WB>(xg + src0, HW, lm0, v);
  for (int n = ng * ipb; n < n_end; ++n, xg += xstep, dst += dstep) {
    uint8_t* const buf = tile + (size_t)((n - ng * ipb) & 1) * 16 * rb * wp;
    if (WB != 0) {
      if (one) {
        if (lm0) {
          pack_store<SW, WB>(v, rp0 & 3, buf, ql, rp0 >> 2, wp, pad0, off, sw, g.Wl, base0);
          if (n + 1 < n_end) pack_load<WB>(xg + xstep + src0, HW, lm0, v);
        }
      } else {
        for (int rp = rp0; rp < npairs; rp += 8 * gpw) {
          const int cq = rp & 3, ii = rp >> 2;
          if (cq >= nq) continue;
          const uint32_t lm = (1u << min(4, nch - 4 * cq)) - 1u;
          const int8_t* const src = xg + cq * 4 * HW + (r0 + ii * g.sh) * g.w;
          for (int q = ql; q < wq; q += lpr) {
            pack_load<WB>(src + q * WB, HW, lm, v);
            pack_store<SW, WB>(v, cq, buf, q, ii, wp, pad0, off, sw, g.Wl, -1);
          }
        }
      }
    } else {
      const int total = nch * rows * g.w;
      for (int idx = threadIdx.x; idx < total; idx += blockDim.x) {
        const int e = idx / (rows * g.w), rem = idx - e * rows * g.w, ii = rem / g.w, ww = rem - ii * g.w;
        if (ii < ilo || ii >= ihi) continue;
        const int jj = ww + off;
        if (jj < 0 || jj % sw) continue;
        const int j = jj / sw;
        if (j >= g.Wl) continue;
        buf[pack_slot(ii * wp + pad0 + j) * 16 + e] = (uint8_t)xg[e * HW + (r0 + ii * g.sh) * g.w + ww];
      }
      // channels nch..4nq-1 of the last quad: zero (phase 2 masks whole quads only)
      if (nch & 3)
        for (int i = threadIdx.x; i < rows * wp; i += blockDim.x)
          for (int e = nch; e < 4 * nq; ++e) buf[i * 16 + e] = 0;
    }
    __syncthreads();
    const uint4* const st4 = reinterpret_cast<const uint4*>(buf);
    if (p2fast) {
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const uint32_t sl = (slots[k >> 1] >> (16 * (k & 1))) & 0xffffu;
        if (sl != 0xfffeu) dst[threadIdx.x + 256 * k] = sl != 0xffffu ? st4[sl] : make_uint4(0, 0, 0, 0);
      }
    } else {
      const float rwl = 1.0f / (float)g.Wl;
      for (int i = threadIdx.x; i < npix; i += blockDim.x) {
        const int ii = __float2int_rz(((float)i + 0.5f) * rwl);  // exact: i < 8 Wl, Wl <= 1536
        const int j = i - ii * g.Wl;
        uint4 v = make_uint4(0, 0, 0, 0);
        if (ii >= ilo && ii < ihi && j >= jlo && j < jhi && nq > 0) {
          v = st4[pack_slot(ii * wp + pad0 + j)];
          if (nq < 4) {
            if (nq < 2) v.y = 0;
            if (nq < 3) v.z = 0;
            v.w = 0;
          }
        }
        dst[i] = v;
      }
    }
    // the next image writes the other buffer; the one after this reuses this one
    // only after the next barrier, which every thread reaches after its phase 2
  }
}

void launch_pack_input(const int8_t* x, const ActGeom& g, int8_t* packed, cudaStream_t st) {
  const int planes = g.n_phase * g.c16;
  const int64_t x_bytes = (int64_t)g.n * g.c * g.h * g.w;
  // smem rows: wp 16-byte slots, output pixel j at slot pad0 + j; with stride 1
  // pad0 makes input column 0 land on a multiple of 8 slots
  const int pad0 = g.sw == 1 ? (8 - (g.pw & 7)) & 7 : 0;
  const int wp = (std::max(pad0 + g.Wl, g.sw == 1 ? pad0 + g.pw + g.w : 0) + 7) & ~7;
  // band height: a power of two <= 8 M-space rows, <= 24 KB of staged pixels (x2 buffers)
  int lrb = 3;
  while (lrb > 0 && (16 << lrb) * wp > 24 * 1024) --lrb;
  if (16 * wp <= 24 * 1024) {
    const int rb = 1 << lrb;
    const int nbands = (g.Hl + rb - 1) / rb;
    const uintptr_t xa = reinterpret_cast<uintptr_t>(x);
    const int wb = (g.w % 8 == 0 && (xa & 7) == 0)   ? 8
                   : (g.w % 4 == 0 && (xa & 3) == 0) ? 4
                   : (g.w % 2 == 0 && (xa & 1) == 0) ? 2
                                                     : 0;
    // images per block: amortise the per-block setup while keeping >= ~4 waves
    const char* ipb_s = getenv("ABED_PACK_IPB");  // tuning / test override
    const int ipb_env = ipb_s ? atoi(ipb_s) : 0;
    int ipb = ipb_env > 0 ? ipb_env : 1;
    if (ipb_env <= 0)
      while (ipb < 4 && (int64_t)((g.n + 2 * ipb - 1) / (2 * ipb)) * nbands * planes >= (int64_t)num_sms() * 8) ipb *= 2;
    const int ngroups = (g.n + ipb - 1) / ipb;
    const size_t smem = (size_t)2 * 16 * rb * wp;
    const dim3 grid((unsigned)(ngroups * nbands + 1), (unsigned)g.c16, (unsigned)g.n_phase);
    const PackDiv div_bands = pack_div((uint32_t)nbands);
#define ABED_PACK_LAUNCH(SWV)                                                                     \
  do {                                                                                             \
    if (wb == 8)                                                                                   \
      pack_input_smem_kernel<SWV, 8><<<grid, 256, smem, st>>>(x, g, lrb, div_bands, ipb, pad0, wp, packed);     \
    else if (wb == 4)                                                                              \
      pack_input_smem_kernel<SWV, 4><<<grid, 256, smem, st>>>(x, g, lrb, div_bands, ipb, pad0, wp, packed);     \
    else if (wb == 2)                                                                              \
      pack_input_smem_kernel<SWV, 2><<<grid, 256, smem, st>>>(x, g, lrb, div_bands, ipb, pad0, wp, packed);     \
    else                                                                                           \
      pack_input_smem_kernel<SWV, 0><<<grid, 256, smem, st>>>(x, g, lrb, div_bands, ipb, pad0, wp, packed);     \
  } while (0)
    if (g.sw == 1)
      ABED_PACK_LAUNCH(1);
    else if (g.sw == 2)
      ABED_PACK_LAUNCH(2);
    else
      ABED_PACK_LAUNCH(0);
#undef ABED_PACK_LAUNCH
    return;
  }
  // very wide rows: the register-transpose kernel
  const int64_t per_plane = (int64_t)g.n * g.Hl * ((g.Wl + 3) / 4) + (g.plane_len - g.m_total + 3) / 4;
  if (per_plane >= (int64_t(1) << 31)) throw_invalid("pack_input: plane too large");
  int64_t bx = ((int64_t)num_sms() * 8 + planes - 1) / planes;
  const int64_t need = (per_plane + 255) / 256;
  if (bx > need) bx = need;
  if (bx < 1) bx = 1;
  const int vec_ok = (reinterpret_cast<uintptr_t>(x) & 3) == 0;  // aligned 32-bit source loads
  pack_input_v4_kernel<<<dim3((unsigned)bx, (unsigned)planes), 256, 0, st>>>(x, g, x_bytes, vec_ok, packed);
}

// ---------------------------------------------------------------------------
// pack_filters: B blocks [nt][ks][tap][gl][row][16B]; rows >= block_n hold the
// balanced base-256 digits of the per-N-tile filter checksum
// fsum_nt[c,r,s] = sum_{k in tile} f[k,c,r,s]  (checksum.hpp:75-90 restricted to
// the tile; the per-tile extras add up to the reference's extra fmap exactly).
// ---------------------------------------------------------------------------
__global__ void pack_filters_kernel(const int8_t* __restrict__ f, ActGeom g, int block_n, int block_n_tot,
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
    const int cbase = (ks * gps + gl) * 16;
    int8_t vals[16];
    if (row < block_n) {
      const int k = nt * block_n + row;
      for (int e = 0; e < 16; ++e) {
        const int c = cbase + e;
        vals[e] = (k < g.k && c < g.c) ? f[(((int64_t)k * g.c + c) * g.r + r) * g.s + s] : (int8_t)0;
      }
    } else {
      const int digit = row - block_n;
      for (int e = 0; e < 16; ++e) {
        const int c = cbase + e;
        int32_t sum = 0;
        if (fc && digit < 3 && c < g.c) {
          const int k_end = min(g.k, (nt + 1) * block_n);
          for (int k = nt * block_n; k < k_end; ++k) sum += f[(((int64_t)k * g.c + c) * g.r + r) * g.s + s];
          // balanced digits: sum = d0 + 256 d1 + 65536 d2, each in [-128, 127]
          int32_t d0 = ((sum + 128) & 0xFF) - 128;
          int32_t rest = (sum - d0) / 256;
          int32_t d1 = ((rest + 128) & 0xFF) - 128;
          int32_t d2 = (rest - d1) / 256;
          sum = digit == 0 ? d0 : digit == 1 ? d1 : d2;
        } else {
          sum = 0;
        }
        vals[e] = (int8_t)sum;
      }
    }
    uint32_t w4[4] = {0, 0, 0, 0};
    for (int e = 0; e < 16; ++e) w4[e >> 2] |= (uint32_t)(uint8_t)vals[e] << (8 * (e & 3));
    reinterpret_cast<uint4*>(out)[idx] = make_uint4(w4[0], w4[1], w4[2], w4[3]);
  }
}

// filter checksum in reference (c,r,s) order, i32 (checksum.hpp:75-90)
// ---------------------------------------------------------------------------
// Input checksum of the packed input.  Stage 1 (HBM-bound, reads the input
// once): batch sum B[phase][c][i][j] = sum_n plane[(n*Hl+i)*Wl+j] (this is the
// ICBatch checksum image, checksum.hpp:350-362, in packed coordinates).
// Stage 2: ic[c,r,s] = box sum of B over i in [r/sh, r/sh+P), j in [s/sw, s/sw+Q)
// in phase (r%sh, s%sw) -- every window position of gen_input_checksum
// (checksum.hpp:248-266) -- fused with the FIC dot against the filter checksum.
// ---------------------------------------------------------------------------
__global__ void batch_sum_packed_kernel(const int8_t* __restrict__ act, ActGeom g, int32_t* __restrict__ bsum) {
  const int64_t HlWl = (int64_t)g.Hl * g.Wl;
  const int64_t total = (int64_t)g.n_phase * g.c16 * HlWl;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t pix = idx % HlWl;
    const int64_t plane = idx / HlWl;
    const uint4* src = reinterpret_cast<const uint4*>(act) + plane * g.plane_len + pix;
    int32_t acc[16];
#pragma unroll
    for (int e = 0; e < 16; ++e) acc[e] = 0;
    for (int n = 0; n < g.n; ++n) {
      const uint4 v = __ldg(src + (int64_t)n * HlWl);
      const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
      for (int e = 0; e < 16; ++e) acc[e] += (int32_t)(int8_t)(w[e >> 2] >> (8 * (e & 3)));
    }
    // layout [plane][16][HlWl] so stage 2 reads contiguous rows per channel
    int32_t* dst = bsum + plane * 16 * HlWl + pix;
#pragma unroll
    for (int e = 0; e < 16; ++e) dst[(int64_t)e * HlWl] = acc[e];
  }
}

// one block per (channel c); computes ic[c,r,s] for all taps, writes ic (reference
// (c,r,s) order) and atomically adds sum_rs fsum[c,r,s]*ic[c,r,s] into *fic_rhs.
__global__ void box_sum_dot_kernel(const int32_t* __restrict__ bsum, ActGeom g, const int32_t* __restrict__ fsum,
                                   int32_t* __restrict__ ic_out, unsigned long long* __restrict__ fic_rhs) {
  const int c = blockIdx.x;
  if (c >= g.c) return;
  const int64_t HlWl = (int64_t)g.Hl * g.Wl;
  const int grp = c >> 4, e = c & 15;
  __shared__ long long red[32];
  long long dot_local = 0;
  for (int tap = 0; tap < g.r * g.s; ++tap) {
    const int r = tap / g.s, s = tap % g.s;
    const int phase = (r % g.sh) * g.nph_w + (s % g.sw);
    const int i0 = r / g.sh, j0 = s / g.sw;
    const int32_t* img = bsum + ((int64_t)(phase * g.c16 + grp) * 16 + e) * HlWl;
    long long acc = 0;
    const int64_t cnt = (int64_t)g.p * g.q;
    for (int64_t t = threadIdx.x; t < cnt; t += blockDim.x) {
      const int pp = (int)(t / g.q), qq = (int)(t % g.q);
      const int i = i0 + pp, j = j0 + qq;
      // positions past the image block alias the next image's zero halo
      if (i < g.Hl && j < g.Wl) acc += img[(int64_t)i * g.Wl + j];
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
    __syncthreads();
    if (threadIdx.x == 0) {
      long long tot = 0;
      for (int w = 0; w < (int)(blockDim.x >> 5); ++w) tot += red[w];
      const int64_t ci = ((int64_t)c * g.r + r) * g.s + s;
      if (ic_out) ic_out[ci] = (int32_t)tot;
      if (fsum) dot_local += (long long)fsum[ci] * tot;
    }
    __syncthreads();
  }
  if (threadIdx.x == 0 && fic_rhs) atomicAdd(fic_rhs, (unsigned long long)dot_local);
}

// ---------------------------------------------------------------------------
// FIC right-hand side in ONE pass over the input (FR option).  fic_dot(fc, ic)
// = sum_{c,r,s} fsum[c,r,s] * sum_{windows} x = sum_{pixels} x * G, where
// G[phase][c][i][j] = sum of fsum[c,r,s] over the taps (r,s) of that phase whose
// window position (i - r/sh, j - s/sw) is a valid output (checksum.hpp:248-285
// regrouped by input position).  G depends only on the offline filters.
// ---------------------------------------------------------------------------
__global__ void fic_weight_kernel(const int32_t* __restrict__ fsum, ActGeom g, int32_t* __restrict__ G) {
  const int64_t HlWl = (int64_t)g.Hl * g.Wl;
  const int64_t total = (int64_t)g.n_phase * g.c16 * 16 * HlWl;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total; idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t pix = idx % HlWl;
    const int64_t ce = idx / HlWl;  // phase * c16*16 + channel
    const int c = (int)(ce % (g.c16 * 16));
    const int phase = (int)(ce / (g.c16 * 16));
    const int i = (int)(pix / g.Wl), j = (int)(pix % g.Wl);
    int32_t acc = 0;
    if (c < g.c) {
      for (int r = 0; r < g.r; ++r)
        for (int s = 0; s < g.s; ++s) {
          if ((r % g.sh) * g.nph_w + (s % g.sw) != phase) continue;
          const int p = i - r / g.sh, q = j - s / g.sw;
          if (p >= 0 && p < g.p && q >= 0 && q < g.q) acc += fsum[((int64_t)c * g.r + r) * g.s + s];
        }
    }
    // layout [phase][c16][HlWl][16]: one 64-byte vector per packed pixel
    const int grp = c >> 4, e = c & 15;
    G[(((int64_t)phase * g.c16 + grp) * HlWl + pix) * 16 + e] = acc;
  }
}

// G -> 3 balanced base-256 digits (G = d0 + 256 d1 + 65536 d2, d in [-128, 127]),
// for the conv kernel's dp4a input-checksum warps; flags |G| >= 2^23 (not exact)
__global__ void fic_weight_digits_kernel(const int32_t* __restrict__ G, int64_t cells, int8_t* __restrict__ G8,
                                         int* __restrict__ too_big) {
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < cells * 16; idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t cell = idx >> 4;
    const int e = (int)(idx & 15);
    int32_t v = G[idx];
    if (v >= (1 << 23) - 128 || v <= -(1 << 23) + 128) atomicOr(too_big, 1);
    const int32_t d0 = ((v + 128) & 255) - 128;
    v = (v - d0) >> 8;
    const int32_t d1 = ((v + 128) & 255) - 128;
    v = (v - d1) >> 8;
    if (v != 0) atomicOr(too_big, 2);  // the third digit plane is needed
    G8[(cell * 3 + 0) * 16 + e] = (int8_t)d0;
    G8[(cell * 3 + 1) * 16 + e] = (int8_t)d1;
    G8[(cell * 3 + 2) * 16 + e] = (int8_t)v;
  }
}

// FIC-SM class table, digit-plane major so that pixels of different classes
// read different shared-memory banks: T8[((grp * 3 + digit) * n_rep + cls) * 16 + e]
// = digit `digit` of G for channel grp * 16 + e at class cls's representative
// pixel (cls = (phase * nrc + rc) * ncc + cc); zero for class pairs no pixel has
__global__ void fic_class_table_kernel(const int8_t* __restrict__ G8, ActGeom g, const int* __restrict__ rep, int n_rep,
                                       int8_t* __restrict__ T8) {
  const int64_t HlWl = (int64_t)g.Hl * g.Wl;
  const int64_t total = (int64_t)n_rep * g.c16 * 48;
  const int per_phase = (n_rep - 1) / g.n_phase;  // the last cell is the zero cell
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total; idx += (int64_t)gridDim.x * blockDim.x) {
    const int e = (int)(idx & 15);
    const int cls = (int)((idx >> 4) % n_rep);
    const int64_t gd = (idx >> 4) / n_rep;  // grp * 3 + digit
    const int grp = (int)(gd / 3), digit = (int)(gd % 3);
    const int pix = rep[cls];
    const int phase = cls / per_phase;
    T8[idx] = pix < 0 ? (int8_t)0 : G8[(((int64_t)phase * g.c16 + grp) * HlWl + pix) * 48 + digit * 16 + e];
  }
}

// rhs += sum over (plane, image block pixel, image) of x . G ; images split in
// `nsplit` groups so enough loads are in flight to stream HBM.
__global__ void fic_rhs_kernel(const int8_t* __restrict__ act, ActGeom g, const int32_t* __restrict__ G, int nsplit,
                               unsigned long long* __restrict__ rhs) {
  const int64_t HlWl = (int64_t)g.Hl * g.Wl;
  const int64_t planes = (int64_t)g.n_phase * g.c16;
  const int64_t total = planes * HlWl * nsplit;
  long long acc = 0;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total; idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t pix = idx % HlWl;
    const int64_t rest = idx / HlWl;
    const int split = (int)(rest % nsplit);
    const int64_t plane = rest / nsplit;
    const int4* gw = reinterpret_cast<const int4*>(G + (plane * HlWl + pix) * 16);
    int32_t w[16];
#pragma unroll
    for (int v = 0; v < 4; ++v) {
      const int4 t = __ldg(gw + v);
      w[4 * v] = t.x; w[4 * v + 1] = t.y; w[4 * v + 2] = t.z; w[4 * v + 3] = t.w;
    }
    const uint4* src = reinterpret_cast<const uint4*>(act) + plane * g.plane_len + pix;
    const int n0 = (int)((int64_t)g.n * split / nsplit), n1 = (int)((int64_t)g.n * (split + 1) / nsplit);
#pragma unroll 4
    for (int n = n0; n < n1; ++n) {
      const uint4 x = __ldcs(src + (int64_t)n * HlWl);
      const uint32_t xw[4] = {x.x, x.y, x.z, x.w};
#pragma unroll
      for (int e = 0; e < 16; ++e) acc += (long long)(int8_t)(xw[e >> 2] >> (8 * (e & 3))) * w[e];
    }
  }
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  __shared__ long long red[32];
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    long long t = 0;
    for (int i = 0; i < (int)(blockDim.x >> 5); ++i) t += red[i];
    atomicAdd(rhs, (unsigned long long)t);
  }
}

// The same FR sum with G as three balanced base-256 digit planes (ficw8,
// [plane][pix][3][16 B]): 12 dp4a per 16-byte chunk instead of 16 widened int64
// multiply-adds, G loaded once per item, DEPTH image loads in flight.  Exact:
// every digit partial stays inside int32 between flushes (32 images x 16 x 2^14).
__global__ void fic_rhs_dp4a_kernel(const int8_t* __restrict__ act, ActGeom g, const int8_t* __restrict__ G8,
                                    int nsplit, unsigned long long* __restrict__ rhs) {
  constexpr int DEPTH = 8;
  const int64_t HlWl = (int64_t)g.Hl * g.Wl;
  const int64_t planes = (int64_t)g.n_phase * g.c16;
  const int64_t total = planes * HlWl * nsplit;
  long long acc = 0;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total; idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t pix = idx % HlWl;
    const int64_t rest = idx / HlWl;
    const int split = (int)(rest % nsplit);
    const int64_t plane = rest / nsplit;
    const uint4* gw = reinterpret_cast<const uint4*>(G8) + (plane * HlWl + pix) * 3;
    const uint4 g0 = __ldg(gw), g1 = __ldg(gw + 1), g2 = __ldg(gw + 2);
    const uint4* src = reinterpret_cast<const uint4*>(act) + plane * g.plane_len + pix;
    const int n0 = (int)((int64_t)g.n * split / nsplit), n1 = (int)((int64_t)g.n * (split + 1) / nsplit);
    int32_t d0 = 0, d1 = 0, d2 = 0;
    for (int n = n0; n < n1; n += DEPTH) {
      uint4 x[DEPTH];
#pragma unroll
      for (int j = 0; j < DEPTH; ++j)
        x[j] = n + j < n1 ? __ldcs(src + (int64_t)(n + j) * HlWl) : make_uint4(0u, 0u, 0u, 0u);
#pragma unroll
      for (int j = 0; j < DEPTH; ++j) {
        d0 = __dp4a((int)x[j].x, (int)g0.x, d0); d0 = __dp4a((int)x[j].y, (int)g0.y, d0);
        d0 = __dp4a((int)x[j].z, (int)g0.z, d0); d0 = __dp4a((int)x[j].w, (int)g0.w, d0);
        d1 = __dp4a((int)x[j].x, (int)g1.x, d1); d1 = __dp4a((int)x[j].y, (int)g1.y, d1);
        d1 = __dp4a((int)x[j].z, (int)g1.z, d1); d1 = __dp4a((int)x[j].w, (int)g1.w, d1);
        d2 = __dp4a((int)x[j].x, (int)g2.x, d2); d2 = __dp4a((int)x[j].y, (int)g2.y, d2);
        d2 = __dp4a((int)x[j].z, (int)g2.z, d2); d2 = __dp4a((int)x[j].w, (int)g2.w, d2);
      }
      if (((n - n0) & 31) == 32 - DEPTH) {  // flush before the digit sums can leave int32
        acc += (long long)d0 + ((long long)d1 << 8) + ((long long)d2 << 16);
        d0 = d1 = d2 = 0;
      }
    }
    acc += (long long)d0 + ((long long)d1 << 8) + ((long long)d2 << 16);
  }
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  __shared__ long long red[32];
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    long long t = 0;
    for (int i = 0; i < (int)(blockDim.x >> 5); ++i) t += red[i];
    atomicAdd(rhs, (unsigned long long)t);
  }
}

// ---------------------------------------------------------------------------
// finalize kernels (single block), write an abed_verify_outcome to device memory
// ---------------------------------------------------------------------------
__device__ void write_outcome(abed_verify_outcome* o, int mismatch, int has_locus, int64_t l0, int64_t l1,
                              int64_t l2, int64_t lhs, int64_t rhs, int64_t count) {
  o->status = mismatch;
  o->has_locus = has_locus;
  o->locus[0] = l0; o->locus[1] = l1; o->locus[2] = l2;
  o->lhs = lhs; o->rhs = rhs;
  o->lhs_f = 0.0; o->rhs_f = 0.0;
  o->error_count = count;
}

// FC, single N tile: records in M order -> first mismatching tile gives the locus
__global__ void fc_finalize_rec_kernel(const int64_t* __restrict__ rec, int m_tiles, int P, int Q,
                                       abed_verify_outcome* out) {
  __shared__ long long s_cnt[32];
  __shared__ int s_first[32];
  long long cnt = 0;
  int first = 0x7fffffff;
  for (int t = threadIdx.x; t < m_tiles; t += blockDim.x) {
    cnt += rec[t * 4 + 0];
    if (rec[t * 4 + 0] > 0 && t < first) first = t;
  }
  for (int o = 16; o > 0; o >>= 1) {
    cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
    first = min(first, __shfl_xor_sync(0xffffffffu, first, o));
  }
  if ((threadIdx.x & 31) == 0) { s_cnt[threadIdx.x >> 5] = cnt; s_first[threadIdx.x >> 5] = first; }
  __syncthreads();
  if (threadIdx.x == 0) {
    long long c = 0; int f = 0x7fffffff;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) { c += s_cnt[w]; f = min(f, s_first[w]); }
    if (c == 0) {
      write_outcome(out, 0, 0, 0, 0, 0, 0, 0, 0);
    } else {
      const int64_t key = rec[f * 4 + 1];
      const int64_t PQ = (int64_t)P * Q;
      write_outcome(out, 1, 1, key / PQ, (key % PQ) / Q, key % Q, rec[f * 4 + 2], rec[f * 4 + 3], c);
    }
  }
}

// FC, several N tiles: combine per-row partials over tiles; first mismatching
// valid row in M order (== reference (n, p*Q+q) order).
__global__ void fc_finalize_part_kernel(const int64_t* __restrict__ part, ActGeom g, int n_tiles,
                                        unsigned long long* __restrict__ scratch /*[2]: count, min m*/) {
  const int64_t rows = (int64_t)g.m_tiles * abed_dev::kBlockM;
  const int64_t HlWl = (int64_t)g.Hl * g.Wl;
  for (int64_t m = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; m < g.m_total; m += (int64_t)gridDim.x * blockDim.x) {
    const int64_t rem = m % HlWl;
    if (rem / g.Wl >= g.p || rem % g.Wl >= g.q) continue;
    long long lhs = 0, rhs = 0;
    for (int nt = 0; nt < n_tiles; ++nt) {
      lhs += part[((int64_t)nt * rows + m) * 2 + 0];
      rhs += part[((int64_t)nt * rows + m) * 2 + 1];
    }
    if (lhs != rhs) {
      atomicAdd(&scratch[0], 1ull);
      atomicMin(&scratch[1], (unsigned long long)m);
    }
  }
}
__global__ void fc_finalize_part2_kernel(const int64_t* __restrict__ part, ActGeom g, int n_tiles,
                                         const unsigned long long* __restrict__ scratch, abed_verify_outcome* out) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  const unsigned long long cnt = scratch[0];
  if (cnt == 0) { write_outcome(out, 0, 0, 0, 0, 0, 0, 0, 0); return; }
  const int64_t m = (int64_t)scratch[1];
  const int64_t rows = (int64_t)g.m_tiles * abed_dev::kBlockM;
  const int64_t HlWl = (int64_t)g.Hl * g.Wl;
  long long lhs = 0, rhs = 0;
  for (int nt = 0; nt < n_tiles; ++nt) {
    lhs += part[((int64_t)nt * rows + m) * 2 + 0];
    rhs += part[((int64_t)nt * rows + m) * 2 + 1];
  }
  const int64_t n = m / HlWl, rem = m % HlWl;
  write_outcome(out, 1, 1, n, rem / g.Wl, rem % g.Wl, lhs, rhs, (int64_t)cnt);
}

// FIC: lhs = sum of per-tile output sums; rhs = fic_dot (already reduced)
__global__ void fic_finalize_kernel(const int64_t* __restrict__ part, int n, const unsigned long long* __restrict__ rhs_p,
                                    abed_verify_outcome* out) {
  __shared__ long long red[32];
  long long s = 0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) s += part[i];
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    long long tot = 0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) tot += red[w];
    const long long rhs = (long long)*rhs_p;
    // checksum.hpp:287-294: Pass reports lhs = rhs = sum
    write_outcome(out, tot != rhs ? 1 : 0, 0, 0, 0, 0, tot, rhs, tot != rhs ? 1 : 0);
  }
}

// IC verdicts of many plans in two launches (blockIdx.y = plan): every plan's
// ic from its class sums, then every plan's ic_verify_k.  A pass of 16 IC
// layers was 32 dependent small launches (~25 us per layer of step time).
__global__ void __launch_bounds__(128) ic_from_classes_many_kernel(const __grid_constant__ IcVerdictBatch b) {
  const IcVerdictJob& j = b.job[blockIdx.y];
  if (j.copy_only || !j.S) return;  // input checksum computed ahead / kept (no class sums)
  const int64_t crs = j.crs;
  const int rs = j.R * j.Sd;
  long long dot = 0;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < crs; t += (int64_t)gridDim.x * blockDim.x) {
    const int c = (int)(t / rs), r = (int)((t / j.Sd) % j.R), sc = (int)(t % j.Sd);
    const int a = r % j.sh, bb = sc % j.sw, phase = a * j.nph_w + bb;
    long long v = 0;
    if (j.nrc <= 4 && j.ncc <= 4) {
      // unrolled over at most 4 x 4 classes: the (predicated) class-sum loads are
      // independent and issue together instead of one L2 round trip each
      long long part[4][4];
#pragma unroll
      for (int rc = 0; rc < 4; ++rc) {
        const bool rok = rc < j.nrc && ((j.rowmask[a * j.nrc + (rc < j.nrc ? rc : 0)] >> r) & 1ull);
#pragma unroll
        for (int cc = 0; cc < 4; ++cc) {
          const bool ok = rok && cc < j.ncc && ((j.colmask[bb * j.ncc + (cc < j.ncc ? cc : 0)] >> sc) & 1ull);
          part[rc][cc] = ok ? j.S[((int64_t)(phase * j.nrc + rc) * j.ncc + cc) * j.c256 + c] : 0ll;
        }
      }
#pragma unroll
      for (int rc = 0; rc < 4; ++rc)
#pragma unroll
        for (int cc = 0; cc < 4; ++cc) v += part[rc][cc];
    } else {
      for (int rc = 0; rc < j.nrc; ++rc) {
        if (!((j.rowmask[a * j.nrc + rc] >> r) & 1ull)) continue;
        for (int cc = 0; cc < j.ncc; ++cc)
          if ((j.colmask[bb * j.ncc + cc] >> sc) & 1ull) v += j.S[((int64_t)(phase * j.nrc + rc) * j.ncc + cc) * j.c256 + c];
      }
    }
    j.ic[t] = (int32_t)v;
    if (j.fsum) dot += (long long)j.fsum[t] * v;
  }
  if (j.fic_rhs) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) dot += __shfl_xor_sync(0xffffffffu, dot, o);
    if ((threadIdx.x & 31) == 0 && dot != 0) atomicAdd(j.fic_rhs, (unsigned long long)dot);
  }
}

// ic_verify_k (checksum.hpp:319-347) per plan: a warp per channel k (16-byte
// filter loads), count + first mismatching k into scr, the plan's last block
// (ticket) writes the outcome and resets scr
__global__ void __launch_bounds__(256) ic_finalize_many_kernel(const __grid_constant__ IcVerdictBatch b) {
  const IcVerdictJob& j = b.job[blockIdx.y];
  if (j.copy_only) {  // a second finalize of the same run
    if (blockIdx.x == 0 && threadIdx.x == 0) *j.out = *j.last;
    return;
  }
  __shared__ bool s_last;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  // the class sums were read by ic_from_classes: zero them for the next run
  if (j.S)
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < j.S_len; i += (int64_t)gridDim.x * blockDim.x)
      const_cast<int64_t*>(j.S)[i] = 0;
  const bool vec = (j.crs & 15) == 0 && (reinterpret_cast<uintptr_t>(j.f) & 15) == 0;
  for (int64_t k = (int64_t)blockIdx.x * nw + w; k < j.K; k += (int64_t)gridDim.x * nw) {
    long long dot = 0;
    const int8_t* fk = j.f + k * j.crs;
    if (vec) {
      for (int64_t i = (int64_t)lane * 16; i < j.crs; i += 32 * 16) {
        const int4 fv = __ldg(reinterpret_cast<const int4*>(fk + i));
        const int4 c0 = __ldg(reinterpret_cast<const int4*>(j.ic + i)), c1 = __ldg(reinterpret_cast<const int4*>(j.ic + i + 4));
        const int4 c2 = __ldg(reinterpret_cast<const int4*>(j.ic + i + 8)), c3 = __ldg(reinterpret_cast<const int4*>(j.ic + i + 12));
        const int cv[16] = {c0.x, c0.y, c0.z, c0.w, c1.x, c1.y, c1.z, c1.w, c2.x, c2.y, c2.z, c2.w, c3.x, c3.y, c3.z, c3.w};
        const uint32_t fw[4] = {(uint32_t)fv.x, (uint32_t)fv.y, (uint32_t)fv.z, (uint32_t)fv.w};
#pragma unroll
        for (int e = 0; e < 16; ++e)
          dot += (long long)(int8_t)(fw[e >> 2] >> (8 * (e & 3))) * cv[e];
      }
    } else {
      for (int64_t i = lane; i < j.crs; i += 32) dot += (long long)fk[i] * j.ic[i];
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) dot += __shfl_xor_sync(0xffffffffu, dot, o);
    if (lane == 0) {
      const long long lhs = (long long)j.ksum[k];
      j.ksum[k] = 0ull;  // consumed: the next run accumulates afresh
      j.scr[4 + k] = (unsigned long long)dot;
      j.scr[4 + j.K + k] = (unsigned long long)lhs;
      if (lhs != dot) {
        atomicAdd(&j.scr[0], 1ull);
        atomicMin(&j.scr[1], (unsigned long long)k);
      }
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    s_last = atomicAdd(&j.scr[2], 1ull) == gridDim.x - 1;
  }
  __syncthreads();
  if (!s_last || threadIdx.x != 0) return;
  __threadfence();
  const unsigned long long cnt = __ldcg(&j.scr[0]);
  if (cnt == 0) {
    write_outcome(j.out, 0, 0, 0, 0, 0, 0, 0, 0);
  } else {
    const int64_t k = (int64_t)__ldcg(&j.scr[1]);
    write_outcome(j.out, 1, 1, k, -1, -1, (long long)__ldcg(&j.scr[4 + j.K + k]), (long long)__ldcg(&j.scr[4 + k]),
                  (long long)cnt);
  }
  *j.last = *j.out;
  j.scr[0] = 0ull;
  j.scr[1] = ~0ull;
  j.scr[2] = 0ull;
}

void ic_verdict_many_launch(const IcVerdictJob* jobs, int n, cudaStream_t st) {
  for (int i = 0; i < n; i += kMaxIcJobs) {
    IcVerdictBatch b{};
    const int m = std::min(kMaxIcJobs, n - i);
    int64_t max_crs = 1, max_k = 1;
    for (int q = 0; q < m; ++q) {
      b.job[q] = jobs[i + q];
      if (jobs[i + q].S) max_crs = std::max(max_crs, jobs[i + q].crs);
      max_k = std::max(max_k, jobs[i + q].K);
    }
    const int gx = (int)std::min<int64_t>((max_crs + 127) / 128, 64);
    ic_from_classes_many_kernel<<<dim3(gx, m), 128, 0, st>>>(b);
    const int fx = (int)std::min<int64_t>((max_k + 7) / 8, 64);
    ic_finalize_many_kernel<<<dim3(fx, m), 256, 0, st>>>(b);
    cuda_check(cudaGetLastError(), "ic verdicts");
  }
}

// ---------------------------------------------------------------------------
// plan construction
// ---------------------------------------------------------------------------
// SM count of the CURRENT device (cached per ordinal: one process may drive several GPUs)
static int g_num_sms[64] = {};
int num_sms() {
  int dev = 0;
  cudaGetDevice(&dev);
  int* slot = (dev >= 0 && dev < 64) ? &g_num_sms[dev] : nullptr;
  if (slot && *slot > 0) return *slot;
  int n = 0;
  cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
  if (n <= 0) n = 148;
  if (slot) *slot = n;
  return n;
}

// compile-time unrolled MMA issue routine for this geometry (conv_tc.cu MmaPattern)
int mma_pattern_of(const ActGeom& g, int gps) {
  if (g.sh != g.sw || (g.sh != 1 && g.sh != 2) || (gps != 2 && gps != 4)) return 0;
  const int gi = gps == 4 ? 0 : 1;
  const int si = g.sh == 1 ? 0 : 2;
  if (g.r == 3 && g.s == 3) return 1 + si + gi;
  if (g.r == 1 && g.s == 1) return 5 + si + gi;
  return 0;
}

static constexpr uint32_t kSmemBudget = abed_dev::kConvDynSmemMax - 256;

// Cycles of one M=128 x K=32 SS-mode kind::i8 MMA with N columns, measured on
// B200 with warp-uniform issue (tools/mma_microbench2.cu,
// profiles/mma_microbench2_r01.txt): the tensor floor N/2, or the shared-memory
// operand read (A 4 KB + B 32*N bytes at 128 B/clk) when N < 128.
static double mma_cycles(int n) {
  double c = 0.0;
  while (n > 0) {
    const int part = n > 256 ? 256 : n;
    c += std::max(part / 2.0, (4096.0 + 32.0 * part) / 128.0) + 1.0;
    n -= part;
  }
  return c;
}

bool choose_tiling(const ActGeom& g, bool fc, int force_block_n, ConvTcParams& p, uint32_t reserve) {
  const uint32_t kBudget = kSmemBudget - reserve;  // minus the FIC-SM class table
  // Pick (block_n, channel groups per stage) minimising the modelled kernel time:
  // waves of persistent work units x MMAs per unit x cycles per MMA.
  const int ntaps = g.r * g.s;
  const int k_pad = (int)ceil_div(g.k, 16) * 16;
  const int strip = geom_strip_pix(g);
  const int fcrows = fc ? 16 : 0;
  const int sms = num_sms();
  auto a_stage = [&](int gps) { return (uint32_t)g.n_phase * gps * strip * 16u; };
  int best_tot = -1;
  double best_cost = 1e300;
  ConvTcParams best{};
  // one MMA covers the whole N tile (block_n + FC rows <= 256)
  for (int bn = std::min(k_pad, 256 - fcrows); bn >= 16; bn -= 16) {
    if (force_block_n && bn != force_block_n) continue;
    if (k_pad % bn) continue;
    const int tot = bn + fcrows;
    for (int gps : {4, 2}) {
      if (g.c16 % gps) continue;
      const uint32_t bstage = (uint32_t)tot * ntaps * gps * 16u;
      const uint32_t tab = 8u * ntaps * (gps / 2) + 512;
      // resident B (a CTA keeps its N tile's filters in smem)
      const uint32_t bres = bstage * (g.c16 / gps);
      int stages_res = 0;
      if (bres + tab < kBudget) stages_res = std::min<int>(abed_dev::kStages, (kBudget - bres - tab) / a_stage(gps));
      const int stages_ring = std::min<int>(abed_dev::kStages, (kBudget - tab) / (a_stage(gps) + bstage));
      const bool res_ok = stages_res >= 2;
      const bool ring_ok = stages_ring >= 2;
      if (!res_ok && !ring_ok) continue;
      const int n_tiles = k_pad / bn;
      int64_t waves;
      if (res_ok) {
        const int per = std::max(1, std::min(sms / n_tiles, g.m_tiles));
        waves = ceil_div(g.m_tiles, per);
      } else {
        waves = ceil_div((int64_t)g.m_tiles * n_tiles, sms);
      }
      const double per_unit = (double)ntaps * (g.c16 / 2) * mma_cycles(tot) + 300.0;
      double cost = waves * per_unit;
      if (!res_ok) cost *= 1.02;  // streamed B: extra L2 traffic per unit
      if (2 * ((tot + 31) & ~31) > 512) cost *= 1.10;  // single TMEM accumulator: no epilogue overlap
      if (cost >= best_cost * 0.999) continue;
      best_cost = cost;
      best_tot = tot;
      best = p;
      best.block_n = bn; best.block_n_tot = tot; best.gps = gps; best.n_tiles = n_tiles;
      best.k_stages = g.c16 / gps; best.b_stage_bytes = bstage;
      best.b_resident = res_ok ? 1 : 0;
      best.n_stages = res_ok ? stages_res : stages_ring;
    }
  }
  if (best_tot < 0) return false;
  p = best;
  return true;
}

}  // namespace abed_host
