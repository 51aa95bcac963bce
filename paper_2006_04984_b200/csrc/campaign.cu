// C ABI: tensor-core batch checksum, fused conv+epilog with taps, and the GPU
// fault-injection trial / campaign driver.
//
//  * abed_conv_batch_checksum (checksum.hpp:367-396): the ICBatch checksum image
//    sum_n x (|.| <= 128 N) is split into four balanced int8 digit images and
//    convolved on the tcgen05 path as an extra batch; the digit results are
//    recombined in int64 (linearity keeps it exact).
//  * abed_fused_conv_epilog (checksum.hpp:616-631): the protected plan with the
//    FIC reduction supplies the pre-epilog output checksum tap.
//  * abed_run_trial / abed_run_campaign (faults.hpp:197-333): golden run once,
//    then per trial one seeded single-bit flip applied IN DEVICE MEMORY (packed
//    input plane, packed filter block + the KCRS copy the IC verify reads, or the
//    ConvOut accumulator inside the fused epilogue), the fused conv with the
//    scheme's check, the epilog, and an on-device output compare.  Checksums
//    come from the pristine data (faults.hpp:111-115).  Trial seeds are
//    derive_seed(root, t), so reports are identical for any trial sharding.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <vector>

#include "abed_internal.h"

using namespace abed_host;
using abed_dev::ActGeom;

namespace {

constexpr uint64_t kGolden = 0x9E3779B97F4A7C15ULL;
uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}
struct HostRng {  // rng.hpp:11-37
  uint64_t s;
  uint64_t next() { return mix64(s += kGolden); }
  uint64_t below(uint64_t bound) {
    const uint64_t threshold = (0 - bound) % bound;
    for (;;) {
      const uint64_t r = next();
      if (r >= threshold) return r % bound;
    }
  }
};
uint64_t derive(uint64_t root, uint64_t i) { return HostRng{root ^ (0xA02E9D4BD1C96D4FULL + i * kGolden)}.next(); }

__global__ void digits_kernel(const int32_t* __restrict__ b, int64_t n, int8_t* __restrict__ d) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    int32_t v = b[i];
    for (int j = 0; j < 4; ++j) {  // v = sum_j d_j 256^j, d_j in [-128, 127]
      const int32_t dj = ((v + 128) & 0xFF) - 128;
      d[j * n + i] = (int8_t)dj;
      v = (v - dj) / 256;
    }
  }
}
__global__ void recombine_digits_kernel(const int32_t* __restrict__ e, int64_t n, int64_t* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = (int64_t)e[i] + (int64_t)e[n + i] * 256 + (int64_t)e[2 * n + i] * 65536 + (int64_t)e[3 * n + i] * 16777216;
}
__global__ void xor_byte_kernel(int8_t* a, int64_t ia, int8_t* b, int64_t ib, uint8_t mask) {
  if (a) a[ia] ^= (int8_t)mask;
  if (b) b[ib] ^= (int8_t)mask;
}
__global__ void differ_kernel(const uint4* __restrict__ a, const uint4* __restrict__ b, int64_t n16, int* flag) {
  int d = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n16; i += (int64_t)gridDim.x * blockDim.x) {
    const uint4 x = a[i], y = b[i];
    d |= (x.x != y.x) | (x.y != y.y) | (x.z != y.z) | (x.w != y.w);
  }
  if (__any_sync(0xffffffffu, d) && (threadIdx.x & 31) == 0) atomicOr(flag, 1);
}

template <typename T>
struct Dev {
  T* p = nullptr;
  explicit Dev(size_t n) { cuda_check(cudaMalloc(&p, (n ? n : 1) * sizeof(T)), "cudaMalloc"); }
  ~Dev() { cudaFree(p); }
  Dev(const Dev&) = delete;
  Dev& operator=(const Dev&) = delete;
};

struct PlanGuard {
  abed_conv_plan* p;
  ~PlanGuard() { abed_conv_plan_destroy(p); }
};

// run the tcgen05 conv over NCHW device tensors, int32 NCHW out
void tc_conv_nchw(const abed_layer_shape& s, const int8_t* x, const int8_t* f, int32_t* out, cudaStream_t st) {
  one_shot_run(s, 0, x, f, nullptr, ABED_OUT_I32_NCHW, out, nullptr, st);
  cuda_check(cudaStreamSynchronize(st), "tc_conv sync");
}

int scheme_checks(int scheme) {
  switch (scheme) {
    case ABED_FC: return ABED_CHECK_FC;
    case ABED_IC: return ABED_CHECK_IC;
    case ABED_FIC: return ABED_CHECK_FIC;
    default: throw_invalid("run_trial: batch-checksum IC is not an injection scheme");
  }
}
int scheme_slot(int scheme) { return scheme == ABED_FC ? 0 : scheme == ABED_FIC ? 1 : 2; }

// faults.hpp:116-130 TrialContext, device resident
struct GpuTrialCtx {
  abed_layer_shape s{};
  int scheme = 0, out_kind = ABED_I8;
  abed_conv_plan* plan = nullptr;
  int8_t* packed = nullptr;
  void* golden = nullptr;
  void* trial_out = nullptr;
  float* bias = nullptr;
  abed_epilog_params ep{};
  int64_t out_bytes = 0;
  ~GpuTrialCtx() {
    abed_conv_plan_destroy(plan);
    cudaFree(packed); cudaFree(golden); cudaFree(trial_out); cudaFree(bias);
  }
};

void ctx_make(GpuTrialCtx& c, const abed_layer_shape& s, const int8_t* x, const int8_t* f, int scheme, float scale,
              const float* bias_host, int64_t bias_len, int act, int kind, cudaStream_t st) {
  validate_shape(s);
  c.s = s;
  c.scheme = scheme;
  const int checks = scheme_checks(scheme);
  if (kind != ABED_I8 && kind != ABED_F32) throw_invalid("epilog: output kind must be i8 or f32");
  if (!std::isfinite(scale)) throw_invalid("epilog: non-finite scale");
  std::vector<float> hb((size_t)s.k, 0.0f);  // faults.hpp:167-168: empty bias -> zeros
  if (bias_host && bias_len > 0) {
    if (bias_len != s.k) throw_invalid("epilog: bias length must equal the channel count");
    for (int64_t i = 0; i < s.k; ++i) {
      if (!std::isfinite(bias_host[i])) throw_invalid("epilog: non-finite bias");
      hb[(size_t)i] = bias_host[i];
    }
  }
  c.out_kind = kind;
  cuda_check(cudaMalloc(&c.bias, (size_t)s.k * 4), "cudaMalloc(bias)");
  cuda_check(cudaMemcpy(c.bias, hb.data(), hb.size() * 4, cudaMemcpyHostToDevice), "bias h2d");
  c.ep = abed_epilog_params{scale, c.bias, s.k, act, kind};
  c.plan = plan_create(s, f, checks, 0);
  cuda_check(cudaMalloc(&c.packed, (size_t)geom_packed_bytes(c.plan->g)), "cudaMalloc(packed)");
  abed_pack_input(c.plan, x, c.packed, st);
  const int64_t nkpq = s.n * s.k * s.p * s.q;
  c.out_bytes = (nkpq * (kind == ABED_F32 ? 4 : 1) + 15) / 16 * 16;
  cuda_check(cudaMalloc(&c.golden, (size_t)c.out_bytes), "cudaMalloc(golden)");
  cuda_check(cudaMalloc(&c.trial_out, (size_t)c.out_bytes), "cudaMalloc(trial)");
  cuda_check(cudaMemsetAsync(c.golden, 0, (size_t)c.out_bytes, st), "memset");
  cuda_check(cudaMemsetAsync(c.trial_out, 0, (size_t)c.out_bytes, st), "memset");
  // golden run: checksums from the pristine input, golden output
  c.plan->reuse_input_checksum = 0;
  c.plan->pdl = 0;  // trials patch filter storage right before each run
  plan_run(c.plan, c.packed, &c.ep, kind == ABED_F32 ? ABED_OUT_F32_NCHW : ABED_OUT_I8_NCHW, c.golden, nullptr, -1, 0, st);
  {
    // the verdict reduction of the golden run keeps its FIC rhs (pristine input
    // checksum) for the trials, which reuse it (faults.hpp:111-115)
    Dev<abed_verify_outcome> scratch(3);
    plan_finalize(c.plan, scratch.p, st);
    cuda_check(cudaStreamSynchronize(st), "golden verdict");
  }
  c.plan->reuse_input_checksum = 1;
  cuda_check(cudaStreamSynchronize(st), "golden run");
}

// one trial, asynchronous; outcome -> out3 (3 slots), differs -> flag
void trial_enqueue(GpuTrialCtx& c, int target, int64_t flat, int bit, abed_verify_outcome* out3, int* flag,
                   cudaStream_t st) {
  const abed_layer_shape& s = c.s;
  const ActGeom& g = c.plan->g;
  const abed_dev::ConvTcParams& p = c.plan->base;
  int8_t* a = nullptr;
  int8_t* b = nullptr;
  int64_t ia = 0, ib = 0;
  int64_t fault_key = -1;
  const uint8_t mask = (uint8_t)(1u << (bit % 8));
  if (target == ABED_TARGET_INPUT) {
    const int64_t w = flat % s.w, h = (flat / s.w) % s.h, ch = (flat / (s.w * s.h)) % s.c, n = flat / (s.w * s.h * s.c);
    const int64_t hp = h + s.pad_h, wp = w + s.pad_w;
    const int ph_a = (int)(hp % s.stride_h), ph_b = (int)(wp % s.stride_w);
    if (ph_a < g.nph_h && ph_b < g.nph_w) {  // pixels of untouched phases are never read by the conv
      const int64_t t = (n * g.Hl + hp / s.stride_h) * g.Wl + wp / s.stride_w;
      const int64_t plane = (int64_t)(ph_a * g.nph_w + ph_b) * g.c16 + ch / 16;
      a = c.packed;
      ia = (plane * g.plane_len + t) * 16 + ch % 16;
    }
  } else if (target == ABED_TARGET_FILTER) {
    const int64_t ss = flat % s.s, r = (flat / s.s) % s.r, ch = (flat / (s.s * s.r)) % s.c, k = flat / (s.s * s.r * s.c);
    const int64_t nt = k / p.block_n, row = k % p.block_n, grp = ch / 16, ks = grp / p.gps, gl = grp % p.gps;
    const int64_t tap = r * s.s + ss;
    a = c.plan->d_wpk;
    ia = ((((nt * p.k_stages + ks) * p.ntaps + tap) * p.gps + gl) * p.block_n_tot + row) * 16 + ch % 16;
    b = c.plan->d_filters;  // the IC verify re-reads filter storage (faults.hpp:242-245)
    ib = flat;
  } else {
    fault_key = flat;
  }
  if (a || b) xor_byte_kernel<<<1, 1, 0, st>>>(a, ia, b, ib, mask);
  plan_run(c.plan, c.packed, &c.ep, c.out_kind == ABED_F32 ? ABED_OUT_F32_NCHW : ABED_OUT_I8_NCHW, c.trial_out, nullptr,
           fault_key, bit, st);
  plan_finalize(c.plan, out3, st);
  differ_kernel<<<grid_for(c.out_bytes / 16, 256), 256, 0, st>>>(static_cast<const uint4*>(c.trial_out),
                                                                 static_cast<const uint4*>(c.golden), c.out_bytes / 16, flag);
  if (a || b) xor_byte_kernel<<<1, 1, 0, st>>>(a, ia, b, ib, mask);  // restore pristine data
  cuda_check(cudaGetLastError(), "trial");
}

int classify(int verify_status, int differs) {  // faults.hpp:255-261
  if (verify_status == 0) return differs ? ABED_SDC : ABED_MASKED;
  return differs ? ABED_DETECTED : ABED_DETECTED_BENIGN;
}

void draw(uint64_t seed, const abed_layer_shape& s, int target, int64_t& flat, int& bit) {  // faults.hpp:200-208
  HostRng g{seed};
  const int64_t count = target == ABED_TARGET_INPUT ? s.n * s.c * s.h * s.w
                        : target == ABED_TARGET_FILTER ? s.k * s.c * s.r * s.s
                                                       : s.n * s.k * s.p * s.q;
  flat = (int64_t)g.below((uint64_t)count);
  bit = (int)g.below(target == ABED_TARGET_CONVOUT ? 32u : 8u);
}


// ---------------------------------------------------------------------------
// Trial-parallel campaign (faults.hpp:276-333 semantics, one CTA per trial).
// A single-bit flip perturbs a known, small set of ConvOut elements -- one
// element (ConvOut target), one channel's N x P x Q outputs scaled by the flipped
// filter byte's delta times the input patch values (filter target), or the
// K x (taps covering the pixel) outputs of one image (input target) -- so each
// trial is evaluated exactly from the golden int32 ConvOut, the pristine
// checksums and the perturbed elements alone, with the reference's int32
// ConvOut wrap, its int64 verify sums and its epilog:
//   FC  fc_verify (:211-236): row (n,p,q) sum vs the extra fmap.  The extra comes
//       from the pristine filter checksum over the (possibly flipped) patches, so
//       an input flip moves both sides by dx * fsum[c,r,s];
//   FIC fic_verify (:287-294): total sum vs the pristine fic_dot;
//   IC  ic_verify_k (:319-347): per-channel sums vs dot(filters used, pristine ic);
//       a filter flip moves both sides of channel k by df * ic[c,r,s];
//   output differs: epilog of every perturbed element vs its golden epilog.
// The exhaustive path above (abed_run_campaign) re-runs the fused protected conv
// per trial; tests check both give the same report.
struct BatchedCampaignArgs {
  abed_layer_shape s;    // this shard's layer (s.n = images of the shard)
  int scheme, target;
  int64_t n0, n_global;  // first global image of the shard, images of the whole batch
  const int8_t* x;       // NCHW, pristine (the shard's images)
  const int8_t* f;       // KCRS, pristine
  const int32_t* conv;   // golden ConvOut NKPQ of the shard
  const int32_t* fsum;   // gen_filter_checksum (c,r,s)
  const int32_t* ic;     // gen_input_checksum (c,r,s) of the shard's pristine input
  const float* bias;
  float scale;
  int relu, f32out;
  const int64_t* flat;   // per trial: flat index into the GLOBAL tensors, bit
  const int32_t* bit;
  int64_t n_trials;
  unsigned long long* counts;  // [4] by classification (ABED_DETECTED, _SDC, _MASKED, _DETECTED_BENIGN)
  long long* records;          // or, when non-null: per trial {hit, differs, total} of this shard
};

__device__ __forceinline__ uint32_t epi_bits(int32_t a, float scale, float b, int relu, int f32out) {
  float v = __fmaf_rn(static_cast<float>(a), scale, b);  // convolution.hpp:353-387 (FMA-contracted)
  if (relu && v < 0.0f) v = 0.0f;
  if (f32out) return __float_as_uint(v);
  return static_cast<uint32_t>(static_cast<int32_t>(truncf(fminf(127.0f, fmaxf(-128.0f, v))))) & 0xFFu;
}

__device__ __forceinline__ int32_t wrap_add(int32_t v, int64_t d) {  // int32 ConvOut of the flipped operands
  return static_cast<int32_t>(static_cast<uint32_t>(v) + static_cast<uint32_t>(static_cast<uint64_t>(d)));
}

// Decision of one trial from the (summed over shards) record {hit, differs, total}:
// FIC -- the ConvOut sum moved (total != 0); IC with a filter flip -- channel k's sum
// and its dot with the flipped filter moved by different amounts (total = their
// difference); otherwise a row (FC) / channel (IC) check failed somewhere (hit).
__host__ __device__ inline int classify_record(int scheme, int target, long long hit, long long differs,
                                               long long total) {
  const bool detected = scheme == ABED_FIC ? total != 0
                        : (scheme == ABED_IC && target == ABED_TARGET_FILTER) ? total != 0
                                                                              : hit != 0;
  return detected ? (differs ? ABED_DETECTED : ABED_DETECTED_BENIGN) : (differs ? ABED_SDC : ABED_MASKED);
}

__global__ void __launch_bounds__(256) campaign_batched_kernel(const __grid_constant__ BatchedCampaignArgs A) {
  const abed_layer_shape& s = A.s;
  const int64_t P = s.p, Q = s.q, PQ = P * Q, K = s.k, C = s.c, R = s.r, S = s.s;
  __shared__ long long sh_tap[64];  // FC, input target: per-tap (= per-(p,q)) delta of the row sum
  __shared__ int sh_flag[2];        // [0] a row / channel check failed, [1] output differs
  __shared__ long long sh_red[8];
  for (int64_t t = blockIdx.x; t < A.n_trials; t += gridDim.x) {
    const int64_t flat = A.flat[t];
    const int bit = A.bit[t];
    if (threadIdx.x < 64) sh_tap[threadIdx.x] = 0;
    if (threadIdx.x < 2) sh_flag[threadIdx.x] = 0;
    __syncthreads();
    int differs = 0, hit = 0;
    long long total = 0;
    // global image of an input / ConvOut flip (filter flips touch every shard)
    int64_t n_img = -1;
    if (A.target == ABED_TARGET_INPUT) n_img = flat / (C * s.h * s.w);
    if (A.target == ABED_TARGET_CONVOUT) n_img = flat / (K * PQ);
    const bool mine = A.target == ABED_TARGET_FILTER || (n_img >= A.n0 && n_img < A.n0 + s.n);
    if (!mine) {
      // another shard's image: nothing changes here
    } else if (A.target == ABED_TARGET_CONVOUT) {
      if (threadIdx.x == 0) {
        const int64_t lf = flat - A.n0 * K * PQ;
        const int64_t k = (lf / PQ) % K;
        const int32_t v = A.conv[lf];
        const int32_t v2 = static_cast<int32_t>(static_cast<uint32_t>(v) ^ (1u << bit));
        const long long d = static_cast<long long>(v2) - v;
        total = d;
        hit = d != 0;  // FC: its row; IC: its channel
        differs = epi_bits(v2, A.scale, A.bias[k], A.relu, A.f32out) != epi_bits(v, A.scale, A.bias[k], A.relu, A.f32out);
      }
    } else if (A.target == ABED_TARGET_FILTER) {
      const int64_t ss = flat % S, r = (flat / S) % R, c = (flat / (S * R)) % C, k = flat / (S * R * C);
      const int8_t f0 = A.f[flat];
      const long long df = static_cast<long long>(static_cast<int8_t>(f0 ^ static_cast<int8_t>(1 << bit))) - f0;
      const float b = A.bias[k];
      const int64_t npq = s.n * PQ;
      for (int64_t i = threadIdx.x; i < npq; i += blockDim.x) {
        const int64_t n = i / PQ, pq = i - n * PQ, pp = pq / Q, qq = pq - pp * Q;
        const int64_t h = pp * s.stride_h + r - s.pad_h, w = qq * s.stride_w + ss - s.pad_w;
        if (h < 0 || h >= s.h || w < 0 || w >= s.w) continue;
        const int8_t xv = A.x[((n * C + c) * s.h + h) * s.w + w];
        if (xv == 0) continue;
        const int64_t o = (n * K + k) * PQ + pq;
        const int32_t v = A.conv[o], v2 = wrap_add(v, df * xv);
        const long long d = static_cast<long long>(v2) - v;
        total += d;
        hit |= d != 0;  // FC: row (n,p,q) moves, its extra does not
        differs |= epi_bits(v2, A.scale, b, A.relu, A.f32out) != epi_bits(v, A.scale, b, A.relu, A.f32out);
      }
      if (A.scheme == ABED_IC) hit = 0;  // decided on total (channel sum vs dot) below
    } else {
      const int64_t w0 = flat % s.w, h0 = (flat / s.w) % s.h, c = (flat / (s.w * s.h)) % C, n = n_img - A.n0;
      const int8_t x0 = A.x[flat - A.n0 * C * s.h * s.w];
      const long long dx = static_cast<long long>(static_cast<int8_t>(x0 ^ static_cast<int8_t>(1 << bit))) - x0;
      const int taps = static_cast<int>(R * S);
      for (int64_t k = threadIdx.x; k < K; k += blockDim.x) {
        const float b = A.bias[k];
        long long ksum = 0;
        for (int tap = 0; tap < taps; ++tap) {
          const int64_t r = tap / S, ss = tap - r * S;
          const int64_t hp = h0 + s.pad_h - r, wp = w0 + s.pad_w - ss;
          if (hp < 0 || wp < 0 || hp % s.stride_h || wp % s.stride_w) continue;
          const int64_t pp = hp / s.stride_h, qq = wp / s.stride_w;
          if (pp >= P || qq >= Q) continue;
          const int8_t fv = A.f[((k * C + c) * R + r) * S + ss];
          if (fv == 0) continue;
          const int64_t o = (n * K + k) * PQ + pp * Q + qq;
          const int32_t v = A.conv[o], v2 = wrap_add(v, dx * fv);
          const long long d = static_cast<long long>(v2) - v;
          ksum += d;
          if (A.scheme == ABED_FC && d) atomicAdd(reinterpret_cast<unsigned long long*>(&sh_tap[tap]),
                                                  static_cast<unsigned long long>(d));
          differs |= epi_bits(v2, A.scale, b, A.relu, A.f32out) != epi_bits(v, A.scale, b, A.relu, A.f32out);
        }
        total += ksum;
        if (A.scheme == ABED_IC) hit |= ksum != 0;  // channel k's sum moves, its dot does not
      }
    }
    // block reductions: hit / differs (or), total (sum)
    if (hit) sh_flag[0] = 1;
    if (differs) sh_flag[1] = 1;
    long long tsum = total;
#pragma unroll
    for (int o = 16; o; o >>= 1) tsum += __shfl_xor_sync(0xffffffffu, tsum, o);
    if ((threadIdx.x & 31) == 0) sh_red[threadIdx.x >> 5] = tsum;
    __syncthreads();
    if (threadIdx.x == 0) {
      long long tot = 0;
      for (int w = 0; w < static_cast<int>(blockDim.x >> 5); ++w) tot += sh_red[w];
      long long rhit = sh_flag[0];
      if (mine && A.scheme == ABED_FC && A.target == ABED_TARGET_INPUT) {
        // per covering tap: the row sum moved by sh_tap[tap], the extra fmap by dx * fsum[c,r,s]
        const int64_t w0 = flat % s.w, h0 = (flat / s.w) % s.h, c = (flat / (s.w * s.h)) % C;
        const int8_t x0 = A.x[flat - A.n0 * C * s.h * s.w];
        const long long dx = static_cast<long long>(static_cast<int8_t>(x0 ^ static_cast<int8_t>(1 << bit))) - x0;
        rhit = 0;
        for (int tap = 0; tap < static_cast<int>(R * S); ++tap) {
          const int64_t r = tap / S, ss = tap - r * S;
          const int64_t hp = h0 + s.pad_h - r, wp = w0 + s.pad_w - ss;
          if (hp < 0 || wp < 0 || hp % s.stride_h || wp % s.stride_w || hp / s.stride_h >= P || wp / s.stride_w >= Q)
            continue;
          if (sh_tap[tap] != dx * static_cast<long long>(A.fsum[(c * R + r) * S + ss])) rhit = 1;
        }
      } else if (mine && A.scheme == ABED_IC && A.target == ABED_TARGET_FILTER) {
        // channel k: this shard's sum moved by tot, its share of dot(flipped filter, ic) by df * ic[c,r,s]
        const int64_t crs = flat % (C * R * S);
        const int8_t f0 = A.f[flat];
        const long long df = static_cast<long long>(static_cast<int8_t>(f0 ^ static_cast<int8_t>(1 << bit))) - f0;
        tot -= df * static_cast<long long>(A.ic[crs]);
      }
      if (A.records) {
        long long* rec = A.records + 3 * t;
        rec[0] = rhit;
        rec[1] = sh_flag[1];
        rec[2] = tot;
      } else {
        atomicAdd(A.counts + classify_record(A.scheme, A.target, rhit, sh_flag[1], tot), 1ull);  // faults.hpp:255-261
      }
    }
    __syncthreads();
  }
}

// classification counts of summed per-trial records (after the cross-shard all-reduce)
__global__ void campaign_classify_kernel(const long long* __restrict__ rec, int64_t n, int scheme, int target,
                                         unsigned long long* counts) {
  __shared__ unsigned long long c[4];
  if (threadIdx.x < 4) c[threadIdx.x] = 0;
  __syncthreads();
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x)
    atomicAdd(&c[classify_record(scheme, target, rec[3 * t], rec[3 * t + 1], rec[3 * t + 2])], 1ull);
  __syncthreads();
  if (threadIdx.x < 4 && c[threadIdx.x]) atomicAdd(counts + threadIdx.x, c[threadIdx.x]);
}

}  // namespace

// device-resident campaign (one batch shard): data, golden ConvOut, pristine
// checksums and every trial's flip drawn once; runs are single launches over
// trial ranges
struct abed_campaign {
  abed_campaign_config cfg{};
  abed_layer_shape shard{};  // cfg.shape restricted to images [n0, n0 + shard.n)
  int64_t n0 = 0;
  int8_t* x = nullptr;
  int8_t* f = nullptr;
  int32_t* conv = nullptr;
  int32_t* fsum = nullptr;
  int32_t* ic = nullptr;
  float* bias = nullptr;
  int64_t* flat = nullptr;
  int32_t* bit = nullptr;
  unsigned long long* counts = nullptr;
  ~abed_campaign() {
    cudaFree(x); cudaFree(f); cudaFree(conv); cudaFree(fsum); cudaFree(ic); cudaFree(bias);
    cudaFree(flat); cudaFree(bit); cudaFree(counts);
  }
};

namespace {

abed_campaign* campaign_create(const abed_campaign_config& cfg, int64_t n_begin, int64_t n_end) {
  if (cfg.trials < 1) throw_invalid("run_campaign: trials must be >= 1");
  const abed_layer_shape& s = cfg.shape;
  validate_shape(s);
  scheme_checks(cfg.scheme);  // ICBatch is not an injection scheme
  if (cfg.target < ABED_TARGET_INPUT || cfg.target > ABED_TARGET_CONVOUT) throw_invalid("run_campaign: bad target");
  if (cfg.output_kind != ABED_I8 && cfg.output_kind != ABED_F32) throw_invalid("epilog: output kind must be i8 or f32");
  if (!std::isfinite(cfg.scale)) throw_invalid("epilog: non-finite scale");
  if (s.r * s.s > 64) throw_invalid("run_campaign: filters with more than 64 taps are not supported");
  if (n_begin < 0 || n_end > s.n || n_begin >= n_end) throw_invalid("campaign: bad image shard");
  std::vector<float> hb((size_t)s.k, 0.0f);  // faults.hpp:167-168: empty bias -> zeros
  if (cfg.bias_host && cfg.bias_len > 0) {
    if (cfg.bias_len != s.k) throw_invalid("epilog: bias length must equal the channel count");
    for (int64_t i = 0; i < s.k; ++i) {
      if (!std::isfinite(cfg.bias_host[i])) throw_invalid("epilog: non-finite bias");
      hb[(size_t)i] = cfg.bias_host[i];
    }
  }
  auto* c = new abed_campaign();
  c->cfg = cfg;
  c->cfg.bias_host = nullptr;
  c->shard = s;
  c->shard.n = n_end - n_begin;
  c->n0 = n_begin;
  try {
    cudaStream_t st = nullptr;
    const abed_layer_shape& sh = c->shard;
    const int64_t chw = s.c * s.h * s.w, nchw = sh.n * chw, kcrs = s.k * s.c * s.r * s.s, crs = s.c * s.r * s.s;
    const int64_t nkpq = sh.n * s.k * s.p * s.q;
    cuda_check(cudaMalloc(&c->x, (size_t)nchw), "cudaMalloc(x)");
    cuda_check(cudaMalloc(&c->f, (size_t)kcrs), "cudaMalloc(f)");
    cuda_check(cudaMalloc(&c->conv, (size_t)nkpq * 4), "cudaMalloc(conv)");
    cuda_check(cudaMalloc(&c->fsum, (size_t)crs * 4), "cudaMalloc(fsum)");
    cuda_check(cudaMalloc(&c->ic, (size_t)crs * 4), "cudaMalloc(ic)");
    cuda_check(cudaMalloc(&c->bias, (size_t)s.k * 4), "cudaMalloc(bias)");
    cuda_check(cudaMalloc(&c->flat, (size_t)cfg.trials * 8), "cudaMalloc(flat)");
    cuda_check(cudaMalloc(&c->bit, (size_t)cfg.trials * 4), "cudaMalloc(bit)");
    cuda_check(cudaMalloc(&c->counts, 4 * 8), "cudaMalloc(counts)");
    cuda_check(cudaMemcpy(c->bias, hb.data(), hb.size() * 4, cudaMemcpyHostToDevice), "bias h2d");
    if (cfg.mode == ABED_DATA_ONES) {  // faults.hpp:280-283
      cuda_check(cudaMemset(c->x, 1, (size_t)nchw), "memset");
      cuda_check(cudaMemset(c->f, 1, (size_t)kcrs), "memset");
    } else {  // faults.hpp:284-288: one stream, input then filters (the shard's slice of it)
      const uint64_t seed = derive(cfg.root_seed, 0x0DA7Au);
      abed_fill_random_i8(c->x, nchw, seed, (uint64_t)(n_begin * chw), st);
      abed_fill_random_i8(c->f, kcrs, seed, (uint64_t)(s.n * chw), st);
    }
    tc_conv_nchw(sh, c->x, c->f, c->conv, st);  // golden ConvOut on the tensor cores
    dev_colsum_i8(c->f, s.k, crs, c->fsum, st);
    dev_gen_input_checksum(c->x, sh, c->ic, st);
    std::vector<int64_t> hf((size_t)cfg.trials);
    std::vector<int32_t> hbit((size_t)cfg.trials);
    for (int64_t t = 0; t < cfg.trials; ++t) {  // faults.hpp:200-208, seeds derive_seed(root, t), global tensors
      int b;
      draw(derive(cfg.root_seed, (uint64_t)t), s, cfg.target, hf[(size_t)t], b);
      hbit[(size_t)t] = b;
    }
    cuda_check(cudaMemcpy(c->flat, hf.data(), hf.size() * 8, cudaMemcpyHostToDevice), "flat h2d");
    cuda_check(cudaMemcpy(c->bit, hbit.data(), hbit.size() * 4, cudaMemcpyHostToDevice), "bit h2d");
    cuda_check(cudaDeviceSynchronize(), "campaign golden");
  } catch (...) {
    delete c;
    throw;
  }
  return c;
}

void campaign_run(abed_campaign* c, int64_t t_begin, int64_t t_end, unsigned long long* counts, long long* records,
                  cudaStream_t st) {
  if (t_begin < 0) t_begin = 0;
  if (t_end > c->cfg.trials) t_end = c->cfg.trials;
  const int64_t nt = t_end > t_begin ? t_end - t_begin : 0;
  if (!nt) return;
  BatchedCampaignArgs a{};
  a.s = c->shard;
  a.scheme = c->cfg.scheme;
  a.target = c->cfg.target;
  a.n0 = c->n0;
  a.n_global = c->cfg.shape.n;
  a.x = c->x; a.f = c->f; a.conv = c->conv; a.fsum = c->fsum; a.ic = c->ic; a.bias = c->bias;
  a.scale = c->cfg.scale;
  a.relu = c->cfg.activation == ABED_RELU ? 1 : 0;
  a.f32out = c->cfg.output_kind == ABED_F32 ? 1 : 0;
  a.flat = c->flat + t_begin;
  a.bit = c->bit + t_begin;
  a.n_trials = nt;
  a.counts = counts;
  a.records = records;
  const int64_t grid = nt < (int64_t)num_sms() * 8 ? nt : (int64_t)num_sms() * 8;
  campaign_batched_kernel<<<(unsigned)grid, 256, 0, st>>>(a);
  cuda_check(cudaGetLastError(), "campaign_batched");
}

void fill_report(const abed_campaign_config& cfg, int64_t nt, const unsigned long long* h, abed_campaign_report* rep) {
  std::memset(rep, 0, sizeof(*rep));
  rep->scheme = cfg.scheme; rep->target = cfg.target; rep->seed = cfg.root_seed; rep->trials = nt;
  rep->detected = (int64_t)h[ABED_DETECTED];
  rep->sdc = (int64_t)h[ABED_SDC];
  rep->masked = (int64_t)h[ABED_MASKED];
  rep->detected_benign = (int64_t)h[ABED_DETECTED_BENIGN];
}

}  // namespace

#define GUARD(...)              \
  try {                         \
    require_device();           \
    __VA_ARGS__;                \
    return ABED_OK;             \
  } catch (const AbedError& e) { \
    return set_error(e.code, e.what()); \
  } catch (const std::exception& e) { \
    return set_error(ABED_ERR_RUNTIME, e.what()); \
  }

extern "C" {

int abed_conv_batch_checksum(const int32_t* batch, const int8_t* filters, const abed_layer_shape* shape, int64_t* out,
                             void* stream) {
  GUARD(
      validate_shape(*shape); cudaStream_t st = (cudaStream_t)stream;
      abed_layer_shape four = *shape; four.n = 4;  // four digit images as one batch
      const int64_t chw = shape->c * shape->h * shape->w, kpq = shape->k * shape->p * shape->q;
      Dev<int8_t> dig((size_t)(4 * chw)); Dev<int32_t> e((size_t)(4 * kpq));
      digits_kernel<<<grid_for(chw, 256), 256, 0, st>>>(batch, chw, dig.p);
      tc_conv_nchw(four, dig.p, filters, e.p, st);
      recombine_digits_kernel<<<grid_for(kpq, 256), 256, 0, st>>>(e.p, kpq, out);
      cuda_check(cudaGetLastError(), "conv_batch_checksum"));
}

int abed_fused_conv_epilog(const int8_t* x, const int8_t* f, const abed_layer_shape* s, const abed_epilog_params* ep,
                           void* out, int64_t* out_checksum, const abed_layer_shape* next, int32_t* next_ic, void* stream) {
  GUARD(
      validate_shape(*s); cudaStream_t st = (cudaStream_t)stream;
      if (s->c * s->r * s->s > 65536) throw_invalid("conv_direct: CRS > 65536 exceeds the int32 accumulator plan");
      if (ep->bias_len != s->k) throw_invalid("epilog: bias length must equal the channel count");
      if (!std::isfinite(ep->scale)) throw_invalid("epilog: non-finite scale");
      {
        std::vector<float> hb((size_t)s->k);
        cuda_check(cudaMemcpy(hb.data(), ep->bias, hb.size() * 4, cudaMemcpyDeviceToHost), "bias d2h");
        for (float v : hb) if (!std::isfinite(v)) throw_invalid("epilog: non-finite bias");
      }
      if (ep->output_kind != ABED_I8 && ep->output_kind != ABED_F32) throw_invalid("epilog: output kind must be i8 or f32");
      // cached plan (FIC on only for the output-checksum tap: the FIC lhs is the
      // sum of the ConvOut before the epilog)
      Dev<abed_verify_outcome> oc(out_checksum ? 3 : 1);
      one_shot_run(*s, out_checksum ? ABED_CHECK_FIC : 0, x, f, ep,
                   ep->output_kind == ABED_F32 ? ABED_OUT_F32_NCHW : ABED_OUT_I8_NCHW, out,
                   out_checksum ? oc.p : nullptr, st);
      if (out_checksum) {
        abed_verify_outcome h;
        cuda_check(cudaMemcpyAsync(&h, oc.p + 1, sizeof(h), cudaMemcpyDeviceToHost, st), "d2h");
        cuda_check(cudaStreamSynchronize(st), "sync");
        *out_checksum = h.lhs;
      }
      if (next) {  // checksum.hpp:623-629 AF tap
        if (ep->output_kind != ABED_I8) throw_invalid("fused_conv_epilog: next-layer checksum tap needs an i8 epilog");
        if (next->n != s->n || next->c != s->k || next->h != s->p || next->w != s->q)
          throw_invalid("fused_conv_epilog: next-layer shape does not match the output");
        dev_gen_input_checksum(static_cast<const int8_t*>(out), *next, next_ic, st);
      }
      cuda_check(cudaStreamSynchronize(st), "fused sync"));
}

int abed_run_trial(const abed_layer_shape* s, const int8_t* x, const int8_t* f, int32_t scheme, int32_t target,
                   float scale, const float* bias_host, int64_t bias_len, int32_t act, int32_t kind, uint64_t seed,
                   abed_trial_outcome* out) {
  GUARD(
      cudaStream_t st = nullptr; GpuTrialCtx c;
      ctx_make(c, *s, x, f, scheme, scale, bias_host, bias_len, act, kind, st);
      int64_t flat; int bit; draw(seed, *s, target, flat, bit);
      Dev<abed_verify_outcome> oc(3); Dev<int> flag(1);
      cuda_check(cudaMemset(flag.p, 0, 4), "memset");
      trial_enqueue(c, target, flat, bit, oc.p, flag.p, st);
      abed_verify_outcome h[3]; int differs = 0;
      cuda_check(cudaMemcpy(h, oc.p, sizeof(h), cudaMemcpyDeviceToHost), "d2h");
      cuda_check(cudaMemcpy(&differs, flag.p, 4, cudaMemcpyDeviceToHost), "d2h");
      std::memset(out, 0, sizeof(*out));
      out->target = target; out->flat_index = flat; out->bit = bit; out->final_output_differs = differs;
      out->verify = h[scheme_slot(scheme)];
      out->classification = classify(out->verify.status, differs));
}

int abed_run_campaign(const abed_campaign_config* cfg, int64_t t_begin, int64_t t_end, abed_campaign_report* rep) {
  GUARD(
      if (cfg->trials < 1) throw_invalid("run_campaign: trials must be >= 1");
      const abed_layer_shape& s = cfg->shape; validate_shape(s);
      cudaStream_t st = nullptr;
      const int64_t nchw = s.n * s.c * s.h * s.w, kcrs = s.k * s.c * s.r * s.s;
      Dev<int8_t> x((size_t)nchw), f((size_t)kcrs);
      if (cfg->mode == ABED_DATA_ONES) {
        cuda_check(cudaMemset(x.p, 1, (size_t)nchw), "memset"); cuda_check(cudaMemset(f.p, 1, (size_t)kcrs), "memset");
      } else {  // faults.hpp:284-288: one stream, input then filters
        const uint64_t seed = derive(cfg->root_seed, 0x0DA7Au);
        abed_fill_random_i8(x.p, nchw, seed, 0, st);
        abed_fill_random_i8(f.p, kcrs, seed, (uint64_t)nchw, st);
      }
      GpuTrialCtx c;
      ctx_make(c, s, x.p, f.p, cfg->scheme, cfg->scale, cfg->bias_host, cfg->bias_len, cfg->activation, cfg->output_kind, st);
      if (t_begin < 0) t_begin = 0;
      if (t_end > cfg->trials) t_end = cfg->trials;
      const int64_t nt = t_end > t_begin ? t_end - t_begin : 0;
      Dev<abed_verify_outcome> oc((size_t)(3 * nt)); Dev<int> flags((size_t)nt);
      cuda_check(cudaMemset(flags.p, 0, (size_t)(nt ? nt : 1) * 4), "memset");
      for (int64_t t = 0; t < nt; ++t) {
        int64_t flat; int bit; draw(derive(cfg->root_seed, (uint64_t)(t_begin + t)), s, cfg->target, flat, bit);
        trial_enqueue(c, cfg->target, flat, bit, oc.p + 3 * t, flags.p + t, st);
      }
      std::vector<abed_verify_outcome> h((size_t)(3 * nt)); std::vector<int> hf((size_t)nt);
      if (nt) {
        cuda_check(cudaMemcpy(h.data(), oc.p, h.size() * sizeof(abed_verify_outcome), cudaMemcpyDeviceToHost), "d2h");
        cuda_check(cudaMemcpy(hf.data(), flags.p, hf.size() * 4, cudaMemcpyDeviceToHost), "d2h");
      }
      std::memset(rep, 0, sizeof(*rep));
      rep->scheme = cfg->scheme; rep->target = cfg->target; rep->seed = cfg->root_seed; rep->trials = nt;
      const int slot = scheme_slot(cfg->scheme);
      for (int64_t t = 0; t < nt; ++t) {  // fold in trial order (faults.hpp:319-331)
        switch (classify(h[(size_t)(3 * t + slot)].status, hf[(size_t)t])) {
          case ABED_DETECTED: ++rep->detected; break;
          case ABED_DETECTED_BENIGN: ++rep->detected_benign; break;
          case ABED_SDC: ++rep->sdc; break;
          default: ++rep->masked; break;
        }
      });
}

int abed_campaign_create(const abed_campaign_config* config, abed_campaign** campaign) {
  GUARD(if (!config || !campaign) throw_invalid("campaign: null argument");
        *campaign = campaign_create(*config, 0, config->shape.n));
}

int abed_campaign_create_shard(const abed_campaign_config* config, int64_t image_begin, int64_t image_end,
                               abed_campaign** campaign) {
  GUARD(if (!config || !campaign) throw_invalid("campaign: null argument");
        *campaign = campaign_create(*config, image_begin, image_end));
}

int abed_campaign_run_records(abed_campaign* campaign, int64_t trial_begin, int64_t trial_end, int64_t* records_dev,
                              void* stream) {
  GUARD(if (!campaign || !records_dev) throw_invalid("campaign: null argument");
        campaign_run(campaign, trial_begin, trial_end, nullptr, reinterpret_cast<long long*>(records_dev),
                     (cudaStream_t)stream));
}

int abed_campaign_classify(const abed_campaign* campaign, const int64_t* records_dev, int64_t n_records,
                           int64_t* counts_dev, void* stream) {
  GUARD(if (!campaign || !records_dev || !counts_dev) throw_invalid("campaign: null argument");
        if (n_records > 0) {
          const int blocks = (int)std::min<int64_t>((n_records + 255) / 256, 148);
          campaign_classify_kernel<<<blocks, 256, 0, (cudaStream_t)stream>>>(
              reinterpret_cast<const long long*>(records_dev), n_records, campaign->cfg.scheme, campaign->cfg.target,
              reinterpret_cast<unsigned long long*>(counts_dev));
          cuda_check(cudaGetLastError(), "campaign classify");
        });
}

int abed_campaign_destroy(abed_campaign* campaign) {
  GUARD(delete campaign);
}

int abed_campaign_run(abed_campaign* campaign, int64_t trial_begin, int64_t trial_end, int64_t* counts_dev,
                      void* stream) {
  GUARD(if (!campaign || !counts_dev) throw_invalid("campaign: null argument");
        if (campaign->shard.n != campaign->cfg.shape.n)
          throw_invalid("campaign: a batch shard reports per-trial records (abed_campaign_run_records)");
        campaign_run(campaign, trial_begin, trial_end, reinterpret_cast<unsigned long long*>(counts_dev), nullptr,
                     (cudaStream_t)stream));
}

int abed_campaign_report_of(const abed_campaign* campaign, const int64_t* counts_host, int64_t trials,
                            abed_campaign_report* report) {
  GUARD(if (!campaign || !counts_host || !report) throw_invalid("campaign: null argument");
        fill_report(campaign->cfg, trials, reinterpret_cast<const unsigned long long*>(counts_host), report));
}

int abed_run_campaign_batched(const abed_campaign_config* cfg, int64_t t_begin, int64_t t_end,
                              abed_campaign_report* rep) {
  GUARD(
      if (!cfg || !rep) throw_invalid("campaign: null argument");
      abed_campaign* c = campaign_create(*cfg, 0, cfg->shape.n);
      try {
        cuda_check(cudaMemset(c->counts, 0, 32), "memset counts");
        campaign_run(c, t_begin, t_end, c->counts, nullptr, nullptr);
        unsigned long long h[4];
        cuda_check(cudaMemcpy(h, c->counts, 32, cudaMemcpyDeviceToHost), "counts d2h");
        const int64_t b = t_begin < 0 ? 0 : t_begin, e = t_end > cfg->trials ? cfg->trials : t_end;
        fill_report(*cfg, e > b ? e - b : 0, h, rep);
      } catch (...) {
        delete c;
        throw;
      }
      delete c);
}

}  // extern "C"
