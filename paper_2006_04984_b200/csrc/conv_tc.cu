// tcgen05 implicit-GEMM convolution: host launcher, verdict reduction kernel.
// The conv kernel itself lives in conv_tc_kernel.cuh (see its header comment);
// its (dtype, output flavour) variants are compiled in conv_inst_*.cu.
#include <algorithm>

#include "conv_tc_kernel.cuh"

namespace abed_host {
#define ABED_EXTERN_EPI(DT, EPI, XT) \
  extern template cudaError_t launch_epi<DT, EPI, XT>(const ConvTcParams&, int, bool, cudaStream_t);
#define ABED_EXTERN_DT(DT, XT)                 \
  ABED_EXTERN_EPI(DT, abed_dev::EPI_NONE, XT)  \
  ABED_EXTERN_EPI(DT, abed_dev::EPI_NCHW, XT)  \
  ABED_EXTERN_EPI(DT, abed_dev::EPI_PACKED, XT) \
  ABED_EXTERN_EPI(DT, abed_dev::EPI_COMPARE, XT)
ABED_EXTERN_DT(abed_dev::DT_I8, 0)
ABED_EXTERN_DT(abed_dev::DT_I8, 1)
ABED_EXTERN_DT(abed_dev::DT_I8, 2)
ABED_EXTERN_EPI(abed_dev::DT_I8, abed_dev::EPI_PACKED, 3)
ABED_EXTERN_DT(abed_dev::DT_I8, 4)
ABED_EXTERN_DT(abed_dev::DT_F16, 0)
ABED_EXTERN_DT(abed_dev::DT_BF16, 0)
}  // namespace abed_host

namespace abed_dev {
// ---------------------------------------------------------------- verdicts
// One block per plan: reduce the conv kernel's per-CTA records into the
// reference VerifyOutcomes -- FC: mismatch count and the first mismatching
// (n, p, q) in reference loop order with its lhs / rhs (fc_verify,
// checksum.hpp:211-236; fc_verify_f32 :541-565); FIC: lhs = sum of the outputs,
// rhs = fic_dot (fic_verify :287-294; fic_verify_f32 / float_verify :474-539).
__global__ void __launch_bounds__(256) verdict_kernel(const __grid_constant__ VerdictBatch b) {
  // a plain (stream-ordered) launch after the conv kernels; the wait is a no-op
  // then and only matters if a caller launches it as a programmatic dependent
  pdl_wait();
  const VerdictJob& j = b.job[blockIdx.x];
  const int t = threadIdx.x, lane = t & 31, w = t >> 5;
  __shared__ FcRec s_fc[8];
  __shared__ long long s_l[8], s_r[8];
  FcRec fc{0, kNoKey, 0, 0};
  long long li = 0, ri = 0;
  double lf = 0.0, rf = 0.0;
  if ((j.checks & CHECK_FC) && j.n_tiles > 1) {
    // full-channel row sums of the flagged M tiles (fc_verify, checksum.hpp:211-236)
    const int64_t HlWl = static_cast<int64_t>(j.Hl) * j.Wl;
    const int64_t PQ = static_cast<int64_t>(j.P) * j.Q;
    const int64_t stride = static_cast<int64_t>(j.m_tiles) * kBlockM * 2;
    // flags of the last run, one per (N tile, M tile, lane quarter), read by all
    // threads in parallel into a count of raised M tiles (usually zero: the
    // serial per-tile recheck below then costs nothing)
    const int64_t nflags = static_cast<int64_t>(j.n_tiles) * j.m_tiles * 4;
    int any = 0;
    for (int64_t i = t; i < nflags; i += blockDim.x) any |= __ldcg(j.tile_flag + i) != 0u;
    const bool some_raised = __syncthreads_or(any) != 0;
    for (int mt = 0; some_raised && mt < j.m_tiles; ++mt) {
      unsigned raised = 0;
      for (int i = 0; i < j.n_tiles * 4; ++i)
        raised |= j.tile_flag[(static_cast<int64_t>(i >> 2) * j.m_tiles + mt) * 4 + (i & 3)];
      if (!raised) continue;
      for (int r = t; r < kBlockM; r += blockDim.x) {
        const int64_t m = static_cast<int64_t>(mt) * kBlockM + r;
        if (m >= j.m_total) continue;
        const int64_t n = m / HlWl, rem = m % HlWl, pp = rem / j.Wl, qq = rem % j.Wl;
        if (pp >= j.P || qq >= j.Q) continue;
        const int64_t key = n * PQ + pp * j.Q + qq;
        const int64_t* q = j.fc_part + m * 2;
        if (j.dtype == DT_I8) {
          long long l = 0, rr = 0;
          for (int nt = 0; nt < j.n_tiles; ++nt) {
            l += __ldcg(q + nt * stride);
            rr += __ldcg(q + nt * stride + 1);
          }
          if (l != rr) fc_note(fc, key, l, rr);
        } else {
          double l = 0.0, rr = 0.0;
          for (int nt = 0; nt < j.n_tiles; ++nt) {
            l += __longlong_as_double(__ldcg(q + nt * stride));
            rr += __longlong_as_double(__ldcg(q + nt * stride + 1));
          }
          if (!(fabs(l - rr) <= j.tau_fc)) fc_note(fc, key, __double_as_longlong(l), __double_as_longlong(rr));
        }
      }
    }
  }
  for (int c = t; c < j.grid; c += blockDim.x) {
    const int64_t* rec = j.rec + static_cast<int64_t>(c) * kCtaRec;
    if (j.checks & CHECK_FC) {
      const int64_t cnt = rec[0];
      if (cnt > 0) {
        fc.cnt += cnt;
        if (rec[1] < fc.key) {
          fc.key = rec[1];
          fc.lhs = rec[2];
          fc.rhs = rec[3];
        }
      }
    }
    if (j.checks & CHECK_FIC) {
      if (j.dtype == DT_I8) {
        li += rec[4];
        ri += rec[5];
      } else {
        lf += __longlong_as_double(rec[4]);
        rf += __longlong_as_double(rec[5]);
      }
    }
  }
  fc = fc_warp_reduce(fc);
  li = warp_sum(li);
  ri = warp_sum(ri);
  lf = warp_sum_d(lf);
  rf = warp_sum_d(rf);
  if (lane == 0) {
    s_fc[w] = fc;
    s_l[w] = j.dtype == DT_I8 ? li : __double_as_longlong(lf);
    s_r[w] = j.dtype == DT_I8 ? ri : __double_as_longlong(rf);
  }
  __syncthreads();
  if (t != 0) return;
  FcRec r{0, kNoKey, 0, 0};
  long long L = 0, Rr = 0;
  double Lf = 0.0, Rf = 0.0;
  for (int q = 0; q < static_cast<int>(blockDim.x >> 5); ++q) {
    r.cnt += s_fc[q].cnt;
    if (s_fc[q].key < r.key) {
      r.key = s_fc[q].key;
      r.lhs = s_fc[q].lhs;
      r.rhs = s_fc[q].rhs;
    }
    L += s_l[q];
    Rr += s_r[q];
    Lf += __longlong_as_double(s_l[q]);
    Rf += __longlong_as_double(s_r[q]);
  }
  abed_verify_outcome* out = static_cast<abed_verify_outcome*>(j.out);
  if (j.checks & CHECK_FC) {
    const int64_t PQ = static_cast<int64_t>(j.P) * j.Q;
    if (r.cnt == 0) {
      write_outcome_dev(out + 0, 0, 0, 0, 0, 0, 0, 0, 0);
    } else if (j.dtype == DT_I8) {
      write_outcome_dev(out + 0, 1, 1, r.key / PQ, (r.key % PQ) / j.Q, r.key % j.Q, r.lhs, r.rhs, r.cnt);
    } else {
      write_outcome_dev(out + 0, 1, 1, r.key / PQ, (r.key % PQ) / j.Q, r.key % j.Q, 0, 0, r.cnt);
      out[0].lhs_f = __longlong_as_double(r.lhs);
      out[0].rhs_f = __longlong_as_double(r.rhs);
    }
  }
  if (j.icb) out[2] = *static_cast<const abed_verify_outcome*>(j.icb);  // ICBatch (icb_scan_kernel)
  if (j.checks & CHECK_FIC) {
    if (j.dtype == DT_I8) {
      long long rhs;
      if (j.rhs_mode == 2) {
        rhs = static_cast<long long>(*j.af_acc);
        *j.af_acc = 0ull;  // consumed: the next pass's producer accumulates afresh
      } else {
        // rhs_mode 1 / 3: the kernel's input-checksum warps; 0 / 4: computed ahead
        // (reused, or from the IC input checksum at the verdict) in rhs_ext
        rhs = (j.rhs_mode == 1 || j.rhs_mode == 3) ? Rr : static_cast<long long>(*j.rhs_ext);
      }
      // checksum.hpp:287-294: Pass reports lhs = rhs = sum
      write_outcome_dev(out + 1, L != rhs ? 1 : 0, 0, 0, 0, 0, L, rhs, L != rhs ? 1 : 0);
      // kept for later runs that reuse the pristine input checksum (campaigns)
      if (j.rhs_mode == 1 || j.rhs_mode == 3) *j.rhs_ext = static_cast<unsigned long long>(rhs);
    } else {
      const double rhs = j.rhs_mode ? Rf : *j.rhs_ext_f;
      const int bad = !(fabs(Lf - rhs) <= j.tau_fic);
      write_outcome_dev(out + 1, bad, 0, 0, 0, 0, 0, 0, bad);
      out[1].lhs_f = Lf;
      out[1].rhs_f = rhs;
      if (j.rhs_mode) *j.rhs_ext_f = rhs;
    }
  }
}

// ICBatch verdict (ic_batch_verify, checksum.hpp:398-421) after the fused conv:
// for every (k, p, q) the batch sum of the outputs (icb_lhs, accumulated by the
// epilogue) against conv_batch_checksum = sum_j 256^j conv(d_j) (icb_dig, the
// digit images' rows); mismatch count and the first mismatch in the reference's
// (k, p, q) order with its lhs / rhs.  Resets icb_lhs and the writer counter for
// the next run; the last block (ticket) folds the per-block records.
__global__ void __launch_bounds__(256) icb_scan_kernel(const __grid_constant__ IcbScanBatch b) {
  const IcbScanJob& j = b.job[blockIdx.y];
  unsigned long long* const lhs = j.lhs;
  const int32_t* const dig = j.dig;
  const int D = j.D, Q = j.Q;
  const int64_t kpq = j.kpq, PQ = j.PQ;
  int64_t* const rec = j.rec;
  unsigned int* const ctl = j.ctl;
  abed_verify_outcome* const out = static_cast<abed_verify_outcome*>(j.out);
  const int t = threadIdx.x, lane = t & 31, w = t >> 5;
  FcRec r{0, kNoKey, 0, 0};
  // 4 consecutive (k, p, q) per thread, every load of a group issued before use
  // (the scan is latency-bound: one dependent load chain per element is ~3x slower)
  const int64_t groups = (kpq + 3) / 4;
  for (int64_t gi = static_cast<int64_t>(blockIdx.x) * blockDim.x + t; gi < groups;
       gi += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t i0 = gi * 4;
    long long l[4], d0[4], d1[4], d2[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int64_t i = i0 + u;
      const bool ok = i < kpq;
      l[u] = ok ? static_cast<long long>(__ldcg(lhs + i)) : 0;
      d0[u] = ok ? __ldcg(dig + i) : 0;
      d1[u] = ok ? __ldcg(dig + kpq + i) : 0;
      d2[u] = (ok && D > 2) ? __ldcg(dig + 2 * kpq + i) : 0;
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int64_t i = i0 + u;
      if (i >= kpq) break;
      const long long rr = d0[u] + (d1[u] << 8) + (d2[u] << 16);
      if (l[u] != rr) fc_note(r, i, l[u], rr);
      lhs[i] = 0ull;
    }
  }
  __shared__ FcRec s_r[8];
  __shared__ bool s_last;
  r = fc_warp_reduce(r);
  if (lane == 0) s_r[w] = r;
  __syncthreads();
  if (t == 0) {
    FcRec b{0, kNoKey, 0, 0};
    for (int q = 0; q < static_cast<int>(blockDim.x >> 5); ++q) {
      b.cnt += s_r[q].cnt;
      if (s_r[q].key < b.key) b = FcRec{b.cnt, s_r[q].key, s_r[q].lhs, s_r[q].rhs};
    }
    int64_t* my = rec + static_cast<int64_t>(blockIdx.x) * 4;
    my[0] = b.cnt;
    my[1] = b.key;
    my[2] = b.lhs;
    my[3] = b.rhs;
    __threadfence();
    s_last = atomicAdd(&ctl[1], 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  FcRec a{0, kNoKey, 0, 0};
  for (int c = t; c < static_cast<int>(gridDim.x); c += blockDim.x) {
    const int64_t* q = rec + static_cast<int64_t>(c) * 4;
    const int64_t cnt = __ldcg(q);
    if (cnt > 0) {
      a.cnt += cnt;
      const int64_t key = __ldcg(q + 1);
      if (key < a.key) a = FcRec{a.cnt, key, __ldcg(q + 2), __ldcg(q + 3)};
    }
  }
  a = fc_warp_reduce(a);
  if (lane == 0) s_r[w] = a;
  __syncthreads();
  if (t != 0) return;
  FcRec f{0, kNoKey, 0, 0};
  for (int q = 0; q < static_cast<int>(blockDim.x >> 5); ++q) {
    f.cnt += s_r[q].cnt;
    if (s_r[q].key < f.key) f = FcRec{f.cnt, s_r[q].key, s_r[q].lhs, s_r[q].rhs};
  }
  if (f.cnt == 0)  // checksum.hpp:420 VerifyOutcome::ok()
    write_outcome_dev(out, 0, 0, 0, 0, 0, 0, 0, 0);
  else  // locus (k, p, q)
    write_outcome_dev(out, 1, 1, f.key / PQ, (f.key % PQ) / Q, f.key % Q, f.lhs, f.rhs, f.cnt);
  ctl[0] = 0u;  // icb_ready
  ctl[1] = 0u;  // ticket
}

}  // namespace abed_dev

// --------------------------------------------------------------------------
// host side launcher
// --------------------------------------------------------------------------
namespace abed_host {

using abed_dev::ConvTcParams;

uint32_t conv_tc_smem_bytes(const ConvTcParams& p) { return abed_dev::smem_layout(p).total; }

int conv_tc_grid(const ConvTcParams& p, int num_sms) {
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
  return grid;
}

template <int DT, int XT>
static cudaError_t launch_dt(const ConvTcParams& p, int grid, bool pdl, cudaStream_t stream) {
  switch (p.out_mode) {
    case abed_dev::OUT_NONE: return launch_epi<DT, abed_dev::EPI_NONE, XT>(p, grid, pdl, stream);
    case abed_dev::OUT_I8_PACKED:
    case abed_dev::OUT_H_PACKED: return launch_epi<DT, abed_dev::EPI_PACKED, XT>(p, grid, pdl, stream);
    case abed_dev::OUT_I8_COMPARE:
    case abed_dev::OUT_H_COMPARE: return launch_epi<DT, abed_dev::EPI_COMPARE, XT>(p, grid, pdl, stream);
    default: return launch_epi<DT, abed_dev::EPI_NCHW, XT>(p, grid, pdl, stream);
  }
}

cudaError_t verdict_launch(const abed_dev::VerdictJob* jobs, int n, cudaStream_t stream) {
  for (int i = 0; i < n; i += abed_dev::kMaxVerdictJobs) {
    abed_dev::VerdictBatch b{};
    b.n = n - i < abed_dev::kMaxVerdictJobs ? n - i : abed_dev::kMaxVerdictJobs;
    for (int k = 0; k < b.n; ++k) b.job[k] = jobs[i + k];
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(b.n);
    cfg.blockDim = dim3(256);
    cfg.stream = stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    // a plain launch: measured 5.5 -> 3.8 us per 16-layer pass against the
    // programmatic-dependent launch (its early-launched blocks only wait here)
    cfg.numAttrs = 0;
    const cudaError_t e = cudaLaunchKernelEx(&cfg, abed_dev::verdict_kernel, b);
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

cudaError_t icb_scan_launch(const abed_dev::IcbScanJob* jobs, int n, cudaStream_t stream) {
  for (int i = 0; i < n; i += abed_dev::kMaxIcbScanJobs) {
    abed_dev::IcbScanBatch b{};
    const int m = std::min(abed_dev::kMaxIcbScanJobs, n - i);
    int64_t max_kpq = 1;
    for (int q = 0; q < m; ++q) {
      b.job[q] = jobs[i + q];
      max_kpq = std::max(max_kpq, jobs[i + q].kpq);
    }
    int blocks = static_cast<int>((max_kpq + 1023) / 1024);
    if (blocks > abed_dev::kIcbScanBlocks) blocks = abed_dev::kIcbScanBlocks;
    // plain launch (as the verdict): one per finalize, for every ICBatch plan of the
    // pass (was one per run: 16 launches on the b32 step)
    abed_dev::icb_scan_kernel<<<dim3(blocks, m), 256, 0, stream>>>(b);
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

cudaError_t conv_tc_launch(const ConvTcParams& p_in, int num_sms, bool pdl, cudaStream_t stream) {
  ConvTcParams p = p_in;
  if (p.conv_grid <= 0) {
    p.conv_grid = conv_tc_grid(p, num_sms);
    p.ic_ctas = 0;
  }
  const int grid = p.conv_grid + p.ic_ctas;
  switch (p.dtype) {
    case abed_dev::DT_F16: return launch_dt<abed_dev::DT_F16, 0>(p, grid, pdl, stream);
    case abed_dev::DT_BF16: return launch_dt<abed_dev::DT_BF16, 0>(p, grid, pdl, stream);
    default:
      if (p.check & abed_dev::CHECK_IC) return launch_dt<abed_dev::DT_I8, 1>(p, grid, pdl, stream);
      if (p.rhs_mode == 3) return launch_dt<abed_dev::DT_I8, 4>(p, grid, pdl, stream);
      if (p.icb_d) return launch_dt<abed_dev::DT_I8, 2>(p, grid, pdl, stream);
      // FIC-AF producer: packed output dotted into the next layer's rhs
      if (p.af_ficw8 && p.out_mode == abed_dev::OUT_I8_PACKED)
        return launch_epi<abed_dev::DT_I8, abed_dev::EPI_PACKED, 3>(p, grid, pdl, stream);
      return launch_dt<abed_dev::DT_I8, 0>(p, grid, pdl, stream);
  }
}

}  // namespace abed_host
