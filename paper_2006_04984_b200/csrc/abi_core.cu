// C ABI: library utilities, the protected-conv plan (hot path) and the
// reference-facing convolution entry points built on it.
#include <cuda_runtime.h>
#include <memory>
#include <list>
#include <mutex>

#include <algorithm>
#include <vector>
#include <cmath>
#include <cstring>
#include <string>

#include "abed_internal.h"

using namespace abed_host;
using abed_dev::ActGeom;
using abed_dev::ConvTcParams;

namespace abed_host {
thread_local std::string g_last_error;

int set_error(int code, const std::string& msg) {
  g_last_error = msg;
  return code;
}


void require_device() {
  // checked per device ordinal (a process may drive several GPUs)
  static int ok_dev[64];
  static bool init = false;
  if (!init) {
    for (int& v : ok_dev) v = -1;
    init = true;
  }
  int dev = 0, n = 0, ok = 0;
  if (cudaGetDeviceCount(&n) == cudaSuccess && n > 0 && cudaGetDevice(&dev) == cudaSuccess) {
    if (dev >= 0 && dev < 64 && ok_dev[dev] >= 0) {
      ok = ok_dev[dev];
    } else {
      int major = 0;
      cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev);
      ok = major == 10 ? 1 : 0;
      if (dev >= 0 && dev < 64) ok_dev[dev] = ok;
    }
  }
  if (!ok) throw AbedError(ABED_ERR_NO_DEVICE, "abed: no sm_100 (B200) device available; the library has no host fallback");
}

int grid_for(int64_t n, int threads = 256) {
  int64_t g = (n + threads - 1) / threads;
  const int cap = num_sms() * 16;
  if (g > cap) g = cap;
  if (g < 1) g = 1;
  return (int)g;
}

void validate_shape(const abed_layer_shape& s) {
  if (s.n < 1 || s.c < 1 || s.h < 1 || s.w < 1 || s.k < 1 || s.r < 1 || s.s < 1)
    throw_invalid("LayerShape: extents must be >= 1");
  if (s.stride_h < 1 || s.stride_w < 1) throw_invalid("LayerShape: strides must be >= 1");
  if (s.pad_h < 0 || s.pad_w < 0) throw_invalid("LayerShape: pads must be >= 0");
  if (s.r > s.h + 2 * s.pad_h || s.s > s.w + 2 * s.pad_w)
    throw_invalid("LayerShape: filter exceeds padded input");
  if (s.p != (s.h + 2 * s.pad_h - s.r) / s.stride_h + 1 || s.q != (s.w + 2 * s.pad_w - s.s) / s.stride_w + 1)
    throw_invalid("LayerShape: p/q inconsistent with extents");
}

// ---------------------------------------------------------------- plan
void plan_init_common(abed_conv_plan* pl, const abed_layer_shape& shape, int checks, int force_bn, int cpg) {
  pl->shape = shape;
  pl->checks = checks;
  if (checks & ~(ABED_CHECK_FC | ABED_CHECK_FIC | ABED_CHECK_IC | ABED_CHECK_ICBATCH))
    throw_invalid("conv plan: unknown check bits");
  int n_extra = 0;
  if (checks & ABED_CHECK_ICBATCH) {
    // ic_batch_checksum / conv_batch_checksum / ic_batch_verify fused (checksum.hpp:350-421)
    if (cpg != 16) throw_invalid("ICBatch: the fused batch checksum is an int8 scheme");
    if (checks & ABED_CHECK_IC) throw_invalid("ICBatch and IC share the third verdict slot: choose one");
    if (shape.n > 65536) throw_invalid("ICBatch: batch too large for the 3-digit batch-sum image");
    n_extra = shape.n <= 256 ? 2 : 3;  // balanced base-256 digits of sum_n x in [-128 N, 127 N]
  }
  pl->g = make_geom(shape, cpg, n_extra);
  const ActGeom& g = pl->g;
  ConvTcParams& p = pl->base;
  std::memset(&p, 0, sizeof(p));
  // int8 FIC: shared memory for the staged input checksum's class table
  const uint32_t fic_smem = (cpg == 16 && (checks & ABED_CHECK_FIC)) ? fic_classes_host(pl) : 0u;
  // IC: per-CTA shared per-channel output sums (K int64)
  const uint32_t ic_smem = (checks & ABED_CHECK_IC) ? (uint32_t)((shape.k * 8 + 15) & ~15) : 0u;
  const uint32_t ic_res = ic_smem ? ic_smem + 16 : 0u;  // + alignment
  bool tiled = choose_tiling(g, (checks & ABED_CHECK_FC) != 0, force_bn, p, fic_smem + ic_res);
  if (tiled && fic_smem) {
    p.fic_smem = fic_smem;
    p.fic_tab_bytes = (uint32_t)(pl->h_rep.size() * g.c16 * 48);
  } else if (fic_smem) {
    pl->h_rep.clear();  // no room: FIC keeps the FR re-read
    tiled = choose_tiling(g, (checks & ABED_CHECK_FC) != 0, force_bn, p, ic_res);
  }
  if (tiled && ic_smem) p.ic_smem = ic_smem;
  if (!tiled) throw_invalid("conv: no tiling fits shared memory for this layer");
  p.plane_len = g.plane_len;
  p.n_phase = g.n_phase;
  p.c16 = g.c16;
  p.strip_pix = geom_strip_pix(g);
  p.ntaps = g.r * g.s;
  p.R = g.r; p.S = g.s; p.sh = g.sh; p.sw = g.sw; p.nph_w = g.nph_w;
  p.mma_pattern = mma_pattern_of(g, p.gps);
  for (int r = 0; r < g.r; ++r)
    for (int s = 0; s < g.s; ++s) {
      const int t = r * g.s + s;
      p.tap_phase[t] = (r % g.sh) * g.nph_w + (s % g.sw);
      p.tap_shift[t] = (r / g.sh) * g.Wl + (s / g.sw);
      p.tap_a16[t] = (uint32_t)(p.tap_phase[t] * p.gps * p.strip_pix + p.tap_shift[t]);
    }
  p.m_total = g.m_total;
  p.m_real = (int64_t)g.n * g.Hl * g.Wl;
  p.m_tiles = g.m_tiles;
  p.Hl = g.Hl; p.Wl = g.Wl; p.P = g.p; p.Q = g.q; p.N = g.n; p.K = g.k;
  p.fault_key = -1;
  if (p.n_tiles > 1) {
    cuda_check(cudaMalloc(&pl->d_fc_part, (size_t)p.n_tiles * p.m_tiles * 128 * 2 * 8), "cudaMalloc(fc_part)");
    // int8: per-(N tile, M tile, lane quarter) FC flags; float: per-M-tile counters
    const size_t sem_bytes = (size_t)p.n_tiles * p.m_tiles * 4 * 4;
    cuda_check(cudaMalloc(&pl->d_tile_sem, sem_bytes), "cudaMalloc(tile_sem)");
    cuda_check(cudaMemset(pl->d_tile_sem, 0, sem_bytes), "memset tile_sem");
  }
  // one record per CTA of any launch (conv CTAs + input-checksum CTAs <= SMs)
  cuda_check(cudaMalloc(&pl->d_cta_rec, (size_t)std::max(num_sms(), conv_tc_grid(p, num_sms())) * abed_dev::kCtaRec * 8),
             "cudaMalloc(cta_rec)");
  pl->last_grid = conv_tc_grid(p, num_sms());
  cuda_check(cudaMalloc(&pl->d_kacc, 4 * 8), "cudaMalloc(kacc)");
  cuda_check(cudaMemset(pl->d_kacc, 0, 4 * 8), "memset kacc");
  cuda_check(cudaMalloc(&pl->d_outcome, 3 * sizeof(abed_verify_outcome)), "cudaMalloc(outcome)");
  cuda_check(cudaMemset(pl->d_outcome, 0, 3 * sizeof(abed_verify_outcome)), "memset outcome");
  cuda_check(cudaMalloc(&pl->d_acc, (4 + shape.k) * 8), "cudaMalloc(acc)");
  cuda_check(cudaMemset(pl->d_acc, 0, (4 + shape.k) * 8), "memset acc");
  cuda_check(cudaMalloc(&pl->d_zero_bias, shape.k * 4), "cudaMalloc(bias)");
  cuda_check(cudaMemset(pl->d_zero_bias, 0, shape.k * 4), "memset bias");
  cuda_check(cudaMalloc(&pl->d_af_acc, 8), "cudaMalloc(af_acc)");
  cuda_check(cudaMemset(pl->d_af_acc, 0, 8), "memset af_acc");
  if (checks & ABED_CHECK_IC) {
    // {count, first k, ticket, -, dot[K], lhs[K]}
    cuda_check(cudaMalloc(&pl->d_ic_scr, (4 + 2 * shape.k) * 8), "cudaMalloc(ic_scr)");
    const unsigned long long init[4] = {0ull, ~0ull, 0ull, 0ull};
    cuda_check(cudaMemcpy(pl->d_ic_scr, init, sizeof(init), cudaMemcpyHostToDevice), "ic_scr init");
    cuda_check(cudaMalloc(&pl->d_ic_last, sizeof(abed_verify_outcome)), "cudaMalloc(ic_last)");
    cuda_check(cudaMemset(pl->d_ic_last, 0, sizeof(abed_verify_outcome)), "memset ic_last");
  }
  if (n_extra) {
    const size_t kpq = (size_t)shape.k * shape.p * shape.q;
    cuda_check(cudaMalloc(&pl->d_icb_lhs, kpq * 8), "cudaMalloc(icb_lhs)");
    cuda_check(cudaMemset(pl->d_icb_lhs, 0, kpq * 8), "memset icb_lhs");
    cuda_check(cudaMalloc(&pl->d_icb_dig, kpq * 4 * n_extra), "cudaMalloc(icb_dig)");
    cuda_check(cudaMalloc(&pl->d_icb_ctl, 8), "cudaMalloc(icb_ctl)");
    cuda_check(cudaMemset(pl->d_icb_ctl, 0, 8), "memset icb_ctl");
    cuda_check(cudaMalloc(&pl->d_icb_rec, (size_t)abed_dev::kIcbScanBlocks * 4 * 8), "cudaMalloc(icb_rec)");
    cuda_check(cudaMalloc(&pl->d_icb_out, sizeof(abed_verify_outcome)), "cudaMalloc(icb_out)");
    cuda_check(cudaMemset(pl->d_icb_out, 0, sizeof(abed_verify_outcome)), "memset icb_out");
  }
}

// Position classes of a plane axis: phase row i is reached by the filter rows
// {r : r % st == a, 0 <= i - r / st < P}; rows with equal sets share a class.
// cls[a * L + i] = class id, masks[a * ncls + id] = its filter-row bit mask.
static void axis_classes(int L, int R, int st, int P, int nph, std::vector<uint8_t>& cls, std::vector<uint64_t>& masks,
                         int& ncls) {
  cls.assign((size_t)nph * L, 0);
  std::vector<std::vector<uint64_t>> m(nph);
  for (int a = 0; a < nph; ++a)
    for (int i = 0; i < L; ++i) {
      uint64_t b = 0;
      for (int r = 0; r < R; ++r)
        if (r % st == a && i - r / st >= 0 && i - r / st < P) b |= uint64_t(1) << r;
      int id = -1;
      for (size_t k = 0; k < m[a].size(); ++k)
        if (m[a][k] == b) id = (int)k;
      if (id < 0) {
        id = (int)m[a].size();
        m[a].push_back(b);
      }
      cls[(size_t)a * L + i] = (uint8_t)std::min(id, 255);
    }
  ncls = 0;
  for (int a = 0; a < nph; ++a) ncls = std::max(ncls, (int)m[a].size());
  masks.assign((size_t)nph * ncls, 0);
  for (int a = 0; a < nph; ++a)
    for (size_t k = 0; k < m[a].size(); ++k) masks[(size_t)a * ncls + k] = m[a][k];
}

// IC input checksum in-kernel: classes, masks and the class-sum buffer
static void build_ic_classes(abed_conv_plan* pl) {
  const ActGeom& g = pl->g;
  std::vector<uint8_t> rc, cc;
  std::vector<uint64_t> rm, cm;
  axis_classes(g.Hl, g.r, g.sh, g.p, g.nph_h, rc, rm, pl->ic_nrc);
  axis_classes(g.Wl, g.s, g.sw, g.q, g.nph_w, cc, cm, pl->ic_ncc);
  if (pl->ic_nrc > 255 || pl->ic_ncc > 255 || g.r > 64 || g.s > 64) throw_invalid("IC: too many position classes");
  cuda_check(cudaMalloc(&pl->d_ic_cls, rc.size() + cc.size()), "cudaMalloc(ic_cls)");
  cuda_check(cudaMemcpy(pl->d_ic_cls, rc.data(), rc.size(), cudaMemcpyHostToDevice), "ic_cls h2d");
  cuda_check(cudaMemcpy(pl->d_ic_cls + rc.size(), cc.data(), cc.size(), cudaMemcpyHostToDevice), "ic_cls h2d");
  cuda_check(cudaMalloc(&pl->d_ic_mask, (rm.size() + cm.size()) * 8), "cudaMalloc(ic_mask)");
  cuda_check(cudaMemcpy(pl->d_ic_mask, rm.data(), rm.size() * 8, cudaMemcpyHostToDevice), "ic_mask h2d");
  cuda_check(cudaMemcpy(pl->d_ic_mask + rm.size(), cm.data(), cm.size() * 8, cudaMemcpyHostToDevice), "ic_mask h2d");
  pl->ic_S_bytes = (size_t)g.n_phase * pl->ic_nrc * pl->ic_ncc * g.c16 * 16 * 8;
  cuda_check(cudaMalloc(&pl->d_ic_S, pl->ic_S_bytes), "cudaMalloc(ic_S)");
  cuda_check(cudaMemset(pl->d_ic_S, 0, pl->ic_S_bytes), "memset ic_S");
}

// IC verdict job: ic (+ FIC rhs) from the class sums, then ic_verify_k
// The run's in-kernel sums (class sums S, per-channel output sums) are consumed
// -- and zeroed -- by this verdict, so runs need no memsets; a second finalize of
// the same run repeats the stored outcome.
static IcVerdictJob ic_verdict_job(abed_conv_plan* pl, abed_verify_outcome* out, cudaStream_t st) {
  const ActGeom& g = pl->g;
  IcVerdictJob j{};
  j.last = pl->d_ic_last;
  j.out = out;
  if (!pl->ic_pending) {
    j.copy_only = 1;
    return j;
  }
  pl->ic_pending = 0;
  if (pl->d_ic_S && pl->last_rhs_mode == 4) {  // (reuse runs keep the earlier ic)
    const bool fic = (pl->checks & ABED_CHECK_FIC) != 0;
    if (fic) cuda_check(cudaMemsetAsync(pl->d_acc, 0, 8, st), "memset rhs");
    j.S = pl->d_ic_S;
    j.rowmask = pl->d_ic_mask;
    j.colmask = pl->d_ic_mask + (size_t)g.nph_h * pl->ic_nrc;
    j.nrc = pl->ic_nrc; j.ncc = pl->ic_ncc;
    j.R = g.r; j.Sd = g.s; j.sh = g.sh; j.sw = g.sw; j.nph_w = g.nph_w; j.c256 = g.c16 * 16;
    j.fsum = fic ? pl->d_fsum : nullptr;
    j.fic_rhs = fic ? pl->d_acc : nullptr;
    j.S_len = (int64_t)(pl->ic_S_bytes / 8);
  }
  j.ic = pl->d_ic;
  j.ksum = pl->d_acc + 4;
  j.f = pl->d_filters;
  j.K = pl->shape.k;
  j.crs = pl->shape.c * pl->shape.r * pl->shape.s;
  j.scr = pl->d_ic_scr;
  return j;
}
static void ic_verdict(abed_conv_plan* pl, abed_verify_outcome* out, cudaStream_t st) {
  const IcVerdictJob j = ic_verdict_job(pl, out, st);
  ic_verdict_many_launch(&j, 1, st);
}

// FIC-SM class table.  A phase row i is reached by the filter rows
// {r : r % sh == a, 0 <= i - r / sh < P} (the same test fic_weight_kernel applies
// per pixel); rows with equal sets share one class, likewise columns, so G is a
// function of (phase, row class, column class, channel).  The table copies G
// from one representative pixel per class pair (rows / columns never reached
// get a class whose G is zero).
uint32_t fic_classes_host(abed_conv_plan* pl) {
  const ActGeom& g = pl->g;
  if (g.n_phase > 4) return 0;  // the kernel's staged path handles up to 2 x 2 stride phases
  auto classes = [](int L, int R, int st, int P, int nph, std::vector<uint8_t>& cls, std::vector<int>& rep, int& ncls) {
    cls.assign((size_t)nph * L, 0);
    ncls = 0;
    std::vector<std::vector<uint64_t>> masks(nph);
    std::vector<std::vector<int>> reps(nph);
    for (int a = 0; a < nph; ++a) {
      for (int i = 0; i < L; ++i) {
        uint64_t m = 0;
        for (int r = 0; r < R; ++r)
          if (r % st == a && i - r / st >= 0 && i - r / st < P) m |= uint64_t(1) << r;
        int id = -1;
        for (size_t k = 0; k < masks[a].size(); ++k)
          if (masks[a][k] == m) id = (int)k;
        if (id < 0) {
          id = (int)masks[a].size();
          masks[a].push_back(m);
          reps[a].push_back(i);
        }
        cls[(size_t)a * L + i] = (uint8_t)std::min(id, 255);
      }
      ncls = std::max(ncls, (int)masks[a].size());
    }
    rep.assign((size_t)nph * ncls, -1);
    for (int a = 0; a < nph; ++a)
      for (size_t k = 0; k < reps[a].size(); ++k) rep[(size_t)a * ncls + k] = reps[a][k];
  };
  std::vector<int> rrep, crep;
  int nrc = 0, ncc = 0;
  classes(g.Hl, g.r, g.sh, g.p, g.nph_h, pl->h_rowcls, rrep, nrc);
  classes(g.Wl, g.s, g.sw, g.q, g.nph_w, pl->h_colcls, crep, ncc);
  // + one all-zero cell that pixels outside the images point at (branch-free kernel loop)
  const uint64_t tab = ((uint64_t)g.n_phase * nrc * ncc + 1) * g.c16 * 48;
  if (nrc > 255 || ncc > 255 || tab > 48 * 1024) return 0;  // keep the FR re-read
  // representative plane pixel (or -1) of every (phase, row class, column class)
  pl->h_rep.assign((size_t)g.n_phase * nrc * ncc, -1);
  for (int ph = 0; ph < g.n_phase; ++ph) {
    const int a = ph / g.nph_w, b = ph % g.nph_w;
    for (int i = 0; i < nrc; ++i)
      for (int j = 0; j < ncc; ++j) {
        const int ri = rrep[(size_t)a * nrc + i], cj = crep[(size_t)b * ncc + j];
        if (ri >= 0 && cj >= 0) pl->h_rep[((size_t)ph * nrc + i) * ncc + j] = ri * g.Wl + cj;
      }
  }
  pl->h_rep.push_back(-1);  // the zero cell
  pl->nrc = nrc;
  pl->ncc = ncc;
  return (uint32_t)(tab + ((pl->h_rowcls.size() + 15) & ~size_t(15)) + ((pl->h_colcls.size() + 15) & ~size_t(15)));
}

// FIC-SM class table.  A phase row i is reached by the filter rows
// {r : r % sh == a, 0 <= i - r / sh < P} (the test fic_weight_kernel applies per
// pixel); rows with equal sets share one class, likewise columns, so G is a
// function of (phase, row class, column class, channel).  The table copies G
// from one representative pixel per class pair (rows / columns never reached
// get a class whose G is zero).  The conv kernel keeps the table and the class
// arrays in shared memory (ConvTcParams::fic_smem, reserved by choose_tiling).
void build_fic_classes(abed_conv_plan* pl) {
  // one buffer [table | row classes (16-B padded) | column classes (padded)],
  // copied into shared memory by one bulk copy per CTA
  const ActGeom& g = pl->g;
  const std::vector<int>& rep = pl->h_rep;
  const ConvTcParams& p = pl->base;
  int* d_rep = nullptr;
  cuda_check(cudaMalloc(&d_rep, rep.size() * 4), "cudaMalloc(rep)");
  cuda_check(cudaMemcpy(d_rep, rep.data(), rep.size() * 4, cudaMemcpyHostToDevice), "rep h2d");
  const int64_t cells = (int64_t)rep.size() * g.c16;
  cuda_check(cudaMalloc(&pl->d_ficc8, p.fic_smem), "cudaMalloc(ficc8)");
  cuda_check(cudaMemset(pl->d_ficc8, 0, p.fic_smem), "memset ficc8");
  fic_class_table_kernel<<<grid_for(cells * 48), 256>>>(pl->d_ficw8, g, d_rep, (int)rep.size(), pl->d_ficc8);
  cuda_check(cudaGetLastError(), "fic_class_table");
  pl->d_rowcls = reinterpret_cast<uint8_t*>(pl->d_ficc8) + p.fic_tab_bytes;
  pl->d_colcls = pl->d_rowcls + ((pl->h_rowcls.size() + 15) & ~size_t(15));
  cuda_check(cudaMemcpy(pl->d_rowcls, pl->h_rowcls.data(), pl->h_rowcls.size(), cudaMemcpyHostToDevice), "rowcls h2d");
  cuda_check(cudaMemcpy(pl->d_colcls, pl->h_colcls.data(), pl->h_colcls.size(), cudaMemcpyHostToDevice), "colcls h2d");
  cuda_check(cudaDeviceSynchronize(), "fic classes sync");
  cudaFree(d_rep);
}

// ---------------------------------------------------------------- one-shot plan cache
// abed_conv_i8 (the reference's conv_fast_i8 / conv_direct, called once per
// layer by reference code) keeps an unchecked plan + packed-input buffer per
// (device, shape); at most kOneShotCap entries per device (oldest evicted).
struct OneShot {
  abed_layer_shape shape{};
  int device = -1;
  int checks = 0;
  abed_conv_plan* plan = nullptr;
  int8_t* packed = nullptr;
  std::mutex mu;
};
constexpr size_t kOneShotCap = 8;
static std::mutex g_one_shot_mu;
static std::list<std::unique_ptr<OneShot>> g_one_shot;

static bool same_shape(const abed_layer_shape& a, const abed_layer_shape& b) {
  return a.n == b.n && a.c == b.c && a.h == b.h && a.w == b.w && a.k == b.k && a.r == b.r && a.s == b.s &&
         a.stride_h == b.stride_h && a.stride_w == b.stride_w && a.pad_h == b.pad_h && a.pad_w == b.pad_w;
}

// returns the entry with its mutex held by `hold` (taken under the cache mutex, so
// an entry in use is never evicted)
OneShot& one_shot_acquire(const abed_layer_shape& shape, int checks, std::unique_lock<std::mutex>& hold) {
  int dev = 0;
  cuda_check(cudaGetDevice(&dev), "cudaGetDevice");
  std::lock_guard<std::mutex> lock(g_one_shot_mu);
  for (auto it = g_one_shot.begin(); it != g_one_shot.end(); ++it)
    if ((*it)->device == dev && (*it)->checks == checks && same_shape((*it)->shape, shape)) {
      g_one_shot.splice(g_one_shot.begin(), g_one_shot, it);  // most recent first
      hold = std::unique_lock<std::mutex>(g_one_shot.front()->mu);
      return *g_one_shot.front();
    }
  auto e = std::make_unique<OneShot>();
  e->shape = shape;
  e->device = dev;
  e->checks = checks;
  int8_t* zeros = nullptr;
  const int64_t fbytes = shape.k * shape.c * shape.r * shape.s;
  cuda_check(cudaMalloc(&zeros, (size_t)fbytes), "cudaMalloc(filters)");
  cuda_check(cudaMemset(zeros, 0, (size_t)fbytes), "memset filters");
  try {
    e->plan = plan_create(shape, zeros, checks, 0);
    // one-shot FIC plans serve the output-checksum tap only (fused_conv_epilog):
    // the kernel skips the input pass
    e->plan->reuse_input_checksum = 1;
    cuda_check(cudaMalloc(&e->packed, geom_packed_bytes(e->plan->g)), "cudaMalloc(packed)");
  } catch (...) {
    cudaFree(zeros);
    if (e->plan) abed_conv_plan_destroy(e->plan);
    throw;
  }
  cudaFree(zeros);
  if (g_one_shot.size() >= kOneShotCap) {
    // evict the oldest entry of this device that no call is using
    for (auto it = std::prev(g_one_shot.end());; --it) {
      if ((*it)->device == dev && (*it)->mu.try_lock()) {
        (*it)->mu.unlock();
        abed_conv_plan_destroy((*it)->plan);
        cudaFree((*it)->packed);
        g_one_shot.erase(it);
        break;
      }
      if (it == g_one_shot.begin()) break;
    }
  }
  g_one_shot.push_front(std::move(e));
  hold = std::unique_lock<std::mutex>(g_one_shot.front()->mu);
  return *g_one_shot.front();
}

// One reference-style call on the cached plan: re-pack the filters (they may
// change between calls), pack the input, run; with outcomes_dev the plan's
// verdicts (FIC: lhs = the sum of the ConvOut) follow.  Stream-ordered.
void one_shot_run(const abed_layer_shape& shape, int checks, const int8_t* input, const int8_t* filters,
                  const abed_epilog_params* ep, int out_mode, void* out, abed_verify_outcome* outcomes_dev,
                  cudaStream_t st) {
  std::unique_lock<std::mutex> hold;
  OneShot& o = one_shot_acquire(shape, checks, hold);
  abed_conv_plan* pl = o.plan;
  const ConvTcParams& p = pl->base;
  const int64_t rows = (int64_t)p.n_tiles * p.k_stages * p.ntaps * p.gps * p.block_n_tot;
  pack_filters_kernel<<<grid_for(rows, 256), 256, 0, st>>>(filters, pl->g, p.block_n, p.block_n_tot, p.n_tiles, p.gps,
                                                           p.k_stages, 0, pl->d_wpk);
  launch_pack_input(input, pl->g, o.packed, st);
  plan_run(pl, o.packed, ep, out_mode, out, nullptr, -1, 0, st);
  if (outcomes_dev) plan_finalize(pl, outcomes_dev, st);
  cuda_check(cudaGetLastError(), "one-shot conv");
}

abed_conv_plan* plan_create(const abed_layer_shape& shape, const int8_t* filters, int checks, int force_bn) {
  require_device();
  validate_shape(shape);
  if (shape.c * shape.r * shape.s > 65536)
    throw_invalid("conv: CRS > 65536 exceeds the int32 accumulator plan");
  if (shape.r * shape.s > abed_dev::kMaxTaps) throw_invalid("conv: filters with more than 64 taps are not supported");
  if (shape.k > (int64_t(1) << 24)) throw_invalid("gen_filter_checksum: K too large for i32 checksums");
  auto* pl = new abed_conv_plan();
  try {
    plan_init_common(pl, shape, checks, force_bn, 16);
    const ActGeom& g = pl->g;
    ConvTcParams& p = pl->base;
    const int64_t crs = shape.c * shape.r * shape.s;
    const size_t wpk_bytes = (size_t)p.n_tiles * p.k_stages * p.b_stage_bytes;
    cuda_check(cudaMalloc(&pl->d_wpk, wpk_bytes), "cudaMalloc(wpk)");
    cuda_check(cudaMalloc(&pl->d_filters, (size_t)(shape.k * crs)), "cudaMalloc(filters)");
    cuda_check(cudaMemcpy(pl->d_filters, filters, (size_t)(shape.k * crs), cudaMemcpyDeviceToDevice), "copy filters");
    cuda_check(cudaMalloc(&pl->d_fsum, crs * 4), "cudaMalloc(fsum)");
    cuda_check(cudaMalloc(&pl->d_ic, crs * 4), "cudaMalloc(ic)");
    cuda_check(cudaMalloc(&pl->d_bsum, (size_t)g.n_phase * g.c16 * 16 * g.Hl * g.Wl * 4), "cudaMalloc(bsum)");

    const int64_t rows = (int64_t)p.n_tiles * p.k_stages * p.ntaps * p.gps * p.block_n_tot;
    pack_filters_kernel<<<grid_for(rows), 256>>>(filters, g, p.block_n, p.block_n_tot, p.n_tiles, p.gps,
                                                 p.k_stages, (checks & ABED_CHECK_FC) ? 1 : 0, pl->d_wpk);
    cuda_check(cudaGetLastError(), "pack_filters");
    dev_colsum_i8(filters, shape.k, crs, pl->d_fsum, nullptr);  // gen_filter_checksum (offline)
    if (checks & ABED_CHECK_FIC) {
      const int64_t nw = (int64_t)g.n_phase * g.c16 * 16 * g.Hl * g.Wl;
      cuda_check(cudaMalloc(&pl->d_ficw, nw * 4), "cudaMalloc(ficw)");
      fic_weight_kernel<<<grid_for(nw), 256>>>(pl->d_fsum, g, pl->d_ficw);
      cuda_check(cudaMalloc(&pl->d_ficw8, nw * 3), "cudaMalloc(ficw8)");
      int* d_big = nullptr;
      cuda_check(cudaMalloc(&d_big, 4), "cudaMalloc(flag)");
      cuda_check(cudaMemset(d_big, 0, 4), "memset flag");
      fic_weight_digits_kernel<<<grid_for(nw), 256>>>(pl->d_ficw, nw / 16, pl->d_ficw8, d_big);
      int big = 0;
      cuda_check(cudaMemcpy(&big, d_big, 4, cudaMemcpyDeviceToHost), "flag d2h");
      cudaFree(d_big);
      pl->ficw8_ok = (big & 1) ? 0 : 1;
      pl->ficw8_ndig = (big & 2) ? 3 : 2;  // every |G| within two balanced digits: 8 dp4a per chunk
      cuda_check(cudaGetLastError(), "fic_weight");
      if (pl->ficw8_ok && !pl->h_rep.empty()) build_fic_classes(pl);
    }
    if (checks & ABED_CHECK_IC) build_ic_classes(pl);
    cuda_check(cudaDeviceSynchronize(), "plan_create sync");
  } catch (...) {
    abed_conv_plan_destroy(pl);
    throw;
  }
  return pl;
}

void plan_run(abed_conv_plan* pl, const int8_t* packed, const abed_epilog_params* ep, int out_mode, void* out,
              const abed_conv_plan* next, int64_t fault_key, int fault_bit, cudaStream_t st) {
  if (pl->dw) {
    plan_run_dw(pl, packed, ep, out_mode, out, next, fault_key, fault_bit, st);
    return;
  }
  ConvTcParams p = pl->base;
  p.act = packed;
  p.wpk = pl->d_wpk;
  p.out_mode = out_mode;
  p.out = out;
  p.check = pl->checks;
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
  const bool fmode = pl->dtype != abed_dev::DT_I8;
  const bool h_out = out_mode == ABED_OUT_H_PACKED || out_mode == ABED_OUT_H_COMPARE;
  const bool i_out = out_mode == ABED_OUT_I32_NCHW || out_mode == ABED_OUT_I8_NCHW || out_mode == ABED_OUT_I8_PACKED ||
                     out_mode == ABED_OUT_I8_COMPARE;
  if ((fmode && i_out) || (!fmode && h_out))
    throw_invalid("conv plan: output mode does not match the plan's operand type");
  p.dtype = pl->dtype;
  p.tau_fc = pl->tau_fc;
  p.tau_fic = pl->tau_fic;
  p.facc = pl->d_facc;
  p.rhs_ext_f = pl->d_rhs_f;
  p.ficwf = pl->d_ficwf;
  if (out_mode == ABED_OUT_I8_PACKED || out_mode == ABED_OUT_I8_COMPARE || out_mode == ABED_OUT_H_PACKED ||
      out_mode == ABED_OUT_H_COMPARE) {
    if (next) {
      const ActGeom& o = next->g;
      if (o.c != pl->g.k || o.h != pl->g.p || o.w != pl->g.q || o.n != pl->g.n || o.cpg != pl->g.cpg)
        throw_invalid("conv plan: next layer input does not match this layer's output");
      p.o_plane_len = o.plane_len; p.o_Hl = o.Hl; p.o_Wl = o.Wl; p.o_ph = o.ph; p.o_pw = o.pw;
      p.o_sh = o.sh; p.o_sw = o.sw; p.o_nph_w = o.nph_w; p.o_c16 = o.c16;
      if (out_mode == ABED_OUT_I8_PACKED && next->af_input && (next->checks & ABED_CHECK_FIC)) {
        // FIC-AF: accumulate the consumer's rhs from the values this epilogue stores
        p.af_ficw8 = next->d_ficw8;
        p.af_acc = next->d_af_acc;
        p.af_HlWl = (int64_t)o.Hl * o.Wl;
      }
    } else {
      // identity consumer geometry: 1x1, stride 1, pad 0
      abed_layer_shape s1{pl->shape.n, pl->shape.k, pl->shape.p, pl->shape.q, 1, 1, 1, 1, 1, 0, 0, pl->shape.p, pl->shape.q};
      const ActGeom o = make_geom(s1, pl->g.cpg);
      p.o_plane_len = o.plane_len; p.o_Hl = o.Hl; p.o_Wl = o.Wl; p.o_ph = 0; p.o_pw = 0;
      p.o_sh = 1; p.o_sw = 1; p.o_nph_w = 1; p.o_c16 = o.c16;
    }
  }
  p.fc_part = pl->d_fc_part;
  p.tile_sem = pl->d_tile_sem;
  p.cta_rec = pl->d_cta_rec;
  p.kacc = pl->d_kacc;
  p.outcome = pl->d_outcome;
  p.rhs_ext = pl->d_acc;
  p.ficw8 = pl->d_ficw8;
  p.ic_sum = pl->d_acc + 4;
  p.cmp_count = pl->d_acc + 1;
  p.fault_key = fault_key;
  p.fault_bit = fault_bit;
  // IC: the per-channel sums (and class sums) of a run are zeroed by its verdict;
  // a run whose predecessor was never finalized clears them here.  Under stream
  // capture the host cannot see how replays interleave with finalizes, so captured
  // runs clear them too -- unless the caller declared that its graphs pair every
  // run with a finalize (abed_conv_plan_set_paired_finalize)
  cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
  cuda_check(cudaStreamIsCapturing(st, &cap), "capture status");
  const bool ic_dirty = (pl->checks & ABED_CHECK_IC) &&
                        (pl->ic_pending || (cap != cudaStreamCaptureStatusNone && !pl->paired_finalize));
  if (ic_dirty) cuda_check(cudaMemsetAsync(pl->d_acc + 4, 0, pl->shape.k * 8, st), "memset ic");
  if (pl->checks & ABED_CHECK_IC) pl->ic_pending = 1;
  // ICBatch: the same for the batch sums and the digit-writer counter, which the
  // scan at finalize consumes and resets
  const bool icb_dirty = (pl->checks & ABED_CHECK_ICBATCH) &&
                         (pl->icb_pending || (cap != cudaStreamCaptureStatusNone && !pl->paired_finalize));
  if (icb_dirty) {
    cuda_check(cudaMemsetAsync(pl->d_icb_lhs, 0, (size_t)pl->shape.k * pl->shape.p * pl->shape.q * 8, st),
               "memset icb_lhs");
    cuda_check(cudaMemsetAsync(pl->d_icb_ctl, 0, 8, st), "memset icb_ctl");
  }
  if (pl->checks & ABED_CHECK_ICBATCH) pl->icb_pending = 1;
  // compare runs accumulate mismatches; compare_count reports the increase
  p.rhs_mode = 0;
  p.conv_grid = conv_tc_grid(p, num_sms());
  p.ic_ctas = 0;
  // FR input checksum: a conv grid that leaves SMs idle gets extra CTAs there
  // that do the whole checksum with all their warps; otherwise the conv CTAs'
  // input-checksum warps do it.  Returns the image split of the work items.
  auto fr_split = [&](const ActGeom& g) {
    if (p.n_tiles == 1 && p.conv_grid > 0) {
      // wave-quantisation slack: the fewest conv CTAs with the same units per CTA
      // (same makespan) leave SMs free for the input-checksum CTAs -- used when
      // it frees enough of them to carry the whole checksum (measured: 12 idle
      // SMs are too few for ResNet-50 layer1, 42 beat the in-CTA warps on layer2)
      const int per = (p.m_tiles + p.conv_grid - 1) / p.conv_grid;
      const int g2 = (p.m_tiles + per - 1) / per;
      if (num_sms() - g2 >= 24) p.conv_grid = g2;
    }
    const int idle = num_sms() - p.conv_grid;
    int64_t want;
    if (idle >= 16) {
      p.ic_ctas = idle;
      want = 2LL * idle * abed_dev::kConvThreads_host;
    } else {
      want = 2LL * p.conv_grid * 64;
    }
    const int64_t cells = (int64_t)g.n_phase * g.c16 * g.Hl * g.Wl;
    // ResNet-50 b32: the 256->64/128 1x1 layers at 56x56 (26 MB inputs) gain ~2 us
    // with 16 loads in flight; the <= 7 MB inputs lose ~0.4 us (tools/r50net_layer_times.py)
    p.rhs_deep = geom_packed_bytes(g) >= (int64_t(16) << 20) ? 1 : 0;
    p.g_ndig = pl->ficw8_ndig;
    return (int)std::max<int64_t>(1, std::min<int64_t>(g.n, (want + cells - 1) / cells));
  };
  if (!fmode && pl->af_input && (pl->checks & ABED_CHECK_FIC) && !pl->reuse_input_checksum) {
    p.rhs_mode = 2;  // FIC-AF: the producer's epilogue supplies the rhs
  } else if (fmode && (pl->checks & ABED_CHECK_FIC) && !pl->reuse_input_checksum) {
    // float mode: the input-checksum warps compute rhs = sum x * G in-kernel
    p.rhs_mode = 1;
    p.rhs_nsplit = fr_split(pl->g);
  } else if (!fmode && (pl->checks & (ABED_CHECK_FIC | ABED_CHECK_IC)) && !pl->reuse_input_checksum) {
    // input checksum of the pristine input (FR option)
    const ActGeom& g = pl->g;
    if (pl->checks & ABED_CHECK_IC) {
      // IC (and FIC's rhs, derived from ic at the verdict): the input checksum's
      // class sums accumulated in-kernel by the input-checksum warps / CTAs
      if (ic_dirty) cuda_check(cudaMemsetAsync(pl->d_ic_S, 0, pl->ic_S_bytes, st), "memset ic_S");
      p.rhs_mode = 4;
      p.ic_S = pl->d_ic_S;
      p.ic_rowcls = pl->d_ic_cls;
      p.ic_colcls = pl->d_ic_cls + (size_t)g.nph_h * g.Hl;
      p.ic_nrc = pl->ic_nrc;
      p.ic_ncc = pl->ic_ncc;
      p.rhs_nsplit = fr_split(g);
    } else {
      const int64_t cells = (int64_t)g.n_phase * g.c16 * g.Hl * g.Wl;
      if (pl->ficw8_ok && pl->d_ficc8 && pl->rhs_src == ABED_RHS_STAGED && g.n_phase <= 4) {
        // FIC only: rhs = sum x * G computed by the conv kernel's input-checksum
        // warps from the activation tiles already staged for the MMAs
        p.rhs_mode = 3;
        p.ficc8 = pl->d_ficc8;
        p.rowcls = pl->d_rowcls;
        p.colcls = pl->d_colcls;
        p.nrc = pl->nrc;
        p.ncc = pl->ncc;
      } else if (pl->ficw8_ok) {
        // FIC only: rhs = sum x * G computed by the conv kernel's input-checksum
        // warps from their own read of the stored input
        p.rhs_mode = 1;
        p.rhs_nsplit = fr_split(g);
      } else {
        // |G| too large for the 3-digit map: one separate pass ahead of the conv
        cuda_check(cudaMemsetAsync(pl->d_acc, 0, 8, st), "memset rhs");
        const int nsplit = g.n >= 8 ? 8 : g.n;
        fic_rhs_kernel<<<grid_for(cells * nsplit), 256, 0, st>>>(packed, g, pl->d_ficw, nsplit, pl->d_acc);
        cuda_check(cudaGetLastError(), "fic_rhs");
      }
    }
  }
  if (pl->checks & ABED_CHECK_ICBATCH) {
    p.icb_d = pl->g.n_extra;
    p.icb_lhs = pl->d_icb_lhs;
    p.icb_dig = pl->d_icb_dig;
    p.icb_ready = pl->d_icb_ctl;
    // SMs the conv grid leaves idle help write the digit images
    if (p.ic_ctas == 0 && num_sms() - p.conv_grid >= 16) p.ic_ctas = num_sms() - p.conv_grid;
    p.icb_writers = (unsigned)(2 * p.conv_grid + (abed_dev::kConvThreads_host / 32) * p.ic_ctas);
  }
  pl->last_rhs_mode = p.rhs_mode;
  pl->last_grid = p.conv_grid + p.ic_ctas;
  cuda_check(conv_tc_launch(p, num_sms(), pl->pdl != 0, st), "conv_i8_tc launch");
}

// ICBatch scan of the plan's last run (ic_batch_verify, checksum.hpp:398-421) --
// launched by the finalize that first follows the run, batched over the pass
static abed_dev::IcbScanJob icb_scan_job(abed_conv_plan* pl) {
  abed_dev::IcbScanJob j{};
  j.lhs = pl->d_icb_lhs;
  j.dig = pl->d_icb_dig;
  j.D = pl->g.n_extra;
  j.Q = (int)pl->g.q;
  j.PQ = (int64_t)pl->g.p * pl->g.q;
  j.kpq = (int64_t)pl->shape.k * j.PQ;
  j.rec = pl->d_icb_rec;
  j.ctl = pl->d_icb_ctl;
  j.out = pl->d_icb_out;
  pl->icb_pending = 0;
  return j;
}

abed_dev::VerdictJob plan_verdict_job(const abed_conv_plan* pl, abed_verify_outcome* out_dev) {
  abed_dev::VerdictJob j{};
  j.rec = pl->d_cta_rec;
  j.grid = pl->dw ? dw_grid() : pl->last_grid;
  j.P = pl->g.p;
  j.Q = pl->g.q;
  j.dtype = pl->dtype;
  j.checks = pl->checks & (ABED_CHECK_FC | ABED_CHECK_FIC);
  j.icb = pl->d_icb_out;  // ICBatch verdict of the last run -> slot 2 (nullptr: not an ICBatch plan)
  j.rhs_mode = pl->last_rhs_mode;
  j.rhs_ext = pl->d_acc;
  j.af_acc = pl->d_af_acc;
  j.rhs_ext_f = pl->d_rhs_f;
  j.tau_fic = pl->tau_fic;
  j.out = out_dev;
  j.fc_part = pl->d_fc_part;
  j.tile_flag = pl->d_tile_sem;
  // int8 plans with several N tiles: the verdict rechecks flagged M tiles; float
  // plans keep the full-channel FC check in-kernel
  j.n_tiles = (pl->dw || pl->dtype != abed_dev::DT_I8) ? 1 : pl->base.n_tiles;
  j.m_tiles = pl->g.m_tiles;
  j.Hl = pl->g.Hl;
  j.Wl = pl->g.Wl;
  j.m_total = (int64_t)pl->g.n * pl->g.Hl * pl->g.Wl;  // real images only
  j.tau_fc = pl->tau_fc;
  return j;
}

void plan_finalize(abed_conv_plan* pl, abed_verify_outcome* out_dev, cudaStream_t st) {
  // IC first: with FIC its input checksum also gives FIC's rhs
  if (pl->checks & ABED_CHECK_IC) ic_verdict(pl, out_dev + 2, st);
  if ((pl->checks & ABED_CHECK_ICBATCH) && pl->icb_pending) {
    const abed_dev::IcbScanJob j = icb_scan_job(pl);
    cuda_check(icb_scan_launch(&j, 1, st), "icb_scan");
  }
  // FC / FIC: reduce the conv kernel's per-CTA records into VerifyOutcomes
  if (pl->checks & (ABED_CHECK_FC | ABED_CHECK_FIC | ABED_CHECK_ICBATCH)) {
    const abed_dev::VerdictJob j = plan_verdict_job(pl, out_dev);
    cuda_check(verdict_launch(&j, 1, st), "verdict");
  }
  cuda_check(cudaGetLastError(), "finalize");
}

}  // namespace abed_host

extern "C" {

const char* abed_last_error(void) { return g_last_error.c_str(); }
int abed_version(void) { return 1; }
int abed_device_check(void) {
  return guarded([] { require_device(); });
}
int abed_malloc(void** dptr, size_t bytes) {
  return guarded([&] { require_device(); cuda_check(cudaMalloc(dptr, bytes ? bytes : 16), "cudaMalloc"); });
}
int abed_free(void* dptr) {
  return guarded([&] { cuda_check(cudaFree(dptr), "cudaFree"); });
}
int abed_memcpy_h2d(void* dst, const void* src, size_t bytes) {
  return guarded([&] { cuda_check(cudaMemcpy(dst, src, bytes, cudaMemcpyHostToDevice), "h2d"); });
}
int abed_memcpy_d2h(void* dst, const void* src, size_t bytes) {
  return guarded([&] { cuda_check(cudaMemcpy(dst, src, bytes, cudaMemcpyDeviceToHost), "d2h"); });
}
int abed_memset(void* dptr, int value, size_t bytes) {
  return guarded([&] { cuda_check(cudaMemset(dptr, value, bytes), "memset"); });
}
int abed_synchronize(void) {
  return guarded([] { cuda_check(cudaDeviceSynchronize(), "synchronize"); });
}

int abed_layer_shape_make(int64_t n, int64_t c, int64_t h, int64_t w, int64_t k, int64_t r, int64_t s,
                          int64_t stride_h, int64_t stride_w, int64_t pad_h, int64_t pad_w,
                          abed_layer_shape* out) {
  return guarded([&] {
    // tensor.hpp:178-193
    if (n < 1 || c < 1 || h < 1 || w < 1 || k < 1 || r < 1 || s < 1) throw_invalid("LayerShape: extents must be >= 1");
    if (stride_h < 1 || stride_w < 1) throw_invalid("LayerShape: strides must be >= 1");
    if (pad_h < 0 || pad_w < 0) throw_invalid("LayerShape: pads must be >= 0");
    if (r > h + 2 * pad_h || s > w + 2 * pad_w) throw_invalid("LayerShape: filter exceeds padded input");
    *out = abed_layer_shape{n, c, h, w, k, r, s, stride_h, stride_w, pad_h, pad_w,
                            (h + 2 * pad_h - r) / stride_h + 1, (w + 2 * pad_w - s) / stride_w + 1};
  });
}

// ---------------------------------------------------------------- plan API
int abed_conv_plan_create(const abed_layer_shape* shape, const int8_t* filters, int32_t checks,
                          int32_t force_block_n, abed_conv_plan** plan) {
  return guarded([&] { *plan = plan_create(*shape, filters, checks, force_block_n); });
}
int abed_conv_plan_destroy(abed_conv_plan* pl) {
  if (!pl) return ABED_OK;
  cudaFree(pl->d_wpk); cudaFree(pl->d_filters); cudaFree(pl->d_fsum); cudaFree(pl->d_ic);
  cudaFree(pl->d_bsum); cudaFree(pl->d_ficw); cudaFree(pl->d_ficw8); cudaFree(pl->d_fc_part); cudaFree(pl->d_tile_sem);
  cudaFree(pl->d_cta_rec); cudaFree(pl->d_kacc); cudaFree(pl->d_outcome);
  cudaFree(pl->d_facc); cudaFree(pl->d_rhs_f); cudaFree(pl->d_ficwf); cudaFree(pl->d_fsum_f); cudaFree(pl->d_dwf);
  cudaFree(pl->d_af_acc); cudaFree(pl->d_ficc8);  // row / column classes live inside it
  cudaFree(pl->d_acc); cudaFree(pl->d_zero_bias);
  cudaFree(pl->d_icb_lhs); cudaFree(pl->d_icb_dig); cudaFree(pl->d_icb_ctl); cudaFree(pl->d_icb_rec);
  cudaFree(pl->d_icb_out); cudaFree(pl->d_ic_scr); cudaFree(pl->d_ic_last); cudaFree(pl->d_ic_S); cudaFree(pl->d_ic_cls); cudaFree(pl->d_ic_mask);
  delete pl;
  return ABED_OK;
}
int abed_conv_plan_info(const abed_conv_plan* pl, abed_plan_info* info) {
  return guarded([&] {
    info->packed_input_bytes = geom_packed_bytes(pl->g);
    info->block_n = pl->base.block_n;
    info->n_tiles = pl->base.n_tiles;
    info->m_tiles = pl->base.m_tiles;
    info->gps = pl->base.gps;
    info->b_resident = pl->base.b_resident;
    info->n_phase = pl->g.n_phase;
    info->Hl = pl->g.Hl;
    info->Wl = pl->g.Wl;
    info->smem_bytes = conv_tc_smem_bytes(pl->base);
  });
}
int abed_pack_input(const abed_conv_plan* pl, const int8_t* input, int8_t* packed, void* stream) {
  return guarded([&] {
    launch_pack_input(input, pl->g, packed, (cudaStream_t)stream);
    cuda_check(cudaGetLastError(), "pack_input");
  });
}
int abed_conv_plan_run(abed_conv_plan* pl, const int8_t* packed, const abed_epilog_params* params, int32_t out_mode,
                       void* out, const abed_conv_plan* next, int64_t fault_key, int32_t fault_bit, void* stream) {
  return guarded([&] { plan_run(pl, packed, params, out_mode, out, next, fault_key, fault_bit, (cudaStream_t)stream); });
}
int abed_conv_plan_finalize(abed_conv_plan* pl, abed_verify_outcome* outcome_dev, void* stream) {
  return guarded([&] { plan_finalize(pl, outcome_dev, (cudaStream_t)stream); });
}
int abed_conv_plan_set_af_input(abed_conv_plan* pl, int32_t on) {
  return guarded([&] {
    if (on) {
      if (!(pl->checks & ABED_CHECK_FIC) || pl->dtype != abed_dev::DT_I8)
        throw_invalid("FIC-AF: the consumer must be an int8 plan with the FIC check");
      if (!pl->ficw8_ok) throw_invalid("FIC-AF: the position-weight map exceeds the 3-digit range");
    }
    pl->af_input = on ? 1 : 0;
  });
}
int abed_conv_plan_finalize_many(abed_conv_plan* const* plans, int32_t n, abed_verify_outcome* outcomes_dev,
                                 void* stream) {
  return guarded([&] {
    if (n < 0) throw_invalid("finalize_many: negative plan count");
    std::vector<abed_dev::VerdictJob> jobs;
    std::vector<IcVerdictJob> ic_jobs;
    std::vector<abed_dev::IcbScanJob> icb_jobs;
    for (int i = 0; i < n; ++i) {
      abed_conv_plan* pl = plans[i];
      if ((pl->checks & ABED_CHECK_ICBATCH) && pl->icb_pending) icb_jobs.push_back(icb_scan_job(pl));
      if (pl->checks & (ABED_CHECK_FC | ABED_CHECK_FIC | ABED_CHECK_ICBATCH))
        jobs.push_back(plan_verdict_job(pl, outcomes_dev + 3 * i));
      if (pl->checks & ABED_CHECK_IC) ic_jobs.push_back(ic_verdict_job(pl, outcomes_dev + 3 * i + 2, (cudaStream_t)stream));
    }
    // IC first (with FIC its input checksum also gives FIC's rhs): two launches for all plans
    if (!ic_jobs.empty()) ic_verdict_many_launch(ic_jobs.data(), (int)ic_jobs.size(), (cudaStream_t)stream);
    // ICBatch: one scan launch for every plan of the pass (its outcome goes to slot 2 in the verdict)
    if (!icb_jobs.empty())
      cuda_check(icb_scan_launch(icb_jobs.data(), (int)icb_jobs.size(), (cudaStream_t)stream), "icb_scan");
    if (!jobs.empty()) cuda_check(verdict_launch(jobs.data(), (int)jobs.size(), (cudaStream_t)stream), "verdict");
  });
}
int abed_conv_plan_set_input_checksum_source(abed_conv_plan* pl, int32_t source) {
  return guarded([&] {
    if (!pl) throw_invalid("plan is null");
    if (source != ABED_RHS_STAGED && source != ABED_RHS_REREAD) throw_invalid("input checksum source must be 0 or 1");
    pl->rhs_src = source;
  });
}
int abed_conv_plan_set_paired_finalize(abed_conv_plan* pl, int32_t paired) {
  return guarded([&] {
    if (!pl) throw_invalid("plan is null");
    pl->paired_finalize = paired ? 1 : 0;
  });
}
int abed_conv_plan_set_reuse_input_checksum(abed_conv_plan* pl, int32_t reuse) {
  return guarded([&] { pl->reuse_input_checksum = reuse ? 1 : 0; });
}
int abed_conv_plan_compare_count(abed_conv_plan* pl, int64_t* count) {
  return guarded([&] {
    unsigned long long c = 0;
    cuda_check(cudaMemcpy(&c, pl->d_acc + 1, 8, cudaMemcpyDeviceToHost), "cmp count");
    *count = (int64_t)(c - pl->cmp_seen);  // the counter only grows: no memset per run
    pl->cmp_seen = c;
  });
}

// ---------------------------------------------------------------- conv_direct
int abed_conv_i8(const int8_t* input, const int8_t* filters, const abed_layer_shape* shape, int32_t* convout,
                 void* stream) {
  return guarded([&] {
    validate_shape(*shape);
    if (shape->c * shape->r * shape->s > 65536)
      throw_invalid("conv_direct: CRS > 65536 exceeds the int32 accumulator plan");
    cudaStream_t st = (cudaStream_t)stream;
    one_shot_run(*shape, 0, input, filters, nullptr, ABED_OUT_I32_NCHW, convout, nullptr, st);
    cuda_check(cudaStreamSynchronize(st), "conv_i8 sync");
  });
}

// ---------------------------------------------------------------- diagnostics
// Per-CTA clock timeline of the conv kernel (conv_tc.cuh kTraceSlots int64 per
// CTA, zeroed by the caller); nullptr switches it off.  Not on any reference path.
int abed_debug_set_conv_trace(abed_conv_plan* pl, int64_t* trace_dev, int32_t flags) {
  return guarded([&] {
    pl->base.trace = trace_dev;
    pl->base.dbg = flags;
  });
}

}  // extern "C"
