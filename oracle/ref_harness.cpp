// ref_harness.cpp -- TEST INFRASTRUCTURE ONLY.
//
// extern "C" shims over the UNMODIFIED reference implementation, compiled from
// the reference headers where they lie (-I /root/reference/proj/include) by
// oracle/Makefile into oracle/_ref/libabed_ref.so.  Used to (1) pin the C oracle
// (abed_oracle.c) against the reference itself, (2) generate tests/golden/, and
// (3) time the reference's own CPU path for bench.py (cpu_baseline / --impl
// reference).  No reference source is copied into this repository.
#include <abed/abft_gemm.hpp>
#include <abed/checksum.hpp>
#include <abed/convolution.hpp>
#include <abed/faults.hpp>
#include <abed/rng.hpp>
#include <abed/tensor.hpp>

#include <chrono>
#include <cstring>
#include <stdexcept>
#include <thread>
#include <vector>

#include "../include/abed_b200.h"

using namespace abed;

namespace {

LayerShape to_ls(const abed_layer_shape* s) {
  return LayerShape::make(s->n, s->c, s->h, s->w, s->k, s->r, s->s, s->stride_h, s->stride_w, s->pad_h, s->pad_w);
}
Tensor4D make(Dims4 d, ElemKind k, const void* src) {
  Tensor4D t(d, k);
  std::memcpy(t.raw(), src, t.byte_size());
  return t;
}
void put(const Tensor4D& t, void* dst) { std::memcpy(dst, t.raw(), t.byte_size()); }
void put_outcome(const VerifyOutcome& v, abed_verify_outcome* o) {
  std::memset(o, 0, sizeof(*o));
  o->status = v.pass() ? 0 : 1;
  o->has_locus = v.locus.has_value() ? 1 : 0;
  if (v.locus) {
    o->locus[0] = (*v.locus)[0];
    o->locus[1] = (*v.locus)[1];
    o->locus[2] = (*v.locus)[2];
  }
  o->lhs = v.lhs;
  o->rhs = v.rhs;
  o->lhs_f = v.lhs_f;
  o->rhs_f = v.rhs_f;
}
template <typename Fn>
int guard(Fn&& fn) {
  try {
    fn();
    return ABED_OK;
  } catch (const std::invalid_argument&) {
    return ABED_ERR_INVALID_ARGUMENT;
  } catch (const std::out_of_range&) {
    return ABED_ERR_OUT_OF_RANGE;
  } catch (...) {
    return ABED_ERR_RUNTIME;
  }
}
Dims4 dd(abed_dims4 d) { return {d.d0, d.d1, d.d2, d.d3}; }
EpilogParams ep(float scale, const float* bias, int64_t n, int act, int kind) {
  EpilogParams p;
  p.scale = scale;
  if (bias) p.bias.assign(bias, bias + n);
  p.activation = act == ABED_RELU ? Activation::ReLU : Activation::Identity;
  p.output_kind = static_cast<ElemKind>(kind);
  return p;
}

}  // namespace

extern "C" {

uint64_t ref_derive_seed(uint64_t root, uint64_t index) { return derive_seed(root, index); }
void ref_fill_random_i8(int8_t* t, int64_t n, uint64_t seed) {
  Tensor4D x({1, 1, 1, n}, ElemKind::I8);
  SplitMix64 g(seed);
  fill_random_i8(x, g);
  put(x, t);
}
void ref_fill_random_f32(float* t, int64_t n, uint64_t seed, float lo, float hi) {
  Tensor4D x({1, 1, 1, n}, ElemKind::F32);
  SplitMix64 g(seed);
  fill_random_f32(x, g, lo, hi);
  put(x, t);
}
uint64_t ref_below(uint64_t seed, uint64_t bound) {
  SplitMix64 g(seed);
  return g.below(bound);
}
int ref_layer_shape_make(int64_t n, int64_t c, int64_t h, int64_t w, int64_t k, int64_t r, int64_t s, int64_t sh,
                         int64_t sw, int64_t ph, int64_t pw, abed_layer_shape* o) {
  return guard([&] {
    const LayerShape ls = LayerShape::make(n, c, h, w, k, r, s, sh, sw, ph, pw);
    *o = abed_layer_shape{ls.n, ls.c, ls.h, ls.w, ls.k, ls.r, ls.s, ls.stride_h, ls.stride_w, ls.pad_h, ls.pad_w, ls.p, ls.q};
  });
}
int ref_conv_fast_i8(const int8_t* x, const int8_t* f, const abed_layer_shape* s, int32_t* out) {
  return guard([&] {
    const LayerShape ls = to_ls(s);
    put(detail::conv_fast_i8(make(ls.input_dims(), ElemKind::I8, x), make(ls.filter_dims(), ElemKind::I8, f), ls), out);
  });
}
int ref_conv_direct(const int8_t* x, const int8_t* f, const abed_layer_shape* s, int32_t* out) {
  return guard([&] {
    const LayerShape ls = to_ls(s);
    put(conv_direct(make(ls.input_dims(), ElemKind::I8, x), make(ls.filter_dims(), ElemKind::I8, f), ls), out);
  });
}
int ref_conv_direct_f32(const float* x, const float* f, const abed_layer_shape* s, float* out) {
  return guard([&] {
    const LayerShape ls = to_ls(s);
    put(conv_direct_f32(make(ls.input_dims(), ElemKind::F32, x), make(ls.filter_dims(), ElemKind::F32, f), ls), out);
  });
}
int ref_epilog(const int32_t* in, abed_dims4 d, float scale, const float* bias, int64_t nb, int act, int kind, void* out) {
  return guard([&] { put(epilog(make(dd(d), ElemKind::I32, in), ep(scale, bias, nb, act, kind)), out); });
}
int ref_gen_filter_checksum(const int8_t* f, abed_dims4 fd, int32_t* sums) {
  return guard([&] { put(gen_filter_checksum(make(dd(fd), ElemKind::I8, f)).sums, sums); });
}
int ref_decompose_checksum_filters(const int32_t* sums, int64_t n, int8_t* planes) {
  return guard([&] {
    FilterChecksum fc;
    fc.sums = make({1, 1, 1, n}, ElemKind::I32, sums);
    const auto p = decompose_checksum_filters(fc);
    for (int i = 0; i < 4; ++i) put(p[i], planes + i * n);
  });
}
int ref_conv_checksum_planes(const int8_t* x, const abed_layer_shape* s, const int8_t* planes, int32_t* extra) {
  return guard([&] {
    const LayerShape ls = to_ls(s);
    const int64_t crs = ls.crs();
    std::array<Tensor4D, 4> p{make({1, ls.c, ls.r, ls.s}, ElemKind::I8, planes),
                              make({1, ls.c, ls.r, ls.s}, ElemKind::I8, planes + crs),
                              make({1, ls.c, ls.r, ls.s}, ElemKind::I8, planes + 2 * crs),
                              make({1, ls.c, ls.r, ls.s}, ElemKind::I8, planes + 3 * crs)};
    const auto e = conv_checksum_planes(make(ls.input_dims(), ElemKind::I8, x), ls, p);
    for (int i = 0; i < 4; ++i) put(e[i], extra + i * ls.npq());
  });
}
int ref_recombine_extra_fmaps(const int32_t* e, int64_t n, int64_t* out) {
  return guard([&] {
    std::array<Tensor4D, 4> t{make({1, 1, 1, n}, ElemKind::I32, e), make({1, 1, 1, n}, ElemKind::I32, e + n),
                              make({1, 1, 1, n}, ElemKind::I32, e + 2 * n), make({1, 1, 1, n}, ElemKind::I32, e + 3 * n)};
    put(recombine_extra_fmaps(t), out);
  });
}
int ref_fc_verify(const int32_t* cv, abed_dims4 d, const int64_t* ev, int64_t original_k, abed_verify_outcome* o) {
  return guard([&] {
    put_outcome(fc_verify(make(dd(d), ElemKind::I32, cv), make({d.d0, 1, d.d2, d.d3}, ElemKind::I64, ev), original_k), o);
  });
}
int ref_gen_input_checksum(const int8_t* x, const abed_layer_shape* s, int32_t* sums) {
  return guard([&] {
    const LayerShape ls = to_ls(s);
    put(gen_input_checksum(make(ls.input_dims(), ElemKind::I8, x), ls).sums, sums);
  });
}
int ref_fic_dot(const int32_t* a, const int32_t* b, int64_t n, int64_t* out) {
  return guard([&] {
    FilterChecksum fc;
    InputChecksum ic;
    fc.sums = make({1, 1, 1, n}, ElemKind::I32, a);
    ic.sums = make({1, 1, 1, n}, ElemKind::I32, b);
    *out = fic_dot(fc, ic);
  });
}
int ref_fic_verify(const int32_t* c, int64_t n, int64_t expected, int forced32, abed_verify_outcome* o) {
  return guard([&] {
    const Tensor4D t = make({1, 1, 1, n}, ElemKind::I32, c);
    put_outcome(forced32 ? fic_verify_forced32(t, expected) : fic_verify(t, expected), o);
  });
}
int ref_ic_verify_k(const int32_t* cv, abed_dims4 d, const int8_t* f, abed_dims4 fd, const int32_t* ic,
                    abed_verify_outcome* o) {
  return guard([&] {
    InputChecksum icc;
    icc.sums = make({1, fd.d1, fd.d2, fd.d3}, ElemKind::I32, ic);
    put_outcome(ic_verify_k(make(dd(d), ElemKind::I32, cv), make(dd(fd), ElemKind::I8, f), icc), o);
  });
}
int ref_ic_batch_checksum(const int8_t* x, abed_dims4 d, int32_t* out) {
  return guard([&] { put(ic_batch_checksum(make(dd(d), ElemKind::I8, x)), out); });
}
int ref_conv_batch_checksum(const int32_t* b, const int8_t* f, const abed_layer_shape* s, int64_t* out) {
  return guard([&] {
    const LayerShape ls = to_ls(s);
    put(conv_batch_checksum(make({1, ls.c, ls.h, ls.w}, ElemKind::I32, b), make(ls.filter_dims(), ElemKind::I8, f), ls), out);
  });
}
int ref_ic_batch_verify(const int32_t* cv, abed_dims4 d, const int64_t* ev, abed_verify_outcome* o) {
  return guard([&] {
    put_outcome(ic_batch_verify(make(dd(d), ElemKind::I32, cv), make({1, d.d1, d.d2, d.d3}, ElemKind::I64, ev)), o);
  });
}
int ref_plan_precision(const abed_layer_shape* s, int bits, abed_precision_plan* p) {
  return guard([&] {
    const PrecisionPlan pl = plan_precision(to_ls(s), bits);
    p->operand_bits = pl.operand_bits;
    p->bits_output_fmap = pl.bits_output_fmap;
    p->bits_reduced_fc = pl.bits_reduced_fc;
    p->bits_reduced_fic = pl.bits_reduced_fic;
    p->bits_filter_checksum = pl.bits_filter_checksum;
    p->bits_input_checksum = pl.bits_input_checksum;
    p->output_fmap_kind = (int)pl.output_fmap_kind;
    p->reduced_fc_kind = (int)pl.reduced_fc_kind;
    p->reduced_fic_kind = (int)pl.reduced_fic_kind;
    p->filter_checksum_kind = (int)pl.filter_checksum_kind;
    p->input_checksum_kind = (int)pl.input_checksum_kind;
  });
}
int ref_float_mode(const float* x, const float* f, const abed_layer_shape* s, double tau, float* convout,
                   double* out6 /* fic lhs, fic rhs, fc status, ic status, fic status, unused */) {
  return guard([&] {
    const LayerShape ls = to_ls(s);
    const Tensor4D in = make(ls.input_dims(), ElemKind::F32, x), ft = make(ls.filter_dims(), ElemKind::F32, f);
    const Tensor4D conv = conv_direct_f32(in, ft, ls);
    put(conv, convout);
    const auto fs = filter_checksum_f64(ft);
    const auto is = input_checksum_f64(in, ls);
    out6[0] = reduce_all_f64(conv);
    out6[1] = fic_dot_f64(fs, is);
    Tensor4D cs({1, ls.c, ls.r, ls.s}, ElemKind::F32);
    for (std::size_t i = 0; i < fs.size(); ++i) cs.view<float>()[i] = static_cast<float>(fs[i]);
    LayerShape one = ls;
    one.k = 1;
    out6[2] = fc_verify_f32(conv, conv_direct_f32(in, cs, one), tau).pass() ? 0 : 1;
    out6[3] = ic_verify_k_f32(conv, ft, is, tau).pass() ? 0 : 1;
    out6[4] = fic_verify_f32(conv, out6[1], tau).pass() ? 0 : 1;
  });
}
int ref_filter_checksum_f64(const float* f, abed_dims4 fd, double* sums) {
  return guard([&] {
    const auto v = filter_checksum_f64(make(dd(fd), ElemKind::F32, f));
    std::memcpy(sums, v.data(), v.size() * 8);
  });
}
int ref_input_checksum_f64(const float* x, const abed_layer_shape* s, double* sums) {
  return guard([&] {
    const LayerShape ls = to_ls(s);
    const auto v = input_checksum_f64(make(ls.input_dims(), ElemKind::F32, x), ls);
    std::memcpy(sums, v.data(), v.size() * 8);
  });
}
int ref_fused_conv_epilog(const int8_t* x, const int8_t* f, const abed_layer_shape* s, float scale, const float* bias,
                          int act, int kind, void* out, int64_t* out_checksum, const abed_layer_shape* next,
                          int32_t* next_ic) {
  return guard([&] {
    const LayerShape ls = to_ls(s);
    FusedTaps taps;
    taps.output_checksum = out_checksum != nullptr;
    if (next) taps.next_layer = to_ls(next);
    const auto r = fused_conv_epilog(make(ls.input_dims(), ElemKind::I8, x), make(ls.filter_dims(), ElemKind::I8, f), ls,
                                     ep(scale, bias, ls.k, act, kind), taps);
    put(r.output, out);
    if (out_checksum) *out_checksum = *r.output_checksum;
    if (next) put(r.next_input_checksum->sums, next_ic);
  });
}
int ref_run_trial(const abed_layer_shape* s, const int8_t* x, const int8_t* f, int scheme, int target, float scale,
                  const float* bias, int64_t nb, int act, int kind, uint64_t seed, abed_trial_outcome* out) {
  return guard([&] {
    const LayerShape ls = to_ls(s);
    const TrialOutcome t = run_trial(ls, make(ls.input_dims(), ElemKind::I8, x), make(ls.filter_dims(), ElemKind::I8, f),
                                     static_cast<Scheme>(scheme), static_cast<InjectionTarget>(target),
                                     ep(scale, bias, nb, act, kind), seed);
    std::memset(out, 0, sizeof(*out));
    out->classification = (int)t.classification;
    out->target = (int)t.flipped.target;
    out->flat_index = t.flipped.flat_index;
    out->bit = t.flipped.bit;
    out->final_output_differs = t.final_output_differs ? 1 : 0;
    put_outcome(t.verify, &out->verify);
  });
}
int ref_run_campaign(const abed_campaign_config* c, abed_campaign_report* rep) {
  return guard([&] {
    CampaignConfig cfg;
    cfg.shape = to_ls(&c->shape);
    cfg.scheme = static_cast<Scheme>(c->scheme);
    cfg.target = static_cast<InjectionTarget>(c->target);
    cfg.trials = c->trials;
    cfg.root_seed = c->root_seed;
    cfg.mode = static_cast<DataMode>(c->mode);
    cfg.epilog = ep(c->scale, c->bias_host, c->bias_len, c->activation, c->output_kind);
    cfg.jobs = c->jobs;
    const CampaignReport r = run_campaign(cfg);
    rep->scheme = (int)r.scheme;
    rep->target = (int)r.target;
    rep->trials = r.trials;
    rep->detected = r.detected;
    rep->detected_benign = r.detected_benign;
    rep->sdc = r.sdc;
    rep->masked = r.masked;
    rep->seed = r.seed;
  });
}

// CPU baseline: the reference's own protected-layer path (SURVEY 8(d) / BASELINE.md
// section 3): conv_fast_i8 + scheme check + epilog, the batch split over
// `threads` std::threads each calling the reference functions on its sub-batch.
// scheme: -1 unprotected, ABED_FC, ABED_FIC, ABED_ICBATCH.  Returns seconds.
double ref_time_layer(const abed_layer_shape* s, int scheme, int threads, const int8_t* x, const int8_t* f) {
  const LayerShape full = to_ls(s);
  if (threads < 1) threads = 1;
  if (threads > full.n) threads = static_cast<int>(full.n);
  const Tensor4D filters = make(full.filter_dims(), ElemKind::I8, f);
  const FilterChecksum fc = gen_filter_checksum_decomposed(filters);  // offline, untimed
  EpilogParams p;
  p.scale = 0.05f;
  p.bias.assign(static_cast<std::size_t>(full.k), 0.0f);
  std::vector<Tensor4D> parts;
  std::vector<LayerShape> shapes;
  const int64_t chw = full.c * full.h * full.w;
  for (int t = 0; t < threads; ++t) {
    const int64_t n0 = full.n * t / threads, n1 = full.n * (t + 1) / threads;
    const LayerShape ls = LayerShape::make(n1 - n0, full.c, full.h, full.w, full.k, full.r, full.s, full.stride_h,
                                           full.stride_w, full.pad_h, full.pad_w);
    shapes.push_back(ls);
    parts.push_back(make(ls.input_dims(), ElemKind::I8, x + n0 * chw));
  }
  volatile int64_t sink = 0;
  auto work = [&](int t) {
    const LayerShape& ls = shapes[t];
    const Tensor4D convout = detail::conv_fast_i8(parts[t], filters, ls);
    bool ok = true;
    if (scheme == ABED_FC) {
      ok = fc_verify(convout, recombine_extra_fmaps(conv_checksum_planes(parts[t], ls, *fc.decomposed))).pass();
    } else if (scheme == ABED_FIC) {
      ok = fic_verify(convout, fic_dot(fc, gen_input_checksum(parts[t], ls))).pass();
    } else if (scheme == ABED_ICBATCH) {
      ok = ic_batch_verify(convout, conv_batch_checksum(ic_batch_checksum(parts[t]), filters, ls)).pass();
    }
    const Tensor4D out = epilog(convout, p);
    sink = sink + (ok ? 1 : 0) + out.view<const std::int8_t>()[0];
  };
  const auto t0 = std::chrono::steady_clock::now();
  std::vector<std::thread> pool;
  for (int t = 1; t < threads; ++t) pool.emplace_back(work, t);
  work(0);
  for (auto& th : pool) th.join();
  const auto t1 = std::chrono::steady_clock::now();
  return std::chrono::duration<double>(t1 - t0).count();
}

// abft_gemm.hpp:102-152 / :70-96 (row-major i8 operands; c_aug (m+1) x (n+1) i64)
int ref_abft_gemm(const int8_t* a, int64_t m, int64_t k, const int8_t* b, int64_t kb, int64_t n, int32_t* c,
                  int64_t* ca, abed_verify_outcome* row, abed_verify_outcome* col) {
  return guard([&] {
    Matrix am(m, k, ElemKind::I8), bm(kb, n, ElemKind::I8);
    std::memcpy(am.view<std::int8_t>().data(), a, (size_t)(m * k));
    std::memcpy(bm.view<std::int8_t>().data(), b, (size_t)(kb * n));
    const AbftResult r = abft_gemm(am, bm);
    if (c) std::memcpy(c, r.c.view<const std::int32_t>().data(), (size_t)(m * n) * 4);
    std::memcpy(ca, r.c_aug.view<const std::int64_t>().data(), (size_t)((m + 1) * (n + 1)) * 8);
    put_outcome(r.row_check, row);
    put_outcome(r.col_check, col);
  });
}
int ref_abft_check(const int64_t* ca, int64_t rows, int64_t cols, abed_verify_outcome* row, abed_verify_outcome* col) {
  return guard([&] {
    Matrix cm(rows, cols, ElemKind::I64);
    std::memcpy(cm.view<std::int64_t>().data(), ca, (size_t)(rows * cols) * 8);
    const auto [r, c] = abft_check(cm);
    put_outcome(r, row);
    put_outcome(c, col);
  });
}
// abft_gemm.hpp:41-55 abft_costs: 5 tasks x {ops, read, write, moved}
void ref_abft_costs(int64_t m, int64_t n, int64_t k, int single_pass, int64_t* out) {
  const AbftCosts cs = abft_costs(m, n, k, single_pass != 0);
  for (int t = 0; t < 5; ++t) {
    out[4 * t + 0] = cs.tasks[t].ops;
    out[4 * t + 1] = cs.tasks[t].read_bytes;
    out[4 * t + 2] = cs.tasks[t].write_bytes;
    out[4 * t + 3] = cs.tasks[t].elements_moved;
  }
}

}  // extern "C"
