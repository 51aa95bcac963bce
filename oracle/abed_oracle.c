/* abed_oracle.c -- TEST INFRASTRUCTURE ONLY: CPU restatement of the reference
 * ABED convolution path.  See abed_oracle.h for scope and pinning.  Each
 * function cites the reference file:line it restates (paths relative to
 * /root/reference/proj/include/abed/).
 */
#include "abed_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

#define ORA_OK ABED_OK
#define ORA_INVALID ABED_ERR_INVALID_ARGUMENT
#define ORA_RANGE ABED_ERR_OUT_OF_RANGE

static const uint64_t kGolden = 0x9E3779B97F4A7C15ULL;

/* ------------------------------------------------------------------ rng.hpp */
static uint64_t mix64(uint64_t z) { /* rng.hpp:16-19 */
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}
uint64_t ora_rng_next(ora_rng* g) { /* rng.hpp:15-20 */
  g->state += kGolden;
  return mix64(g->state);
}
uint64_t ora_rng_below(ora_rng* g, uint64_t bound) { /* rng.hpp:23-29 rejection sampling */
  const uint64_t threshold = (0 - bound) % bound;
  for (;;) {
    const uint64_t r = ora_rng_next(g);
    if (r >= threshold) return r % bound;
  }
}
uint64_t ora_derive_seed(uint64_t root, uint64_t index) { /* rng.hpp:41-44 */
  ora_rng g = {root ^ (0xA02E9D4BD1C96D4FULL + index * kGolden)};
  return ora_rng_next(&g);
}
int8_t ora_stream_i8(uint64_t seed, uint64_t i) { return (int8_t)(mix64(seed + (i + 1) * kGolden) & 0xFF); }
void ora_fill_random_i8(int8_t* t, int64_t n, ora_rng* g) { /* rng.hpp:46, next_i8 :31 */
  for (int64_t i = 0; i < n; ++i) t[i] = (int8_t)(ora_rng_next(g) & 0xFF);
}
void ora_fill_random_extreme(int8_t* t, int64_t n, ora_rng* g) { /* rng.hpp:51-53 */
  for (int64_t i = 0; i < n; ++i) t[i] = (ora_rng_next(g) & 1) ? (int8_t)127 : (int8_t)-128;
}
void ora_fill_random_f32(float* t, int64_t n, ora_rng* g, float lo, float hi) { /* rng.hpp:55-57, next_unit :33 */
  for (int64_t i = 0; i < n; ++i) {
    const double u = (double)(ora_rng_next(g) >> 11) * 0x1.0p-53;
    t[i] = fmaf((float)u, hi - lo, lo); /* lo + u*(hi-lo), contracted under -march=native */
  }
}
void ora_fill_random_f32_integers(float* t, int64_t n, ora_rng* g) { /* rng.hpp:60-62 */
  for (int64_t i = 0; i < n; ++i) t[i] = (float)(int8_t)(ora_rng_next(g) & 0xFF);
}

/* --------------------------------------------------------------- tensor.hpp */
int ora_layer_shape_make(int64_t n, int64_t c, int64_t h, int64_t w, int64_t k, int64_t r, int64_t s,
                         int64_t sh, int64_t sw, int64_t ph, int64_t pw, abed_layer_shape* o) {
  /* tensor.hpp:178-193 */
  if (n < 1 || c < 1 || h < 1 || w < 1 || k < 1 || r < 1 || s < 1) return ORA_INVALID;
  if (sh < 1 || sw < 1) return ORA_INVALID;
  if (ph < 0 || pw < 0) return ORA_INVALID;
  if (r > h + 2 * ph || s > w + 2 * pw) return ORA_INVALID;
  o->n = n; o->c = c; o->h = h; o->w = w; o->k = k; o->r = r; o->s = s;
  o->stride_h = sh; o->stride_w = sw; o->pad_h = ph; o->pad_w = pw;
  o->p = (h + 2 * ph - r) / sh + 1;
  o->q = (w + 2 * pw - s) / sw + 1;
  return ORA_OK;
}

/* ---------------------------------------------------------- convolution.hpp */
/* conv_reference (convolution.hpp:78-111): out[n,k,p,q] = sum over the window in
 * (c,r,s) order, halo positions skipped.  Loop nest reordered (window position
 * outermost per (n,k)) so the innermost q loop streams; each output still sees
 * its terms in (c,r,s) order, which keeps the f32 variant bit-identical. */
#define ORA_CONV_BODY(TACC, XV, FV, ACCUM)                                                        \
  const int64_t P = ls->p, Q = ls->q, H = ls->h, W = ls->w, C = ls->c, R = ls->r, S = ls->s;     \
  const int64_t K = ls->k;                                                                        \
  for (int64_t n = 0; n < ls->n; ++n)                                                             \
    for (int64_t k = 0; k < K; ++k) {                                                             \
      TACC* o = out + (n * K + k) * P * Q;                                                        \
      for (int64_t i = 0; i < P * Q; ++i) o[i] = 0;                                               \
      for (int64_t c = 0; c < C; ++c)                                                             \
        for (int64_t r = 0; r < R; ++r)                                                           \
          for (int64_t s = 0; s < S; ++s) {                                                       \
            const TACC fv = (TACC)(FV);                                                           \
            for (int64_t p = 0; p < P; ++p) {                                                     \
              const int64_t hi = p * ls->stride_h - ls->pad_h + r;                                \
              if (hi < 0 || hi >= H) continue;                                                    \
              for (int64_t q = 0; q < Q; ++q) {                                                   \
                const int64_t wi = q * ls->stride_w - ls->pad_w + s;                              \
                if (wi < 0 || wi >= W) continue;                                                  \
                const TACC xv = (TACC)(XV);                                                       \
                ACCUM;                                                                            \
              }                                                                                   \
            }                                                                                     \
          }                                                                                       \
    }

#define XIDX x[((n * C + c) * H + hi) * W + wi]
#define FIDX f[((k * C + c) * R + r) * S + s]

int ora_conv_i8(const int8_t* x, const int8_t* f, const abed_layer_shape* ls, int32_t* out) {
  if (ls->c * ls->r * ls->s > 65536) return ORA_INVALID; /* convolution.hpp:239-240 */
  ORA_CONV_BODY(int32_t, XIDX, FIDX, o[p * Q + q] += xv * fv)
  return ORA_OK;
}
int ora_conv_i8_w32_i64(const int8_t* x, const int32_t* f, const abed_layer_shape* ls, int64_t* out) {
  ORA_CONV_BODY(int64_t, XIDX, FIDX, o[p * Q + q] += xv * fv)
  return ORA_OK;
}
int ora_conv_x32_i8_i64(const int32_t* x, const int8_t* f, const abed_layer_shape* ls, int64_t* out) {
  ORA_CONV_BODY(int64_t, XIDX, FIDX, o[p * Q + q] += xv * fv)
  return ORA_OK;
}
int ora_conv_f32(const float* x, const float* f, const abed_layer_shape* ls, float* out) {
  /* convolution.hpp:245-248; acc += x*f contracts to fma(x, f, acc) */
  ORA_CONV_BODY(float, XIDX, FIDX, o[p * Q + q] = fmaf(xv, fv, o[p * Q + q]))
  return ORA_OK;
}
/* Depthwise conv (no reference counterpart -- parity unpinned):
 * conv_reference (convolution.hpp:78-111) with one filter per channel,
 * out[n,c,p,q] = sum_{r,s} x[n,c,..] f[c,0,r,s], halo skipped, int32. */
int ora_dwconv_i8(const int8_t* x, const int8_t* f, const abed_layer_shape* ls, int32_t* out) {
  const int64_t P = ls->p, Q = ls->q, H = ls->h, W = ls->w, C = ls->c, R = ls->r, S = ls->s;
  if (ls->k != ls->c) return ORA_INVALID;
  for (int64_t n = 0; n < ls->n; ++n)
    for (int64_t c = 0; c < C; ++c) {
      int32_t* o = out + (n * C + c) * P * Q;
      for (int64_t i = 0; i < P * Q; ++i) o[i] = 0;
      for (int64_t r = 0; r < R; ++r)
        for (int64_t s = 0; s < S; ++s) {
          const int32_t fv = f[(c * R + r) * S + s];
          for (int64_t p = 0; p < P; ++p) {
            const int64_t hi = p * ls->stride_h - ls->pad_h + r;
            if (hi < 0 || hi >= H) continue;
            for (int64_t q = 0; q < Q; ++q) {
              const int64_t wi = q * ls->stride_w - ls->pad_w + s;
              if (wi < 0 || wi >= W) continue;
              o[p * Q + q] += (int32_t)x[((n * C + c) * H + hi) * W + wi] * fv;
            }
          }
        }
    }
  return ORA_OK;
}

/* Float mode on tensor cores (no reference counterpart -- parity unpinned, see
 * DESIGN.md): conv_reference (convolution.hpp:78-111) with f64 accumulation, the
 * exact-as-possible value the fp16/bf16 tensor-core conv approximates (x, f are
 * f32 arrays already rounded to the 16-bit storage type). */
int ora_conv_f64(const float* x, const float* f, const abed_layer_shape* ls, double* out) {
  ORA_CONV_BODY(double, XIDX, FIDX, o[p * Q + q] += xv * fv)
  return ORA_OK;
}

int ora_epilog(const int32_t* in, abed_dims4 d, float scale, const float* bias, int64_t bias_len,
               int activation, int output_kind, void* out) {
  /* convolution.hpp:353-387 */
  if (bias_len != d.d1) return ORA_INVALID;
  if (!isfinite(scale)) return ORA_INVALID;
  for (int64_t i = 0; i < bias_len; ++i)
    if (!isfinite(bias[i])) return ORA_INVALID;
  if (output_kind != ABED_I8 && output_kind != ABED_F32) return ORA_INVALID;
  const int64_t pq = d.d2 * d.d3;
  int64_t idx = 0;
  for (int64_t n = 0; n < d.d0; ++n)
    for (int64_t k = 0; k < d.d1; ++k)
      for (int64_t j = 0; j < pq; ++j, ++idx) {
        float v = fmaf((float)in[idx], scale, bias[k]); /* float(acc)*scale + bias, FMA-contracted */
        if (activation == ABED_RELU && v < 0.0f) v = 0.0f;
        if (output_kind == ABED_F32) {
          ((float*)out)[idx] = v;
        } else {
          v = fminf(127.0f, fmaxf(-128.0f, v));
          ((int8_t*)out)[idx] = (int8_t)truncf(v);
        }
      }
  return ORA_OK;
}

/* -------------------------------------------------------------- checksum.hpp */
int ora_gen_filter_checksum(const int8_t* f, abed_dims4 fd, int32_t* sums) { /* :75-90 */
  if (fd.d0 > ((int64_t)1 << 24)) return ORA_INVALID;
  const int64_t crs = fd.d1 * fd.d2 * fd.d3;
  for (int64_t i = 0; i < crs; ++i) {
    int32_t acc = 0;
    for (int64_t k = 0; k < fd.d0; ++k) acc += f[k * crs + i];
    sums[i] = acc;
  }
  return ORA_OK;
}
void ora_decompose_value(int32_t v, int8_t out[4]) { /* :93-97 little-endian raw bytes */
  const uint32_t u = (uint32_t)v;
  for (int b = 0; b < 4; ++b) out[b] = (int8_t)(uint8_t)(u >> (8 * b));
}
int64_t ora_recombine_value(const int8_t d[4]) { /* :101-106 digits 0-2 unsigned, 3 signed */
  return (int64_t)(uint8_t)d[0] + ((int64_t)(uint8_t)d[1] << 8) + ((int64_t)(uint8_t)d[2] << 16) +
         ((int64_t)d[3] * 16777216);
}
void ora_decompose_checksum_filters(const int32_t* sums, int64_t n, int8_t* planes) { /* :108-122 */
  for (int64_t i = 0; i < n; ++i) {
    int8_t b[4];
    ora_decompose_value(sums[i], b);
    for (int p = 0; p < 4; ++p) planes[p * n + i] = b[p];
  }
}
int ora_conv_checksum_planes(const int8_t* x, const abed_layer_shape* ls, const int8_t* planes,
                             int32_t* extra) { /* :134-176 */
  const int64_t crs = ls->c * ls->r * ls->s;
  if (crs > 65536) return ORA_INVALID;
  const int64_t npq = ls->n * ls->p * ls->q;
  for (int64_t j = 0; j < npq; ++j) {
    const int64_t n = j / (ls->p * ls->q), p = (j / ls->q) % ls->p, q = j % ls->q;
    uint32_t acc[4] = {0, 0, 0, 0}; /* i32 accumulation (wraps like the reference would) */
    for (int64_t c = 0; c < ls->c; ++c)
      for (int64_t r = 0; r < ls->r; ++r)
        for (int64_t s = 0; s < ls->s; ++s) {
          const int64_t hi = p * ls->stride_h - ls->pad_h + r, wi = q * ls->stride_w - ls->pad_w + s;
          if (hi < 0 || hi >= ls->h || wi < 0 || wi >= ls->w) continue;
          const int32_t xv = x[((n * ls->c + c) * ls->h + hi) * ls->w + wi];
          const int64_t i = (c * ls->r + r) * ls->s + s;
          acc[0] += (uint32_t)(xv * (int32_t)(uint8_t)planes[0 * crs + i]);
          acc[1] += (uint32_t)(xv * (int32_t)(uint8_t)planes[1 * crs + i]);
          acc[2] += (uint32_t)(xv * (int32_t)(uint8_t)planes[2 * crs + i]);
          acc[3] += (uint32_t)(xv * (int32_t)planes[3 * crs + i]);
        }
    for (int p4 = 0; p4 < 4; ++p4) extra[p4 * npq + j] = (int32_t)acc[p4];
  }
  return ORA_OK;
}
void ora_recombine_extra_fmaps(const int32_t* e, int64_t n, int64_t* out) { /* :179-196 */
  for (int64_t i = 0; i < n; ++i)
    out[i] = (int64_t)e[i] + (int64_t)e[n + i] * 256 + (int64_t)e[2 * n + i] * 65536 + (int64_t)e[3 * n + i] * 16777216;
}
int ora_conv_filter_checksum(const int8_t* x, const abed_layer_shape* ls, const int32_t* sums, int64_t* out) {
  abed_layer_shape one = *ls; /* :201-206, conv_reference<i8,i32,i64> with k = 1 */
  one.k = 1;
  return ora_conv_i8_w32_i64(x, sums, &one, out);
}
static void outcome_ok(abed_verify_outcome* o) { memset(o, 0, sizeof(*o)); }
static void outcome_fail(abed_verify_outcome* o, int64_t lhs, int64_t rhs, int has_locus, int64_t l0, int64_t l1,
                         int64_t l2) {
  memset(o, 0, sizeof(*o));
  o->status = 1;
  o->lhs = lhs;
  o->rhs = rhs;
  o->has_locus = has_locus;
  o->locus[0] = l0; o->locus[1] = l1; o->locus[2] = l2;
}
int ora_fc_verify(const int32_t* cv, abed_dims4 d, const int64_t* ev, int64_t original_k, abed_verify_outcome* o) {
  /* :211-236; error_count extends the reference record (number of mismatching (n,p,q)) */
  const int64_t k_lim = original_k < 0 ? d.d1 : original_k;
  if (k_lim < 1 || k_lim > d.d1) return ORA_INVALID;
  const int64_t pq = d.d2 * d.d3;
  int found = 0;
  int64_t count = 0;
  for (int64_t n = 0; n < d.d0; ++n)
    for (int64_t j = 0; j < pq; ++j) {
      int64_t sum = 0;
      for (int64_t k = 0; k < k_lim; ++k) sum += cv[(n * d.d1 + k) * pq + j];
      const int64_t want = ev[n * pq + j];
      if (sum != want) {
        if (!found) outcome_fail(o, sum, want, 1, n, j / d.d3, j % d.d3);
        found = 1;
        ++count;
      }
    }
  if (!found) outcome_ok(o);
  o->error_count = count;
  return ORA_OK;
}
int ora_ceil_log2(int64_t v) { /* :53-62 */
  if (v < 1) return -1;
  int bits = 0;
  uint64_t u = (uint64_t)v - 1;
  while (u) { ++bits; u >>= 1; }
  return bits;
}
int ora_gen_input_checksum(const int8_t* x, const abed_layer_shape* ls, int32_t* sums) { /* :248-266 */
  if (8 + ora_ceil_log2(ls->n * ls->p * ls->q) > 32) return ORA_INVALID;
  const int64_t crs = ls->c * ls->r * ls->s;
  for (int64_t i = 0; i < crs; ++i) sums[i] = 0;
  for (int64_t n = 0; n < ls->n; ++n)
    for (int64_t p = 0; p < ls->p; ++p)
      for (int64_t q = 0; q < ls->q; ++q)
        for (int64_t c = 0; c < ls->c; ++c)
          for (int64_t r = 0; r < ls->r; ++r) {
            const int64_t hi = p * ls->stride_h - ls->pad_h + r;
            if (hi < 0 || hi >= ls->h) continue;
            for (int64_t s = 0; s < ls->s; ++s) {
              const int64_t wi = q * ls->stride_w - ls->pad_w + s;
              if (wi < 0 || wi >= ls->w) continue;
              sums[(c * ls->r + r) * ls->s + s] += x[((n * ls->c + c) * ls->h + hi) * ls->w + wi];
            }
          }
  return ORA_OK;
}
int64_t ora_reduce_all_i64(const int32_t* c, int64_t n) { /* :268-272 */
  int64_t s = 0;
  for (int64_t i = 0; i < n; ++i) s += c[i];
  return s;
}
int64_t ora_fic_dot(const int32_t* a, const int32_t* b, int64_t n) { /* :275-285 */
  int64_t acc = 0;
  for (int64_t i = 0; i < n; ++i) acc += (int64_t)a[i] * (int64_t)b[i];
  return acc;
}
void ora_fic_verify(const int32_t* c, int64_t n, int64_t expected, abed_verify_outcome* o) { /* :287-294 */
  const int64_t sum = ora_reduce_all_i64(c, n);
  if (sum != expected) {
    outcome_fail(o, sum, expected, 0, 0, 0, 0);
    o->error_count = 1;
  } else {
    outcome_ok(o);
    o->lhs = sum; /* Pass reports lhs = rhs = sum */
    o->rhs = expected;
  }
}
int32_t ora_reduce_all_wrap32(const int32_t* c, int64_t n) { /* :299-303 */
  uint32_t s = 0;
  for (int64_t i = 0; i < n; ++i) s += (uint32_t)c[i];
  return (int32_t)s;
}
void ora_fic_verify_forced32(const int32_t* c, int64_t n, int64_t expected, abed_verify_outcome* o) { /* :305-312 */
  const int64_t sum = ora_reduce_all_wrap32(c, n);
  if (sum != expected) {
    outcome_fail(o, sum, expected, 0, 0, 0, 0);
    o->error_count = 1;
  } else {
    outcome_ok(o);
    o->lhs = sum;
    o->rhs = expected;
  }
}
int ora_ic_verify_k(const int32_t* cv, abed_dims4 d, const int8_t* f, abed_dims4 fd, const int32_t* ic,
                    abed_verify_outcome* o) { /* :319-347 */
  if (fd.d0 != d.d1) return ORA_INVALID;
  const int64_t crs = fd.d1 * fd.d2 * fd.d3, pq = d.d2 * d.d3;
  int found = 0;
  int64_t count = 0;
  for (int64_t k = 0; k < d.d1; ++k) {
    int64_t out_sum = 0;
    for (int64_t n = 0; n < d.d0; ++n)
      for (int64_t j = 0; j < pq; ++j) out_sum += cv[(n * d.d1 + k) * pq + j];
    int64_t dot = 0;
    for (int64_t i = 0; i < crs; ++i) dot += (int64_t)f[k * crs + i] * (int64_t)ic[i];
    if (out_sum != dot) {
      if (!found) outcome_fail(o, out_sum, dot, 1, k, -1, -1);
      found = 1;
      ++count;
    }
  }
  if (!found) outcome_ok(o);
  o->error_count = count;
  return ORA_OK;
}
void ora_ic_batch_checksum(const int8_t* x, abed_dims4 d, int32_t* out) { /* :350-362 */
  const int64_t chw = d.d1 * d.d2 * d.d3;
  for (int64_t i = 0; i < chw; ++i) {
    int32_t acc = 0;
    for (int64_t n = 0; n < d.d0; ++n) acc += x[n * chw + i];
    out[i] = acc;
  }
}
int ora_conv_batch_checksum(const int32_t* batch, const int8_t* f, const abed_layer_shape* ls, int64_t* out) {
  /* :367-396: both the i8 fast path and the widened route yield the exact
   * integer convolution of the checksum image, computed here in i64 */
  abed_layer_shape one;
  int st = ora_layer_shape_make(1, ls->c, ls->h, ls->w, ls->k, ls->r, ls->s, ls->stride_h, ls->stride_w, ls->pad_h,
                                ls->pad_w, &one);
  if (st) return st;
  return ora_conv_x32_i8_i64(batch, f, &one, out);
}
int ora_ic_batch_verify(const int32_t* cv, abed_dims4 d, const int64_t* ev, abed_verify_outcome* o) { /* :398-421 */
  const int64_t kpq = d.d1 * d.d2 * d.d3, pq = d.d2 * d.d3;
  int found = 0;
  int64_t count = 0;
  for (int64_t i = 0; i < kpq; ++i) {
    int64_t sum = 0;
    for (int64_t n = 0; n < d.d0; ++n) sum += cv[n * kpq + i];
    if (sum != ev[i]) {
      if (!found) outcome_fail(o, sum, ev[i], 1, i / pq, (i % pq) / d.d3, i % d.d3);
      found = 1;
      ++count;
    }
  }
  if (!found) outcome_ok(o);
  o->error_count = count;
  return ORA_OK;
}
static int narrowest(int bits, int32_t* kind) { /* :444-448 */
  if (bits <= 32) { *kind = ABED_I32; return ORA_OK; }
  if (bits <= 64) { *kind = ABED_I64; return ORA_OK; }
  return ORA_INVALID;
}
int ora_plan_precision(const abed_layer_shape* ls, int b, abed_precision_plan* p) { /* :451-468 */
  if (b != 4 && b != 8) return ORA_INVALID;
  memset(p, 0, sizeof(*p));
  const int64_t crs = ls->c * ls->r * ls->s, npq = ls->n * ls->p * ls->q;
  p->operand_bits = b;
  p->bits_output_fmap = 2 * b + ora_ceil_log2(crs);
  p->bits_reduced_fc = 2 * b + ora_ceil_log2(crs * ls->k);
  p->bits_reduced_fic = 2 * b + ora_ceil_log2(npq * ls->k * crs);
  p->bits_filter_checksum = b + ora_ceil_log2(ls->k);
  p->bits_input_checksum = b + ora_ceil_log2(npq);
  int st = narrowest(p->bits_output_fmap, &p->output_fmap_kind);
  st = st ? st : narrowest(p->bits_reduced_fc, &p->reduced_fc_kind);
  st = st ? st : narrowest(p->bits_reduced_fic, &p->reduced_fic_kind);
  st = st ? st : narrowest(p->bits_filter_checksum, &p->filter_checksum_kind);
  st = st ? st : narrowest(p->bits_input_checksum, &p->input_checksum_kind);
  return st;
}

/* float mode, checksum.hpp:474-595 */
int ora_float_verify(double lhs, double rhs, double tau, abed_verify_outcome* o) { /* :474-481 */
  if (!(tau >= 0.0)) return ORA_INVALID;
  memset(o, 0, sizeof(*o));
  o->lhs_f = lhs;
  o->rhs_f = rhs;
  if (!(fabs(lhs - rhs) <= tau)) { o->status = 1; o->error_count = 1; }
  return ORA_OK;
}
void ora_filter_checksum_f64(const float* f, abed_dims4 fd, double* sums) { /* :483-494 */
  const int64_t crs = fd.d1 * fd.d2 * fd.d3;
  for (int64_t i = 0; i < crs; ++i) sums[i] = 0.0;
  for (int64_t k = 0; k < fd.d0; ++k)
    for (int64_t i = 0; i < crs; ++i) sums[i] += f[k * crs + i];
}
void ora_input_checksum_f64(const float* x, const abed_layer_shape* ls, double* sums) { /* :496-522 */
  const int64_t crs = ls->c * ls->r * ls->s;
  for (int64_t i = 0; i < crs; ++i) sums[i] = 0.0;
  for (int64_t n = 0; n < ls->n; ++n)
    for (int64_t p = 0; p < ls->p; ++p)
      for (int64_t q = 0; q < ls->q; ++q)
        for (int64_t c = 0; c < ls->c; ++c)
          for (int64_t r = 0; r < ls->r; ++r) {
            const int64_t hi = p * ls->stride_h - ls->pad_h + r;
            if (hi < 0 || hi >= ls->h) continue;
            for (int64_t s = 0; s < ls->s; ++s) {
              const int64_t wi = q * ls->stride_w - ls->pad_w + s;
              if (wi < 0 || wi >= ls->w) continue;
              sums[(c * ls->r + r) * ls->s + s] += x[((n * ls->c + c) * ls->h + hi) * ls->w + wi];
            }
          }
}
double ora_reduce_all_f64(const float* c, int64_t n) { /* :524-528 */
  double s = 0.0;
  for (int64_t i = 0; i < n; ++i) s += c[i];
  return s;
}
double ora_fic_dot_f64(const double* a, const double* b, int64_t n) { /* :530-535, acc += a*b -> fma */
  double acc = 0.0;
  for (int64_t i = 0; i < n; ++i) acc = fma(a[i], b[i], acc);
  return acc;
}
int ora_fic_verify_f32(const float* c, int64_t n, double expected, double tau, abed_verify_outcome* o) { /* :537-539 */
  return ora_float_verify(ora_reduce_all_f64(c, n), expected, tau, o);
}
int ora_fc_verify_f32(const float* cv, abed_dims4 d, const float* ev, double tau, abed_verify_outcome* o) { /* :541-565 */
  const int64_t pq = d.d2 * d.d3;
  for (int64_t n = 0; n < d.d0; ++n)
    for (int64_t j = 0; j < pq; ++j) {
      double sum = 0.0;
      for (int64_t k = 0; k < d.d1; ++k) sum += cv[(n * d.d1 + k) * pq + j];
      const double want = ev[n * pq + j];
      if (!(fabs(sum - want) <= tau)) {
        const int st = ora_float_verify(sum, want, tau, o);
        if (st) return st;
        o->has_locus = 1;
        o->locus[0] = n; o->locus[1] = j / d.d3; o->locus[2] = j % d.d3;
        return ORA_OK;
      }
    }
  outcome_ok(o);
  return ORA_OK;
}
int ora_ic_verify_k_f32(const float* cv, abed_dims4 d, const float* f, abed_dims4 fd, const double* ic, double tau,
                        abed_verify_outcome* o) { /* :567-595 */
  const int64_t crs = fd.d1 * fd.d2 * fd.d3, pq = d.d2 * d.d3;
  for (int64_t k = 0; k < d.d1; ++k) {
    double out_sum = 0.0;
    for (int64_t n = 0; n < d.d0; ++n)
      for (int64_t j = 0; j < pq; ++j) out_sum += cv[(n * d.d1 + k) * pq + j];
    double dot = 0.0;
    for (int64_t i = 0; i < crs; ++i) dot = fma((double)f[k * crs + i], ic[i], dot);
    if (!(fabs(out_sum - dot) <= tau)) {
      const int st = ora_float_verify(out_sum, dot, tau, o);
      if (st) return st;
      o->has_locus = 1;
      o->locus[0] = k; o->locus[1] = -1; o->locus[2] = -1;
      return ORA_OK;
    }
  }
  outcome_ok(o);
  return ORA_OK;
}

int ora_fused_conv_epilog(const int8_t* x, const int8_t* f, const abed_layer_shape* ls, float scale,
                          const float* bias, int activation, int output_kind, void* out, int64_t* out_checksum,
                          const abed_layer_shape* next, int32_t* next_ic) { /* :616-631 */
  const int64_t nkpq = ls->n * ls->k * ls->p * ls->q;
  int32_t* conv = (int32_t*)malloc((size_t)nkpq * sizeof(int32_t));
  int st = ora_conv_i8(x, f, ls, conv);
  if (!st && out_checksum) *out_checksum = ora_reduce_all_i64(conv, nkpq);
  const abed_dims4 d = {ls->n, ls->k, ls->p, ls->q};
  if (!st) st = ora_epilog(conv, d, scale, bias, ls->k, activation, output_kind, out);
  if (!st && next) {
    if (output_kind != ABED_I8) st = ORA_INVALID;
    else if (next->n != ls->n || next->c != ls->k || next->h != ls->p || next->w != ls->q) st = ORA_INVALID;
    else st = ora_gen_input_checksum((const int8_t*)out, next, next_ic);
  }
  free(conv);
  return st;
}

/* ---------------------------------------------------------------- faults.hpp */
static int64_t esize(int kind) { return kind == ABED_I8 ? 1 : kind == ABED_I64 ? 8 : 4; }
int ora_flip_bit(void* data, int kind, int64_t count, int64_t flat_index, int bit) { /* :53-62 */
  if (flat_index < 0 || flat_index >= count) return ORA_RANGE;
  if (bit < 0 || bit >= 8 * esize(kind)) return ORA_RANGE;
  uint8_t* b = (uint8_t*)data;
  b[flat_index * esize(kind) + bit / 8] ^= (uint8_t)(1u << (bit % 8));
  return ORA_OK;
}

typedef struct trial_ctx { /* faults.hpp:116-130 */
  abed_layer_shape ls;
  int scheme, activation, output_kind;
  float scale;
  float* bias;
  const int8_t *x, *f;
  int32_t* conv_golden;
  uint8_t* out_golden;
  int32_t *fsum, *icsum;
  int8_t* planes;
  int64_t* fc_extra_golden;
  int64_t fic_expected;
} trial_ctx;

static void ctx_free(trial_ctx* c) {
  free(c->bias); free(c->conv_golden); free(c->out_golden); free(c->fsum); free(c->icsum);
  free(c->planes); free(c->fc_extra_golden);
  memset(c, 0, sizeof(*c));
}

static int64_t fc_extra(const trial_ctx* c, const int8_t* x, int64_t* out) {
  const int64_t npq = c->ls.n * c->ls.p * c->ls.q;
  int32_t* e = (int32_t*)malloc((size_t)(4 * npq) * sizeof(int32_t));
  int st = ora_conv_checksum_planes(x, &c->ls, c->planes, e);
  if (!st) ora_recombine_extra_fmaps(e, npq, out);
  free(e);
  return st;
}

static int ctx_make(trial_ctx* c, const abed_layer_shape* ls, const int8_t* x, const int8_t* f, int scheme,
                    float scale, const float* bias, int64_t bias_len, int activation, int output_kind) {
  /* faults.hpp:158-191 */
  memset(c, 0, sizeof(*c));
  if (scheme == ABED_ICBATCH) return ORA_INVALID;
  c->ls = *ls; c->scheme = scheme; c->scale = scale; c->activation = activation; c->output_kind = output_kind;
  c->x = x; c->f = f;
  c->bias = (float*)calloc((size_t)ls->k, sizeof(float));
  if (bias && bias_len > 0) {
    if (bias_len != ls->k) { ctx_free(c); return ORA_INVALID; }
    memcpy(c->bias, bias, (size_t)ls->k * sizeof(float));
  }
  const int64_t nkpq = ls->n * ls->k * ls->p * ls->q, crs = ls->c * ls->r * ls->s;
  c->conv_golden = (int32_t*)malloc((size_t)nkpq * 4);
  c->out_golden = (uint8_t*)malloc((size_t)nkpq * 4);
  int st = ora_conv_i8(x, f, ls, c->conv_golden);
  const abed_dims4 d = {ls->n, ls->k, ls->p, ls->q};
  if (!st) st = ora_epilog(c->conv_golden, d, scale, c->bias, ls->k, activation, output_kind, c->out_golden);
  if (st) { ctx_free(c); return st; }
  c->fsum = (int32_t*)malloc((size_t)crs * 4);
  c->icsum = (int32_t*)malloc((size_t)crs * 4);
  const abed_dims4 fd = {ls->k, ls->c, ls->r, ls->s};
  if (scheme == ABED_FC) {
    ora_gen_filter_checksum(f, fd, c->fsum);
    c->planes = (int8_t*)malloc((size_t)(4 * crs));
    ora_decompose_checksum_filters(c->fsum, crs, c->planes);
    c->fc_extra_golden = (int64_t*)malloc((size_t)(ls->n * ls->p * ls->q) * 8);
    st = (int)fc_extra(c, x, c->fc_extra_golden);
  } else if (scheme == ABED_IC) {
    st = ora_gen_input_checksum(x, ls, c->icsum);
  } else {
    ora_gen_filter_checksum(f, fd, c->fsum);
    st = ora_gen_input_checksum(x, ls, c->icsum);
    c->fic_expected = ora_fic_dot(c->fsum, c->icsum, crs);
  }
  if (st) ctx_free(c);
  return st;
}

static int trial_exec(const trial_ctx* c, int target, uint64_t seed, abed_trial_outcome* out) {
  /* faults.hpp:197-262 */
  const abed_layer_shape* ls = &c->ls;
  const int64_t nchw = ls->n * ls->c * ls->h * ls->w, kcrs = ls->k * ls->c * ls->r * ls->s;
  const int64_t nkpq = ls->n * ls->k * ls->p * ls->q, npq = ls->n * ls->p * ls->q;
  ora_rng g = {seed};
  const int64_t count = target == ABED_TARGET_INPUT ? nchw : target == ABED_TARGET_FILTER ? kcrs : nkpq;
  const int bits = target == ABED_TARGET_CONVOUT ? 32 : 8;
  memset(out, 0, sizeof(*out));
  out->target = target;
  out->flat_index = (int64_t)ora_rng_below(&g, (uint64_t)count);
  out->bit = (int)ora_rng_below(&g, (uint64_t)bits);

  int32_t* conv = (int32_t*)malloc((size_t)nkpq * 4);
  int8_t* flipped = NULL;
  int64_t* extra = NULL;
  const int8_t* verify_f = c->f;
  if (target == ABED_TARGET_INPUT) {
    flipped = (int8_t*)malloc((size_t)nchw);
    memcpy(flipped, c->x, (size_t)nchw);
    ora_flip_bit(flipped, ABED_I8, nchw, out->flat_index, out->bit);
    ora_conv_i8(flipped, c->f, ls, conv);
    if (c->scheme == ABED_FC) {
      extra = (int64_t*)malloc((size_t)npq * 8);
      fc_extra(c, flipped, extra);
    }
  } else if (target == ABED_TARGET_FILTER) {
    flipped = (int8_t*)malloc((size_t)kcrs);
    memcpy(flipped, c->f, (size_t)kcrs);
    ora_flip_bit(flipped, ABED_I8, kcrs, out->flat_index, out->bit);
    verify_f = flipped;
    ora_conv_i8(c->x, flipped, ls, conv);
  } else {
    memcpy(conv, c->conv_golden, (size_t)nkpq * 4);
    ora_flip_bit(conv, ABED_I32, nkpq, out->flat_index, out->bit);
  }
  const abed_dims4 d = {ls->n, ls->k, ls->p, ls->q};
  const abed_dims4 fd = {ls->k, ls->c, ls->r, ls->s};
  if (c->scheme == ABED_FC) ora_fc_verify(conv, d, extra ? extra : c->fc_extra_golden, ls->k, &out->verify);
  else if (c->scheme == ABED_IC) ora_ic_verify_k(conv, d, verify_f, fd, c->icsum, &out->verify);
  else ora_fic_verify(conv, nkpq, c->fic_expected, &out->verify);

  const int64_t ob = nkpq * (c->output_kind == ABED_F32 ? 4 : 1);
  uint8_t* o = (uint8_t*)malloc((size_t)ob);
  ora_epilog(conv, d, c->scale, c->bias, ls->k, c->activation, c->output_kind, o);
  out->final_output_differs = memcmp(o, c->out_golden, (size_t)ob) != 0;
  if (out->verify.status == 0)
    out->classification = out->final_output_differs ? ABED_SDC : ABED_MASKED;
  else
    out->classification = out->final_output_differs ? ABED_DETECTED : ABED_DETECTED_BENIGN;
  free(o); free(conv); free(flipped); free(extra);
  return ORA_OK;
}

int ora_run_trial(const abed_layer_shape* ls, const int8_t* x, const int8_t* f, int scheme, int target, float scale,
                  const float* bias, int64_t bias_len, int activation, int output_kind, uint64_t seed,
                  abed_trial_outcome* out) { /* faults.hpp:268-274 */
  trial_ctx c;
  int st = ctx_make(&c, ls, x, f, scheme, scale, bias, bias_len, activation, output_kind);
  if (st) return st;
  st = trial_exec(&c, target, seed, out);
  ctx_free(&c);
  return st;
}

int ora_run_campaign(const abed_campaign_config* cfg, int64_t t_begin, int64_t t_end, abed_campaign_report* rep) {
  /* faults.hpp:276-333; trials folded in order, independent of any worker split */
  if (cfg->trials < 1) return ORA_INVALID;
  const abed_layer_shape* ls = &cfg->shape;
  const int64_t nchw = ls->n * ls->c * ls->h * ls->w, kcrs = ls->k * ls->c * ls->r * ls->s;
  int8_t* x = (int8_t*)malloc((size_t)nchw);
  int8_t* f = (int8_t*)malloc((size_t)kcrs);
  if (cfg->mode == ABED_DATA_ONES) {
    memset(x, 1, (size_t)nchw);
    memset(f, 1, (size_t)kcrs);
  } else {
    ora_rng g = {ora_derive_seed(cfg->root_seed, 0x0DA7Au)};
    ora_fill_random_i8(x, nchw, &g);
    ora_fill_random_i8(f, kcrs, &g);
  }
  trial_ctx c;
  int st = ctx_make(&c, ls, x, f, cfg->scheme, cfg->scale, cfg->bias_host, cfg->bias_len, cfg->activation,
                    cfg->output_kind);
  if (!st) {
    memset(rep, 0, sizeof(*rep));
    rep->scheme = cfg->scheme;
    rep->target = cfg->target;
    rep->seed = cfg->root_seed;
    if (t_begin < 0) t_begin = 0;
    if (t_end > cfg->trials) t_end = cfg->trials;
    rep->trials = t_end > t_begin ? t_end - t_begin : 0;
    for (int64_t t = t_begin; t < t_end; ++t) {
      abed_trial_outcome o;
      trial_exec(&c, cfg->target, ora_derive_seed(cfg->root_seed, (uint64_t)t), &o);
      switch (o.classification) {
        case ABED_DETECTED: ++rep->detected; break;
        case ABED_DETECTED_BENIGN: ++rep->detected_benign; break;
        case ABED_SDC: ++rep->sdc; break;
        default: ++rep->masked; break;
      }
    }
    ctx_free(&c);
  }
  free(x);
  free(f);
  return st;
}

/* ------------------------------------------------------------------ ABFT GEMM */
int ora_abft_check(const int64_t* ca, int64_t rows, int64_t cols, abed_verify_outcome* row,
                   abed_verify_outcome* col) { /* abft_gemm.hpp:70-96 */
  const int64_t m = rows - 1, n = cols - 1;
  if (m < 1 || n < 1) return ORA_INVALID;
  int64_t bad = 0;
  outcome_ok(row);
  for (int64_t i = 0; i <= m; ++i) { /* row sums vs the appended column */
    uint64_t sum = 0; /* int64 wraparound, as the reference's two's-complement sums */
    for (int64_t j = 0; j < n; ++j) sum += (uint64_t)ca[i * cols + j];
    if ((int64_t)sum != ca[i * cols + n]) {
      if (!bad) outcome_fail(row, (int64_t)sum, ca[i * cols + n], 1, i, -1, -1);
      ++bad;
    }
  }
  row->error_count = bad;
  bad = 0;
  outcome_ok(col);
  for (int64_t j = 0; j <= n; ++j) { /* column sums vs the appended row */
    uint64_t sum = 0;
    for (int64_t i = 0; i < m; ++i) sum += (uint64_t)ca[i * cols + j];
    if ((int64_t)sum != ca[m * cols + j]) {
      if (!bad) outcome_fail(col, (int64_t)sum, ca[m * cols + j], 1, j, -1, -1);
      ++bad;
    }
  }
  col->error_count = bad;
  return ORA_OK;
}
int ora_abft_gemm(const int8_t* a, int64_t m, int64_t k, const int8_t* b, int64_t kb, int64_t n, int32_t* c,
                  int64_t* ca, abed_verify_outcome* row, abed_verify_outcome* col) { /* abft_gemm.hpp:102-152 */
  if (m < 1 || n < 1 || k < 1 || k != kb) return ORA_INVALID;
  if (16 + ora_ceil_log2(m * n * k) > 63 || 16 + ora_ceil_log2(k) > 31) return ORA_INVALID;
  int32_t* colsum = (int32_t*)calloc((size_t)k, 4); /* task (3): A column sums, B row sums (i32) */
  int32_t* rowsum = (int32_t*)calloc((size_t)k, 4);
  if (!colsum || !rowsum) { free(colsum); free(rowsum); return ORA_INVALID; }
  for (int64_t t = 0; t < k; ++t) {
    for (int64_t i = 0; i < m; ++i) colsum[t] += a[i * k + t];
    for (int64_t j = 0; j < n; ++j) rowsum[t] += b[t * n + j];
  }
  const int64_t cols = n + 1; /* task (4): (m+1) x (n+1) product of the augmented operands in i64 */
  for (int64_t i = 0; i <= m; ++i)
    for (int64_t j = 0; j <= n; ++j) {
      int64_t acc = 0;
      for (int64_t t = 0; t < k; ++t) {
        const int64_t x = i < m ? a[i * k + t] : colsum[t];
        const int64_t y = j < n ? b[t * n + j] : rowsum[t];
        acc += x * y;
      }
      ca[i * cols + j] = acc;
    }
  free(colsum);
  free(rowsum);
  ora_abft_check(ca, m + 1, n + 1, row, col); /* task (5) */
  if (c)                                      /* task (6): trimmed copy-out */
    for (int64_t i = 0; i < m; ++i)
      for (int64_t j = 0; j < n; ++j) c[i * n + j] = (int32_t)ca[i * cols + j];
  return ORA_OK;
}
