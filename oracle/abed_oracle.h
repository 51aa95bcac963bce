/* abed_oracle.h -- TEST INFRASTRUCTURE ONLY.
 *
 * A plain-C (C99) restatement of the reference's ABED convolution path
 * (/root/reference/proj/include/abed/{rng,tensor,convolution,checksum,faults}.hpp),
 * used exclusively as the CPU checker by tests/, __graft_entry__.smoke() and the
 * cpu_baseline leg of bench.py.  Nothing in the product (libabed_b200.so,
 * include/abed/*.hpp) links or calls it.
 *
 * Parity pinning: tests/test_oracle_golden.py checks every function against the
 * reference's own known-answer tests and against golden vectors
 * produced by the reference itself (oracle/_ref, built from the reference
 * headers by oracle/Makefile; tests/golden/make_golden.py).
 *
 * Layouts follow the reference: NCHW activations, KCRS filters, NKPQ ConvOut,
 * 1xCxRxS checksums (tensor.hpp:68-70).  Errors mirror the reference's
 * exceptions as status codes (ABED_ERR_* from include/abed_b200.h).  Floating
 * point: the reference's Release build uses -march=native, under which GCC
 * contracts `a * b + c` to an FMA; the oracle spells those FMAs out
 * with fma()/fmaf() so its rounding does not depend on its own build flags.
 */
#ifndef ABED_ORACLE_H
#define ABED_ORACLE_H

#include <stdint.h>

#include "../include/abed_b200.h"

#ifdef __cplusplus
extern "C" {
#endif

/* rng.hpp:11-62 */
typedef struct ora_rng { uint64_t state; } ora_rng;
uint64_t ora_rng_next(ora_rng* g);
uint64_t ora_rng_below(ora_rng* g, uint64_t bound);
uint64_t ora_derive_seed(uint64_t root, uint64_t index);
void ora_fill_random_i8(int8_t* t, int64_t n, ora_rng* g);
void ora_fill_random_extreme(int8_t* t, int64_t n, ora_rng* g);
void ora_fill_random_f32(float* t, int64_t n, ora_rng* g, float lo, float hi);
void ora_fill_random_f32_integers(float* t, int64_t n, ora_rng* g);
/* index-parallel form used by the device fill: element i of a fresh stream */
int8_t ora_stream_i8(uint64_t seed, uint64_t i);

/* tensor.hpp:178-193 */
int ora_layer_shape_make(int64_t n, int64_t c, int64_t h, int64_t w, int64_t k, int64_t r, int64_t s,
                         int64_t sh, int64_t sw, int64_t ph, int64_t pw, abed_layer_shape* out);

/* convolution.hpp:78-111 conv_reference, the instantiations the reference uses */
int ora_conv_i8(const int8_t* x, const int8_t* f, const abed_layer_shape* ls, int32_t* out);
int ora_conv_i8_w32_i64(const int8_t* x, const int32_t* f, const abed_layer_shape* ls, int64_t* out);
int ora_conv_x32_i8_i64(const int32_t* x, const int8_t* f, const abed_layer_shape* ls, int64_t* out);
int ora_conv_f32(const float* x, const float* f, const abed_layer_shape* ls, float* out);
int ora_dwconv_i8(const int8_t* x, const int8_t* f, const abed_layer_shape* ls, int32_t* out);
int ora_conv_f64(const float* x, const float* f, const abed_layer_shape* ls, double* out);
/* convolution.hpp:353-387 */
int ora_epilog(const int32_t* convout, abed_dims4 d, float scale, const float* bias, int64_t bias_len,
               int activation, int output_kind, void* out);

/* checksum.hpp */
int ora_gen_filter_checksum(const int8_t* f, abed_dims4 fd, int32_t* sums);           /* :75  */
void ora_decompose_value(int32_t v, int8_t out[4]);                                 /* :93  */
int64_t ora_recombine_value(const int8_t d[4]);                                     /* :101 */
void ora_decompose_checksum_filters(const int32_t* sums, int64_t n, int8_t* planes); /* :108 */
int ora_conv_checksum_planes(const int8_t* x, const abed_layer_shape* ls, const int8_t* planes,
                             int32_t* extra);                                       /* :134 */
void ora_recombine_extra_fmaps(const int32_t* extra, int64_t n, int64_t* out);      /* :179 */
int ora_conv_filter_checksum(const int8_t* x, const abed_layer_shape* ls, const int32_t* sums,
                             int64_t* out);                                         /* :201 */
int ora_fc_verify(const int32_t* convout, abed_dims4 d, const int64_t* extra, int64_t original_k,
                  abed_verify_outcome* o);                                          /* :211 */
int ora_gen_input_checksum(const int8_t* x, const abed_layer_shape* ls, int32_t* sums); /* :248 */
int64_t ora_reduce_all_i64(const int32_t* c, int64_t n);                            /* :268 */
int64_t ora_fic_dot(const int32_t* fc, const int32_t* ic, int64_t n);               /* :275 */
void ora_fic_verify(const int32_t* c, int64_t n, int64_t expected, abed_verify_outcome* o);  /* :287 */
int32_t ora_reduce_all_wrap32(const int32_t* c, int64_t n);                         /* :299 */
void ora_fic_verify_forced32(const int32_t* c, int64_t n, int64_t expected, abed_verify_outcome* o); /* :305 */
int ora_ic_verify_k(const int32_t* convout, abed_dims4 d, const int8_t* f, abed_dims4 fd,
                    const int32_t* ic, abed_verify_outcome* o);                     /* :319 */
void ora_ic_batch_checksum(const int8_t* x, abed_dims4 d, int32_t* out);            /* :350 */
int ora_conv_batch_checksum(const int32_t* batch, const int8_t* f, const abed_layer_shape* ls,
                            int64_t* out);                                          /* :367 */
int ora_ic_batch_verify(const int32_t* convout, abed_dims4 d, const int64_t* extra,
                        abed_verify_outcome* o);                                    /* :398 */
int ora_ceil_log2(int64_t v);                                                       /* :53  */
int ora_plan_precision(const abed_layer_shape* ls, int bits, abed_precision_plan* p); /* :451 */

/* float mode, checksum.hpp:474-595 */
int ora_float_verify(double lhs, double rhs, double tau, abed_verify_outcome* o);
void ora_filter_checksum_f64(const float* f, abed_dims4 fd, double* sums);
void ora_input_checksum_f64(const float* x, const abed_layer_shape* ls, double* sums);
double ora_reduce_all_f64(const float* c, int64_t n);
double ora_fic_dot_f64(const double* a, const double* b, int64_t n);
int ora_fic_verify_f32(const float* c, int64_t n, double expected, double tau, abed_verify_outcome* o);
int ora_fc_verify_f32(const float* c, abed_dims4 d, const float* extra, double tau, abed_verify_outcome* o);
int ora_ic_verify_k_f32(const float* c, abed_dims4 d, const float* f, abed_dims4 fd, const double* ic,
                        double tau, abed_verify_outcome* o);

/* checksum.hpp:616-631 fused_conv_epilog; out_checksum/next_ic may be NULL (tap off) */
int ora_fused_conv_epilog(const int8_t* x, const int8_t* f, const abed_layer_shape* ls, float scale,
                          const float* bias, int activation, int output_kind, void* out,
                          int64_t* out_checksum, const abed_layer_shape* next, int32_t* next_ic);

/* faults.hpp */
int ora_flip_bit(void* data, int kind, int64_t count, int64_t flat_index, int bit); /* :53 */
int ora_run_trial(const abed_layer_shape* ls, const int8_t* x, const int8_t* f, int scheme, int target,
                  float scale, const float* bias, int64_t bias_len, int activation, int output_kind,
                  uint64_t seed, abed_trial_outcome* out);                          /* :268 */
int ora_run_campaign(const abed_campaign_config* cfg, int64_t t_begin, int64_t t_end,
                     abed_campaign_report* rep);                                    /* :276 */

/* abft_gemm.hpp:70-96 abft_check / :102-152 abft_gemm (row-major i8 A m x k, B k x n) */
int ora_abft_check(const int64_t* c_aug, int64_t rows, int64_t cols, abed_verify_outcome* row,
                   abed_verify_outcome* col);
int ora_abft_gemm(const int8_t* a, int64_t m, int64_t k, const int8_t* b, int64_t kb, int64_t n, int32_t* c,
                  int64_t* c_aug, abed_verify_outcome* row, abed_verify_outcome* col);

#ifdef __cplusplus
}
#endif
#endif
