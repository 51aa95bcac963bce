/* abed_b200.h -- C ABI of the B200-native ABED convolution library
 * (libabed_b200.so).  Plain C: pointers, sizes and POD structs only.
 *
 * Every entry point replaces one function of the reference's header-only C++
 * API (/root/reference/proj/include/abed/*.hpp); the reference file:line is
 * cited beside each declaration.  Tensors keep the reference layouts (NCHW
 * activations, KCRS filters, N x K x P x Q ConvOut, 1 x C x R x S checksums;
 * tensor.hpp:68-70) and are passed as DEVICE pointers unless stated otherwise;
 * `stream` is a cudaStream_t (NULL = legacy default stream).
 *
 * Error convention (mirrors the reference's exceptions):
 *   ABED_OK                    success
 *   ABED_ERR_INVALID_ARGUMENT  reference throws std::invalid_argument
 *   ABED_ERR_OUT_OF_RANGE      reference throws std::out_of_range
 *   ABED_ERR_RUNTIME           reference throws std::runtime_error
 *   ABED_ERR_CUDA              CUDA failure (no reference counterpart)
 *   ABED_ERR_NO_DEVICE         no usable sm_100 device: the library never falls
 *                              back to host computation
 * A checksum mismatch is NOT an error: it is abed_verify_outcome.status = 1.
 * abed_last_error() returns the message of the last failing call (thread-local).
 */
#ifndef ABED_B200_H
#define ABED_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
  ABED_OK = 0,
  ABED_ERR_INVALID_ARGUMENT = 1,
  ABED_ERR_OUT_OF_RANGE = 2,
  ABED_ERR_RUNTIME = 3,
  ABED_ERR_CUDA = 4,
  ABED_ERR_NO_DEVICE = 5
};

/* element kinds, tensor.hpp:20 (ElemKind : uint8_t {I8, I32, I64, F32}) */
enum { ABED_I8 = 0, ABED_I32 = 1, ABED_I64 = 2, ABED_F32 = 3 };
/* float mode on tensor cores (extension): 16-bit operand storage kinds */
enum { ABED_F16 = 4, ABED_BF16 = 5 };
/* convolution.hpp:342 Activation */
enum { ABED_RELU = 0, ABED_IDENTITY = 1 };
/* checksum.hpp:15 Scheme */
enum { ABED_FC = 0, ABED_IC = 1, ABED_ICBATCH = 2, ABED_FIC = 3 };
/* faults.hpp:17 InjectionTarget, :28 Classification, :71 DataMode */
enum { ABED_TARGET_INPUT = 0, ABED_TARGET_FILTER = 1, ABED_TARGET_CONVOUT = 2 };
enum { ABED_DETECTED = 0, ABED_SDC = 1, ABED_MASKED = 2, ABED_DETECTED_BENIGN = 3 };
enum { ABED_DATA_ONES = 0, ABED_DATA_RANDOM_I8 = 1 };

/* tensor.hpp:58-66 Dims4 */
typedef struct abed_dims4 {
  int64_t d0, d1, d2, d3;
} abed_dims4;

/* tensor.hpp:171-203 LayerShape (same field order) */
typedef struct abed_layer_shape {
  int64_t n, c, h, w, k, r, s, stride_h, stride_w, pad_h, pad_w, p, q;
} abed_layer_shape;

/* convolution.hpp:346-351 EpilogParams; bias = DEVICE pointer, K floats */
typedef struct abed_epilog_params {
  float scale;
  const float* bias;
  int64_t bias_len;
  int32_t activation;  /* ABED_RELU / ABED_IDENTITY */
  int32_t output_kind; /* ABED_I8 / ABED_F32 */
} abed_epilog_params;

/* checksum.hpp:30-51 VerifyOutcome (+ error_count: number of mismatching loci) */
typedef struct abed_verify_outcome {
  int32_t status;    /* 0 = Pass, 1 = Mismatch */
  int32_t has_locus; /* locus present */
  int64_t locus[3];
  int64_t lhs, rhs;
  double lhs_f, rhs_f;
  int64_t error_count;
} abed_verify_outcome;

/* checksum.hpp:429-441 PrecisionPlan */
typedef struct abed_precision_plan {
  int32_t operand_bits, bits_output_fmap, bits_reduced_fc, bits_reduced_fic;
  int32_t bits_filter_checksum, bits_input_checksum;
  int32_t output_fmap_kind, reduced_fc_kind, reduced_fic_kind;
  int32_t filter_checksum_kind, input_checksum_kind;
} abed_precision_plan;

/* faults.hpp:77-86 CampaignConfig (epilog bias is HOST memory here, may be NULL = zeros) */
typedef struct abed_campaign_config {
  abed_layer_shape shape;
  int32_t scheme, target;
  int64_t trials;
  uint64_t root_seed;
  int32_t mode;
  float scale;
  const float* bias_host;
  int64_t bias_len;
  int32_t activation, output_kind;
  int32_t jobs; /* accepted for API parity; the GPU batches trials itself */
} abed_campaign_config;

/* faults.hpp:88-107 CampaignReport */
typedef struct abed_campaign_report {
  int32_t scheme, target;
  int64_t trials, detected, detected_benign, sdc, masked;
  uint64_t seed;
} abed_campaign_report;

/* faults.hpp:40-51 TrialOutcome (FlipSpec folded in) */
typedef struct abed_trial_outcome {
  int32_t classification;
  int32_t target;
  int64_t flat_index;
  int32_t bit;
  int32_t final_output_differs;
  abed_verify_outcome verify;
} abed_trial_outcome;

/* ------------------------------------------------------------ library / device */
const char* abed_last_error(void);
int abed_device_check(void); /* ABED_OK iff an sm_100 device is present */
int abed_version(void);
int abed_malloc(void** dptr, size_t bytes);
int abed_free(void* dptr);
int abed_memcpy_h2d(void* dst, const void* src, size_t bytes);
int abed_memcpy_d2h(void* dst, const void* src, size_t bytes);
int abed_memset(void* dptr, int value, size_t bytes);
int abed_synchronize(void);

/* ------------------------------------------------------------ L0 data / rng */
/* tensor.hpp:178-193 LayerShape::make (validation + derived p, q) */
int abed_layer_shape_make(int64_t n, int64_t c, int64_t h, int64_t w, int64_t k, int64_t r,
                          int64_t s, int64_t stride_h, int64_t stride_w, int64_t pad_h,
                          int64_t pad_w, abed_layer_shape* out);
/* rng.hpp:11-37 SplitMix64 stream element i = mix(seed + (i+1)*golden): index-parallel fill.
 * fill_random_i8 (rng.hpp:46) continuing a stream already advanced by `offset` draws. */
int abed_fill_random_i8(int8_t* data, int64_t count, uint64_t seed, uint64_t offset, void* stream);
/* rng.hpp:51 fill_random_extreme */
int abed_fill_random_extreme(int8_t* data, int64_t count, uint64_t seed, uint64_t offset, void* stream);
/* rng.hpp:41-44 derive_seed (host) */
uint64_t abed_derive_seed(uint64_t root, uint64_t index);

/* ------------------------------------------------------------ L1 convolution */
/* convolution.hpp:237 conv_direct / :224 detail::conv_fast_i8: int8 x int8 -> int32 ConvOut.
 * ABED_ERR_INVALID_ARGUMENT when CRS > 65536 (:239-240).  tcgen05 implicit GEMM. */
int abed_conv_i8(const int8_t* input, const int8_t* filters, const abed_layer_shape* shape,
                 int32_t* convout, void* stream);
/* convolution.hpp:245 conv_direct_f32 (f32 operands and accumulation) */
int abed_conv_f32(const float* input, const float* filters, const abed_layer_shape* shape,
                  float* convout, void* stream);
/* convolution.hpp:353-387 epilog: out is int8 or f32 per params->output_kind */
int abed_epilog(const int32_t* convout, abed_dims4 dims, const abed_epilog_params* params,
                void* out, void* stream);

/* ------------------------------------------------------------ L2 ABED schemes */
/* checksum.hpp:75-90 gen_filter_checksum: sums[c,r,s] (i32).  filters dims K x C x R x S */
int abed_gen_filter_checksum(const int8_t* filters, abed_dims4 fdims, int32_t* sums, void* stream);
/* checksum.hpp:108-122 decompose_checksum_filters: planes = 4 x count raw LE bytes */
int abed_decompose_checksum_filters(const int32_t* sums, int64_t count, int8_t* planes, void* stream);
/* checksum.hpp:134-176 conv_checksum_planes: extra = 4 x (N*P*Q) i32 (planes 0-2 unsigned, 3 signed) */
int abed_conv_checksum_planes(const int8_t* input, const abed_layer_shape* shape,
                              const int8_t* planes, int32_t* extra, void* stream);
/* checksum.hpp:179-196 recombine_extra_fmaps: out[i] = e0 + e1<<8 + e2<<16 + e3<<24 (i64) */
int abed_recombine_extra_fmaps(const int32_t* extra, int64_t count, int64_t* out, void* stream);
/* checksum.hpp:201-206 conv_filter_checksum: direct i64 route (input conv i32 sums) */
int abed_conv_filter_checksum(const int8_t* input, const abed_layer_shape* shape,
                              const int32_t* sums, int64_t* out, void* stream);
/* checksum.hpp:211-236 fc_verify (synchronous; outcome in host memory) */
int abed_fc_verify(const int32_t* convout, abed_dims4 dims, const int64_t* extra,
                   int64_t original_k, abed_verify_outcome* outcome);
/* checksum.hpp:248-266 gen_input_checksum: sums[c,r,s] (i32) */
int abed_gen_input_checksum(const int8_t* input, const abed_layer_shape* shape, int32_t* sums,
                            void* stream);
/* checksum.hpp:268-272 reduce_all_i64 (result in host memory) */
int abed_reduce_all_i64(const int32_t* convout, int64_t count, int64_t* result);
/* checksum.hpp:299-303 reduce_all_wrap32 */
int abed_reduce_all_wrap32(const int32_t* convout, int64_t count, int32_t* result);
/* checksum.hpp:275-285 fic_dot */
int abed_fic_dot(const int32_t* fc_sums, const int32_t* ic_sums, int64_t count, int64_t* result);
/* checksum.hpp:287-294 fic_verify / :305-312 fic_verify_forced32 */
int abed_fic_verify(const int32_t* convout, int64_t count, int64_t expected, abed_verify_outcome* outcome);
int abed_fic_verify_forced32(const int32_t* convout, int64_t count, int64_t expected,
                             abed_verify_outcome* outcome);
/* checksum.hpp:319-347 ic_verify_k */
int abed_ic_verify_k(const int32_t* convout, abed_dims4 dims, const int8_t* filters, abed_dims4 fdims,
                     const int32_t* ic_sums, abed_verify_outcome* outcome);
/* checksum.hpp:350-362 ic_batch_checksum: 1 x C x H x W i32 */
int abed_ic_batch_checksum(const int8_t* input, abed_dims4 dims, int32_t* batch, void* stream);
/* checksum.hpp:367-396 conv_batch_checksum: 1 x K x P x Q i64 */
int abed_conv_batch_checksum(const int32_t* batch, const int8_t* filters, const abed_layer_shape* shape,
                             int64_t* out, void* stream);
/* checksum.hpp:398-421 ic_batch_verify */
int abed_ic_batch_verify(const int32_t* convout, abed_dims4 dims, const int64_t* extra,
                         abed_verify_outcome* outcome);
/* checksum.hpp:451-468 plan_precision (host only) */
int abed_plan_precision(const abed_layer_shape* shape, int32_t operand_bits, abed_precision_plan* out);

/* float mode, checksum.hpp:474-595 (f32 tensors, f64 checksum vectors, absolute tau) */
int abed_float_verify(double lhs, double rhs, double tau, abed_verify_outcome* outcome);
int abed_filter_checksum_f64(const float* filters, abed_dims4 fdims, double* sums, void* stream);
int abed_input_checksum_f64(const float* input, const abed_layer_shape* shape, double* sums, void* stream);
int abed_reduce_all_f64(const float* convout, int64_t count, double* result);
int abed_fic_dot_f64(const double* a, const double* b, int64_t count, double* result);
int abed_fic_verify_f32(const float* convout, int64_t count, double expected, double tau,
                        abed_verify_outcome* outcome);
int abed_fc_verify_f32(const float* convout, abed_dims4 dims, const float* extra, double tau,
                       abed_verify_outcome* outcome);
int abed_ic_verify_k_f32(const float* convout, abed_dims4 dims, const float* filters, abed_dims4 fdims,
                         const double* ic_sums, double tau, abed_verify_outcome* outcome);

/* checksum.hpp:605-631 fused_conv_epilog.  out: int8/f32 per params.  Taps:
 * out_checksum (host int64*, NULL = tap off) is the pre-epilog ConvOut sum;
 * next_shape (NULL = tap off) requests the next layer's input checksum into
 * next_ic (device i32, 1 x C' x R' x S'), needs an int8 epilog. */
int abed_fused_conv_epilog(const int8_t* input, const int8_t* filters, const abed_layer_shape* shape,
                           const abed_epilog_params* params, void* out, int64_t* out_checksum,
                           const abed_layer_shape* next_shape, int32_t* next_ic, void* stream);

/* ------------------------------------------------------------ L3 faults */
/* faults.hpp:53-62 flip_bit_inplace on a device tensor of `kind` with `count` elements */
int abed_flip_bit(void* data, int32_t kind, int64_t count, int64_t flat_index, int32_t bit, void* stream);
/* faults.hpp:268-274 run_trial: input/filters DEVICE tensors, bias HOST (may be NULL) */
int abed_run_trial(const abed_layer_shape* shape, const int8_t* input, const int8_t* filters,
                   int32_t scheme, int32_t target, float scale, const float* bias_host,
                   int64_t bias_len, int32_t activation, int32_t output_kind, uint64_t seed,
                   abed_trial_outcome* outcome);
/* faults.hpp:276-333 run_campaign (deterministic; identical for any jobs / GPU count).
 * trial_begin/trial_end select a sub-range of trials (batch sharding across GPUs);
 * pass 0, config->trials for the whole campaign. */
int abed_run_campaign(const abed_campaign_config* config, int64_t trial_begin, int64_t trial_end,
                      abed_campaign_report* report);
/* faults.hpp:276-333 run_campaign, trial-parallel: the same report as
 * abed_run_campaign, every trial of [trial_begin, trial_end) evaluated in ONE
 * launch (one CTA per trial) from the golden int32 ConvOut, the pristine
 * checksums and the ConvOut elements the flip perturbs (exact: the reference's
 * int32 ConvOut wrap, int64 verify sums and epilog).  abed_run_campaign re-runs
 * the fused protected conv per trial instead; both give identical reports. */
int abed_run_campaign_batched(const abed_campaign_config* config, int64_t trial_begin, int64_t trial_end,
                              abed_campaign_report* report);
/* Device-resident form (bench / multi-GPU sharding): create draws the data, the
 * golden ConvOut, the pristine checksums and every trial's flip once; run adds the
 * classification counts of trials [trial_begin, trial_end) into counts_dev[4]
 * (int64, indexed by ABED_DETECTED / _SDC / _MASKED / _DETECTED_BENIGN) as one
 * stream-ordered launch -- counts_dev is what an NCCL all-reduce sums across
 * ranks; report_of folds host counts into an abed_campaign_report. */
typedef struct abed_campaign abed_campaign;
int abed_campaign_create(const abed_campaign_config* config, abed_campaign** campaign);
int abed_campaign_run(abed_campaign* campaign, int64_t trial_begin, int64_t trial_end, int64_t* counts_dev,
                      void* stream);
int abed_campaign_report_of(const abed_campaign* campaign, const int64_t* counts_host, int64_t trials,
                            abed_campaign_report* report);
/* Batch-sharded form (configs[4]: one rank per GPU owns images [image_begin,
 * image_end) of config->shape's batch; trials are drawn over the WHOLE tensors,
 * so every rank sees every trial).  run_records writes per trial
 * {row/channel check failed, output differs, sum delta} of this shard into
 * records_dev[3 * (t - trial_begin) ...]; summing the records of all shards
 * (one NCCL all-reduce) and classify give the single-GPU report exactly
 * (classify ADDS into counts_dev[4]). */
int abed_campaign_create_shard(const abed_campaign_config* config, int64_t image_begin, int64_t image_end,
                               abed_campaign** campaign);
int abed_campaign_run_records(abed_campaign* campaign, int64_t trial_begin, int64_t trial_end, int64_t* records_dev,
                              void* stream);
int abed_campaign_classify(const abed_campaign* campaign, const int64_t* records_dev, int64_t n_records,
                           int64_t* counts_dev, void* stream);
int abed_campaign_destroy(abed_campaign* campaign);

/* ------------------------------------------------------------ protected conv (hot path)
 * A plan holds the packed filters (+ FC checksum-digit rows), the filter checksum
 * and the per-tile verification workspace of one layer.  The activations live in
 * the packed strip-plane layout; abed_pack_input converts a
 * reference NCHW tensor, and a previous layer can write it directly
 * (ABED_OUT_I8_PACKED).  Scheme bits: ABED_CHECK_FC | ABED_CHECK_FIC | ABED_CHECK_IC |
 * ABED_CHECK_ICBATCH.
 * ABED_CHECK_ICBATCH (int8, not with ABED_CHECK_IC) fuses ic_batch_checksum +
 * conv_batch_checksum + ic_batch_verify (checksum.hpp:350-421): the packed input
 * carries the batch-sum image as 2 (N <= 256) or 3 extra balanced base-256 digit
 * images after the N real ones (written inside the conv kernel; the buffer size is
 * abed_plan_info.packed_input_bytes), the tensor-core conv of those rows is the
 * checksum row of the GEMM, and each run ends with a scan comparing the per-(k,p,q)
 * batch sums of the outputs against it; its VerifyOutcome (locus (k, p, q)) is
 * written into outcome slot 2 by finalize. */
enum { ABED_CHECK_FC = 1, ABED_CHECK_FIC = 2, ABED_CHECK_IC = 4, ABED_CHECK_ICBATCH = 8 };
enum {
  ABED_OUT_NONE = 0, ABED_OUT_I32_NCHW = 1, ABED_OUT_I8_NCHW = 2, ABED_OUT_F32_NCHW = 3,
  ABED_OUT_I8_PACKED = 4, ABED_OUT_I8_COMPARE = 5,
  /* float mode (fp16 / bf16 plans): 16-bit output into the next layer's packed
   * planes, or compared against them (duplication baseline) */
  ABED_OUT_H_PACKED = 6, ABED_OUT_H_COMPARE = 7
};
typedef struct abed_conv_plan abed_conv_plan;
typedef struct abed_plan_info {
  int64_t packed_input_bytes;   /* bytes of the packed activation buffer */
  int32_t block_n, n_tiles, m_tiles, gps, b_resident, n_phase, Hl, Wl;
  int64_t smem_bytes;
} abed_plan_info;
int abed_conv_plan_create(const abed_layer_shape* shape, const int8_t* filters, int32_t checks,
                          int32_t force_block_n, abed_conv_plan** plan);
int abed_conv_plan_destroy(abed_conv_plan* plan);
int abed_conv_plan_info(const abed_conv_plan* plan, abed_plan_info* info);
int abed_pack_input(const abed_conv_plan* plan, const int8_t* input_nchw, int8_t* packed, void* stream);
/* Runs the fused kernel (and, with ABED_CHECK_FIC, the input-checksum kernels)
 * asynchronously.  `next` (may be NULL) gives the consumer layer's plan when
 * out_mode == ABED_OUT_I8_PACKED.  fault_key/fault_bit: ConvOut single-bit
 * fault hook (faults.hpp:230-233), fault_key < 0 = none. */
int abed_conv_plan_run(abed_conv_plan* plan, const int8_t* packed_input, const abed_epilog_params* params,
                       int32_t out_mode, void* out, const abed_conv_plan* next, int64_t fault_key,
                       int32_t fault_bit, void* stream);
/* Reduces the last run's per-CTA records into reference VerifyOutcomes (device
 * side, one small launch), asynchronously; outcome_dev points to 3 device
 * abed_verify_outcome {FC, FIC, IC or ICBatch}. */
int abed_conv_plan_finalize(abed_conv_plan* plan, abed_verify_outcome* outcome_dev, void* stream);
/* FIC-AF (fused_conv_epilog's next-layer input-checksum tap, checksum.hpp:605-631):
 * on = 1 marks that this int8 FIC plan's right-hand side is produced by the
 * previous layer's epilogue, i.e. that layer runs with out_mode
 * ABED_OUT_I8_PACKED and next = this plan; its stored int8 outputs are dotted
 * with this plan's position weights as they are written.  The FR input pass is
 * then skipped; finalize consumes (and resets) the accumulated value. */
int abed_conv_plan_set_af_input(abed_conv_plan* plan, int32_t on);
/* One launch that finalizes n plans (e.g. every layer of a network pass):
 * outcomes_dev[3*i .. 3*i+2] receive plan i's {FC, FIC, IC} VerifyOutcomes. */
int abed_conv_plan_finalize_many(abed_conv_plan* const* plans, int32_t n, abed_verify_outcome* outcomes_dev,
                                 void* stream);
/* reuse = 1: later runs keep the input checksum / FIC right-hand side computed by
 * an earlier run instead of recomputing it from the (possibly corrupted) input;
 * the run is then exactly one kernel launch (fault campaigns, kernel timing). */
int abed_conv_plan_set_reuse_input_checksum(abed_conv_plan* plan, int32_t reuse);
/* IC plans: a run's in-kernel sums are consumed (and cleared) by the finalize of
 * that run, so eager run/finalize pairs need no per-run memsets.  A run captured
 * into a CUDA graph clears them itself (the host cannot see how replays and
 * finalizes interleave) unless paired = 1 declares that every captured run is
 * followed by its finalize in the same graph (the PlanSet pass pattern). */
int abed_conv_plan_set_paired_finalize(abed_conv_plan* plan, int32_t paired);
/* Where an int8 FIC plan's in-kernel input checksum (the FIC right-hand side,
 * gen_input_checksum + fic_dot, checksum.hpp:248-285) reads the input from:
 * ABED_RHS_REREAD (default) reads the stored input a second time (the cost
 * model's "FR" option); ABED_RHS_STAGED dots the activation tiles the conv
 * kernel has already staged in shared memory (each M tile owns 128 plane pixels
 * of every strip), so the input is read from HBM once.  Both are exact and
 * bit-identical; see DESIGN.md for the measured trade-off. */
enum { ABED_RHS_STAGED = 0, ABED_RHS_REREAD = 1 };
int abed_conv_plan_set_input_checksum_source(abed_conv_plan* plan, int32_t source);
/* duplication baseline: mismatch count of the last OUT_I8_COMPARE run (synchronous) */
int abed_conv_plan_compare_count(abed_conv_plan* plan, int64_t* count);
/* ---- depthwise conv (MobileNetV2; no reference counterpart).
 * shape.k == shape.c, filters C x 1 x R x S int8 (device).  checks: 0 or
 * ABED_CHECK_FIC (the FIC identity holds by linearity with the depthwise filter
 * as its own filter checksum).  The plan uses the strip-plane layout and the
 * plan API (abed_pack_input, abed_conv_plan_run with ABED_OUT_I8_* modes,
 * next-layer packed output in both directions, finalize). */
int abed_conv_plan_create_dw(const abed_layer_shape* shape, const int8_t* filters, int32_t checks,
                             abed_conv_plan** plan);
/* ---- float mode on tensor cores (fp16 / bf16 operands, f32 accumulation).
 * The reference's float mode (checksum.hpp:471-595: f32 operands, f64 checksum
 * reductions, Pass iff |lhs - rhs| <= tau) on tcgen05 kind::f16: filters (device
 * f32 KCRS) and inputs (device f32 NCHW, via abed_pack_input_h) are rounded to
 * elem_kind (ABED_F16 / ABED_BF16, round to nearest even).  checks: ABED_CHECK_FC
 * and/or ABED_CHECK_FIC with absolute thresholds tau_fc / tau_fic (float_verify;
 * tau < 0 is invalid_argument).  Run with abed_conv_plan_run (ABED_OUT_F32_NCHW,
 * ABED_OUT_H_PACKED, ABED_OUT_H_COMPARE, ABED_OUT_NONE); verdicts carry lhs_f/rhs_f. */
int abed_conv_plan_create_h(const abed_layer_shape* shape, const float* filters, int32_t elem_kind, int32_t checks,
                            double tau_fc, double tau_fic, int32_t force_block_n, abed_conv_plan** plan);
int abed_pack_input_h(const abed_conv_plan* plan, const float* input, void* packed, void* stream);
int abed_conv_plan_set_tau(abed_conv_plan* plan, double tau_fc, double tau_fic);
/* ------------------------------------------------------------ ABFT GEMM comparison
 * Row/column-checksum ABFT for an int8 GEMM (abft_gemm.hpp:98-152), the classical
 * scheme the paper contrasts with ABED, on the tcgen05 GEMM: A (m x k) and B (k x n)
 * row-major int8 device matrices, c (m x n i32, may be NULL), c_aug ((m+1) x (n+1)
 * i64: the augmented product with the checksum row and column, abft_gemm.hpp:139),
 * row / column VerifyOutcomes of abft_check (:70-96; locus (index, -1, -1)).
 * Guards as the reference: inner-dimension mismatch, 16 + ceil_log2(m n k) > 63,
 * 16 + ceil_log2(k) > 31 are invalid_argument (:106-111). */
enum { ABED_ABFT_CHECKED = 0, ABED_ABFT_PLAIN = 1, ABED_ABFT_FUSED_ROW = 2 };
/* abft_gemm (synchronous; outcomes in host memory) */
int abed_abft_gemm_i8(const int8_t* a, int64_t m, int64_t k, const int8_t* b, int64_t kb, int64_t n, int32_t* c,
                      int64_t* c_aug, abed_verify_outcome* row_check, abed_verify_outcome* col_check);
/* abft_check (:70-96) on a device (rows x cols) i64 c_aug; rows, cols >= 2 */
int abed_abft_check(const int64_t* c_aug, int64_t rows, int64_t cols, abed_verify_outcome* row_check,
                    abed_verify_outcome* col_check);
/* Plan form for timing (allocation-free, stream-ordered runs).  mode:
 * ABED_ABFT_CHECKED = abft_gemm's online tasks (2)-(6) (outcomes_dev[2] = {row, col});
 * ABED_ABFT_PLAIN = the same GEMM pipeline without checksums (unprotected baseline);
 * ABED_ABFT_FUSED_ROW = ABED-style: the row check as a filter-checksum column
 * verified inside the GEMM epilogue (outcomes_dev[0]; [1] is a pass).
 * b == NULL reuses B (and its checksum column) packed by an earlier run in the
 * same mode: the weights-offline setting. */
typedef struct abed_abft_plan abed_abft_plan;
int abed_abft_plan_create(int64_t m, int64_t n, int64_t k, abed_abft_plan** plan);
int abed_abft_plan_destroy(abed_abft_plan* plan);
int abed_abft_plan_run(abed_abft_plan* plan, const int8_t* a, const int8_t* b, int32_t* c, int64_t* c_aug,
                       abed_verify_outcome* outcomes_dev, int32_t mode, void* stream);

/* ------------------------------------------------------------ multi-GPU verdicts
 * The batch is sharded across ranks; each rank verifies its shard
 * and the per-shard VerifyOutcomes are folded into the global ones with one small
 * collective: abed_verdict_records writes 8 int64 per outcome slot
 * {status, has_locus, locus[3], lhs, rhs, error_count} (FC locus n made global by
 * n_offset, the rank's first image), the ranks' records are all-gathered
 * (world x n x 64 bytes; rank order = batch order), and abed_verdict_combine folds
 * them.  kinds[i] = scheme of slot i (ABED_FC, ABED_IC, ABED_ICBATCH, ABED_FIC):
 *   FC: counts add, first mismatch of the lowest failing rank (reference (n,p,q) order)
 *   FIC: lhs and rhs add (both linear in the batch), status = lhs != rhs
 *   IC / ICBATCH: per-shard checks: status = any, counts add, lowest failing rank's locus
 * n <= 256.  Device versions are stream-ordered; the _host versions run the same
 * fold on host memory (no device needed). */
int abed_verdict_records(const abed_verify_outcome* outcomes_dev, int32_t n, const int32_t* kinds_host,
                         int64_t n_offset, int64_t* records_dev, void* stream);
int abed_verdict_combine(const int64_t* gathered_dev, int32_t world, int32_t n, const int32_t* kinds_host,
                         abed_verify_outcome* out_dev, void* stream);
int abed_verdict_records_host(const abed_verify_outcome* outcomes, int32_t n, const int32_t* kinds,
                              int64_t n_offset, int64_t* records);
int abed_verdict_combine_host(const int64_t* gathered, int32_t world, int32_t n, const int32_t* kinds,
                              abed_verify_outcome* out);

/* diagnostics (no reference counterpart): record a per-CTA clock timeline of the
 * conv kernel into trace_dev (16 int64 per CTA, caller-zeroed); NULL disables.
 * flags bit 0 makes the epilogue skip its work (timing experiments only). */
int abed_debug_set_conv_trace(abed_conv_plan* plan, int64_t* trace_dev, int32_t flags);
/* measured tcgen05 kind::i8 dense peak of this device (the int8 roofline
 * denominator): one CTA per SM issuing `iters` x 8 back-to-back M128 N256 K32
 * MMAs, timed with CUDA events (synchronous).  tops = 2 * MACs / time. */
int abed_probe_mma_i8_peak(int32_t iters, double* tops, double* ms);

#ifdef __cplusplus
}
#endif
#endif /* ABED_B200_H */
