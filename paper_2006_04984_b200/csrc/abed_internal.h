// Internal declarations shared by the .cu translation units of libabed_b200.so.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/abed_b200.h"
#include "conv_tc.cuh"

namespace abed_host {

// exceptions carrying the reference's exception class as a status code
struct AbedError : std::runtime_error {
  int code;
  AbedError(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};
[[noreturn]] inline void throw_invalid(const std::string& m) { throw AbedError(ABED_ERR_INVALID_ARGUMENT, m); }
[[noreturn]] inline void throw_range(const std::string& m) { throw AbedError(ABED_ERR_OUT_OF_RANGE, m); }
inline void cuda_check(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw AbedError(ABED_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

int set_error(int code, const std::string& msg);
// runs fn, mapping exceptions to the C-ABI status codes (+ abed_last_error)
template <typename Fn>
int guarded(Fn&& fn) {
  try {
    fn();
    return ABED_OK;
  } catch (const AbedError& e) {
    return set_error(e.code, e.what());
  } catch (const std::exception& e) {
    return set_error(ABED_ERR_RUNTIME, e.what());
  }
}

// plan.cu
// cpg: channels per 16-byte pixel group (16 for int8, 8 for fp16/bf16)
// n_extra: ICBatch digit images appended after the n images (M-space and planes only)
abed_dev::ActGeom make_geom(const abed_layer_shape& s, int cpg = 16, int n_extra = 0);
int geom_strip_pix(const abed_dev::ActGeom& g);
int64_t geom_packed_bytes(const abed_dev::ActGeom& g);
bool choose_tiling(const abed_dev::ActGeom& g, bool fc, int force_block_n, abed_dev::ConvTcParams& p,
                   uint32_t reserve = 0);
int num_sms();

__global__ void pack_input_kernel(const int8_t* x, abed_dev::ActGeom g, int8_t* out);
// NCHW -> strip planes (vectorised 4-pixel quads; plan.cu)
void launch_pack_input(const int8_t* x, const abed_dev::ActGeom& g, int8_t* packed, cudaStream_t st);
__global__ void pack_filters_kernel(const int8_t* f, abed_dev::ActGeom g, int block_n, int block_n_tot,
                                    int n_tiles, int gps, int k_stages, int fc, int8_t* out);
__global__ void batch_sum_packed_kernel(const int8_t* act, abed_dev::ActGeom g, int32_t* bsum);
__global__ void box_sum_dot_kernel(const int32_t* bsum, abed_dev::ActGeom g, const int32_t* fsum,
                                   int32_t* ic_out, unsigned long long* fic_rhs);
__global__ void fic_weight_kernel(const int32_t* fsum, abed_dev::ActGeom g, int32_t* G);
__global__ void fic_weight_digits_kernel(const int32_t* G, int64_t cells, int8_t* G8, int* too_big);
__global__ void fic_class_table_kernel(const int8_t* G8, abed_dev::ActGeom g, const int* rep, int n_rep, int8_t* T8);
__global__ void fic_rhs_dp4a_kernel(const int8_t* act, abed_dev::ActGeom g, const int8_t* G8, int nsplit,
                                    unsigned long long* rhs);
__global__ void fic_rhs_kernel(const int8_t* act, abed_dev::ActGeom g, const int32_t* G, int nsplit,
                               unsigned long long* rhs);
__global__ void fc_finalize_rec_kernel(const int64_t* rec, int m_tiles, int P, int Q, abed_verify_outcome* out);
__global__ void fc_finalize_part_kernel(const int64_t* part, abed_dev::ActGeom g, int n_tiles,
                                        unsigned long long* scratch);
__global__ void fc_finalize_part2_kernel(const int64_t* part, abed_dev::ActGeom g, int n_tiles,
                                         const unsigned long long* scratch, abed_verify_outcome* out);
__global__ void fic_finalize_kernel(const int64_t* part, int n, const unsigned long long* rhs_p,
                                    abed_verify_outcome* out);
// IC verdicts of many plans (two launches): ic from the class sums (S == nullptr:
// computed ahead), FIC rhs when fic_rhs != nullptr, then ic_verify_k
struct IcVerdictJob {
  int copy_only;                  // finalize again without a run: repeat the stored outcome
  abed_verify_outcome* last;      // plan-owned copy of the last outcome
  int64_t S_len;                  // class sums to zero after use (S != nullptr)
  const int64_t* S;
  const uint64_t* rowmask;
  const uint64_t* colmask;
  int nrc, ncc, R, Sd, sh, sw, nph_w, c256;
  const int32_t* fsum;
  int32_t* ic;
  unsigned long long* fic_rhs;
  unsigned long long* ksum;        // consumed and zeroed
  const int8_t* f;
  int64_t K, crs;
  unsigned long long* scr;
  abed_verify_outcome* out;
};
constexpr int kMaxIcJobs = 64;
struct IcVerdictBatch {
  IcVerdictJob job[kMaxIcJobs];
};
void ic_verdict_many_launch(const IcVerdictJob* jobs, int n, cudaStream_t st);

// conv_tc.cu
uint32_t conv_tc_smem_bytes(const abed_dev::ConvTcParams& p);
int conv_tc_grid(const abed_dev::ConvTcParams& p, int num_sms);
int mma_pattern_of(const abed_dev::ActGeom& g, int gps);
// pdl: launch with programmatic stream serialization (griddepcontrol in the kernel)
cudaError_t conv_tc_launch(const abed_dev::ConvTcParams& p, int num_sms, bool pdl, cudaStream_t stream);
// ICBatch: compare and reset after a fused run (p.icb_ready = {writer counter, ticket})
cudaError_t icb_scan_launch(const abed_dev::IcbScanJob* jobs, int n, cudaStream_t stream);
// reduces the per-CTA verdict records of n plans (one block each)
cudaError_t verdict_launch(const abed_dev::VerdictJob* jobs, int n, cudaStream_t stream);

}  // namespace abed_host

struct abed_conv_plan;
namespace abed_host {
// abi_core.cu
int set_error(int code, const std::string& msg);
void require_device();
int grid_for(int64_t n, int threads);
void validate_shape(const abed_layer_shape& s);
void build_fic_classes(abed_conv_plan* pl);
uint32_t fic_classes_host(abed_conv_plan* pl);
abed_conv_plan* plan_create(const abed_layer_shape& shape, const int8_t* filters, int checks, int force_bn);
// dwconv.cu: depthwise plan (shares abed_conv_plan; dispatched by plan_run)
abed_conv_plan* plan_create_dw(const abed_layer_shape& shape, const int8_t* filters, int checks);
void plan_run_dw(abed_conv_plan* pl, const int8_t* packed, const abed_epilog_params* ep, int out_mode, void* out,
                 const abed_conv_plan* next, int64_t fault_key, int fault_bit, cudaStream_t st);
int dw_grid();
// abi_f16.cu: float-mode plan (fp16 / bf16 operands from f32 filters)
abed_conv_plan* plan_create_h(const abed_layer_shape& shape, const float* filters, int elem_kind, int checks,
                              double tau_fc, double tau_fic, int force_bn);
// geometry, tiling and the verdict buffers shared by the int8 and float-mode plans
void plan_init_common(abed_conv_plan* pl, const abed_layer_shape& shape, int checks, int force_bn, int cpg);
void plan_run(abed_conv_plan* pl, const int8_t* packed, const abed_epilog_params* ep, int out_mode, void* out,
              const abed_conv_plan* next, int64_t fault_key, int fault_bit, cudaStream_t st);
void plan_finalize(abed_conv_plan* pl, abed_verify_outcome* out_dev, cudaStream_t st);
// one reference-style conv call on a plan cached per (device, shape, checks)
void one_shot_run(const abed_layer_shape& shape, int checks, const int8_t* input, const int8_t* filters,
                  const abed_epilog_params* ep, int out_mode, void* out, abed_verify_outcome* outcomes_dev,
                  cudaStream_t st);
abed_dev::VerdictJob plan_verdict_job(const abed_conv_plan* pl, abed_verify_outcome* out_dev);
// ref_kernels.cu
void dev_gen_input_checksum(const int8_t* x, const abed_layer_shape& s, int32_t* sums, cudaStream_t st);
// column sums of a rows x len int8 matrix (filter checksum, batch checksum image)
void dev_colsum_i8(const int8_t* x, int64_t rows, int64_t len, int32_t* out, cudaStream_t st);
void dev_epilog(const int32_t* in, abed_dims4 d, const abed_epilog_params* p, void* out, cudaStream_t st);
}  // namespace abed_host

// opaque plan (C ABI handle)
struct abed_conv_plan {
  abed_layer_shape shape;
  abed_dev::ActGeom g;
  abed_dev::ConvTcParams base{};  // tiling + tap tables; pointers filled per run
  int checks;
  int8_t* d_wpk = nullptr;      // packed B blocks
  int8_t* d_filters = nullptr;  // KCRS copy (IC verify reads filter storage)
  int32_t* d_fsum = nullptr;    // filter checksum (c,r,s) order, i32
  int32_t* d_ic = nullptr;      // input checksum of the last run (c,r,s)
  int32_t* d_bsum = nullptr;    // batch-sum image [phase][c16*16][Hl*Wl]
  int32_t* d_ficw = nullptr;    // FIC position weights G [phase][c16][Hl*Wl][16] (offline)
  int8_t* d_ficw8 = nullptr;    // G as 3 balanced base-256 digit planes [phase][c16][Hl*Wl][3][16]
  int ficw8_ok = 0;             // every |G| < 2^23 (3 digits are exact)
  int ficw8_ndig = 3;           // digit planes the FR pass needs (2 when every third digit is 0)
  int8_t* d_ficc8 = nullptr;    // G class table [phase][nrc][ncc][c16][3][16] (FIC-SM)
  uint8_t* d_rowcls = nullptr;  // [nph_h][Hl] / [nph_w][Wl] row / column classes
  uint8_t* d_colcls = nullptr;
  int nrc = 0, ncc = 0;
  std::vector<uint8_t> h_rowcls, h_colcls;  // host copies (FIC-SM)
  std::vector<int> h_rep;                    // representative plane pixel per class pair
  // FIC input checksum source: ABED_RHS_REREAD (default; the input-checksum warps
  // read the stored input a second time, "FR") or ABED_RHS_STAGED (they dot the
  // A stages already in shared memory).  Measured on B200 at batch 32 / 256 / 1024
  // the staged source is slower (its 4 shared-memory loads per 16-byte chunk
  // compete with the SS-mode MMA operand reads and it holds stages), so FR is default.
  int rhs_src = ABED_RHS_REREAD;
  int64_t* d_fc_part = nullptr;     // FC row partials per N tile (n_tiles > 1)
  unsigned int* d_tile_sem = nullptr;  // FC per-M-tile flags (several N tiles), epoch-tagged
  int64_t* d_cta_rec = nullptr;     // FC per-CTA records
  unsigned long long* d_kacc = nullptr;  // kernel accumulators {FIC lhs, FIC rhs, done ticket, -}
  abed_verify_outcome* d_outcome = nullptr;  // {FC, FIC, IC} verdicts written by the conv kernel
  unsigned long long* d_acc = nullptr;  // [0]=fic rhs, [1]=cmp count, [2..3]=fc scratch, [4..4+K) ic sums
  unsigned long long* d_ic_scr = nullptr;  // IC verdict scratch {count, first k, ticket, -, dot[K]}
  // IC input checksum in-kernel: class sums [n_phase][nrc][ncc][c16*16] (int64),
  // row / column classes [nph_h][Hl] / [nph_w][Wl], filter-row / -column masks per class
  int64_t* d_ic_S = nullptr;
  uint8_t* d_ic_cls = nullptr;
  uint64_t* d_ic_mask = nullptr;
  int ic_nrc = 0, ic_ncc = 0;
  size_t ic_S_bytes = 0;
  float* d_zero_bias = nullptr;
  // when set, runs skip the input-checksum kernels and keep d_ic / the FIC
  // right-hand side of an earlier run (fault campaigns: checksums come from
  // the pristine input, faults.hpp:111-115)
  int reuse_input_checksum = 0;
  int last_rhs_mode = 0;
  int ic_pending = 0;                      // IC: a run's in-kernel sums await their verdict
  int icb_pending = 0;                     // ICBatch: a run's batch sums await their scan
  int paired_finalize = 0;                 // IC: captured graphs finalize every run they contain
  abed_verify_outcome* d_ic_last = nullptr;  // IC: last verdict (repeated by a second finalize)
  unsigned long long cmp_seen = 0;         // compare runs: mismatches already reported
  int last_grid = 0;            // CTAs of the last conv launch (records the verdict reduces)        // rhs_mode of the last run (its verdict reduction needs it)
  // FIC-AF: this layer's FIC rhs is accumulated by the previous layer's epilogue
  // (which is run with next = this plan); the verdict consumes and resets it
  int af_input = 0;
  unsigned long long* d_af_acc = nullptr;
  // ICBatch fused (CHECK_ICB): batch sums of the outputs [K*P*Q], conv of the
  // digit images [n_extra][K*P*Q], {writer counter, scan ticket}, scan records,
  // the last run's outcome (copied into slot 2 by finalize)
  unsigned long long* d_icb_lhs = nullptr;
  int32_t* d_icb_dig = nullptr;
  unsigned int* d_icb_ctl = nullptr;
  int64_t* d_icb_rec = nullptr;
  abed_verify_outcome* d_icb_out = nullptr;
  // float mode (fp16 / bf16 operands, f32 accumulators; abi_f16.cu)
  int dtype = 0;                 // abed_dev::DT_I8 / DT_F16 / DT_BF16
  double tau_fc = 0.0, tau_fic = 0.0;
  double* d_facc = nullptr;      // {FIC lhs, FIC rhs} f64 kernel accumulators
  double* d_rhs_f = nullptr;     // FIC rhs of the pristine input (f64)
  float* d_ficwf = nullptr;      // G as f32 [phase][c16][Hl*Wl][8]
  double* d_fsum_f = nullptr;    // filter checksum (c,r,s) of the rounded filters, f64
  // depthwise plan (dwconv.cu): one filter per channel, CUDA-core kernel, FIC only
  int dw = 0;
  uint32_t* d_dwf = nullptr;     // packed depthwise filters [c16][16][quads]
  // programmatic dependent launch of the conv kernel (its prologue overlaps the
  // previous kernel); off for fault campaigns, which patch filter storage
  // right before a run
  int pdl = 1;
};
