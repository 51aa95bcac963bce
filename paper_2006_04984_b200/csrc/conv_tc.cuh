// Shared host/device definitions for the tcgen05 implicit-GEMM convolution.
//
// Packed activation layout ("strip planes").  The reference keeps NCHW int8
// (tensor.hpp:68-70).  On the device an activation tensor consumed by a conv
// is stored as planes of 16-byte pixels:
//
//   plane (phase, g) : pixel t in [0, plane_len)  ->  16 channels g*16..g*16+15
//   address          : act + ((phase * c16 + g) * plane_len + t) * 16
//
// Pixel t = (n * Hl + i) * Wl + j is sub-row i / sub-column j of image n in the
// stride phase (a, b); it holds input pixel (h, w) = (i*sh + a - pad_h,
// j*sw + b - pad_w), or zero outside the image.  For a stride-1 conv there is
// one phase and Hl = H + pad_h, Wl = W + pad_w: the zero halo between two rows
// (images) is shared, so every filter tap (r, s) is a constant pixel shift
// r*Wl + s of the whole GEMM row range.  This is what lets one contiguous strip
// of 128 + max_shift pixels per plane feed all R*S taps of a 128-row M tile
// straight from shared memory (SWIZZLE_NONE K-major UMMA operand: rows 16 B
// apart, so a tap is a descriptor start-address offset).
//
// GEMM view: M = output pixels in this "M-space" (m = (n*Hl + p)*Wl + q, valid
// iff p < P and q < Q), N = output channels, K = taps x channels.
#pragma once
#include <cstdint>

namespace abed_dev {

constexpr int kMaxTaps = 64;
constexpr int kBlockM = 128;
constexpr int kStages = 4;       // activation/filter stage ring depth
constexpr int kStages_host = kStages;
// conv kernel CTA size: producer + MMA warps, 8 epilogue warps, 2 input-checksum
// warps (conv_tc_kernel.cuh kConvThreads)
constexpr int kConvThreads_host = 64 + 8 * 32 + 2 * 32;
// dynamic smem cap for the conv kernel: 227 KB minus its static smem (bias, reductions)
constexpr int kConvDynSmemMax = 232448 - 12288;

enum DType : int { DT_I8 = 0, DT_F16 = 1, DT_BF16 = 2 };

enum OutMode : int {
  OUT_NONE = 0,        // checks only (no activation written)
  OUT_I32_NCHW = 1,    // raw ConvOut, reference layout N x K x P x Q
  OUT_I8_NCHW = 2,     // epilog -> int8, reference layout
  OUT_F32_NCHW = 3,    // epilog -> f32, reference layout
  OUT_I8_PACKED = 4,   // epilog -> int8 straight into the next layer's strip planes
  OUT_I8_COMPARE = 5,  // epilog -> int8 compared against `out` (duplication check)
  OUT_H_PACKED = 6,    // float mode: epilog -> fp16/bf16 into the next layer's strip planes
  OUT_H_COMPARE = 7,   // float mode: epilog -> fp16/bf16 compared against `out`
};

enum CheckBits : int {
  CHECK_FC = 1,   // filter checksum columns ride in B (checksum.hpp:211 fc_verify)
  CHECK_FIC = 2,  // full-output int64 sum per tile (checksum.hpp:287 fic_verify)
  CHECK_IC = 4,   // per-output-channel int64 sums (checksum.hpp:319 ic_verify_k)
  CHECK_ICB = 8,  // ICBatch: the batch-sum image rides as extra A images (checksum.hpp:350-421)
};

// Geometry of one conv layer in packed form (computed on the host).
struct ActGeom {
  int n, c, h, w;          // logical input (reference LayerShape n,c,h,w)
  int k, r, s;             // filters
  int sh, sw, ph, pw;      // stride / pad
  int p, q;                // output extents
  int nph_h, nph_w;        // stride phases actually touched by taps
  int n_phase;             // nph_h * nph_w
  int c16;                 // 16-byte channel groups (even, zero padded)
  int cpg;                 // channels per 16-byte group: 16 (int8) or 8 (fp16/bf16)
  int Hl, Wl;              // M-space rows per image / pixels per row
  int max_shift;           // largest tap pixel shift
  int m_tiles;             // ceil(m_total / 128)
  int n_extra;             // ICBatch: balanced base-256 digit images of the batch sum after the n images
  int64_t m_total;         // (n + n_extra) * Hl * Wl
  int64_t plane_len;       // pixels per plane (covers the last strip)
};

struct ConvTcParams {
  // ---- A operand
  const int8_t* act;
  int64_t plane_len;
  int n_phase, c16, gps, k_stages, strip_pix, ntaps;
  int R, S, sh, sw, nph_w;  // filter taps, strides, stride phases per row
  int mma_pattern;          // compile-time unrolled MMA issue routine (conv_tc.cu), 0 = generic
  int n_stages;  // depth of the smem stage ring actually used (<= kStages)
  int tap_phase[kMaxTaps];
  int tap_shift[kMaxTaps];
  // A-operand start offset of each tap inside a stage, in 16-byte units:
  // (tap_phase * gps * strip_pix + tap_shift) -- read with a uniform index by
  // the MMA issuer, so descriptors stay in uniform registers
  uint32_t tap_a16[kMaxTaps];
  // ---- B operand (packed filters, see pack_filters in conv_tc.cu)
  const int8_t* wpk;
  int block_n;       // output channels per N tile
  int block_n_tot;   // + 16 checksum rows when CHECK_FC
  int n_tiles;
  int b_resident;    // 1: a CTA keeps its N tile's whole B in smem
  uint32_t b_stage_bytes;
  // ---- geometry
  int64_t m_total;
  int m_tiles, Hl, Wl, P, Q, N, K;
  // ---- epilogue
  int out_mode;
  void* out;
  const float* bias;  // K entries (device)
  float scale;
  int relu;
  // next-layer packed output geometry (OUT_I8_PACKED)
  int64_t o_plane_len;
  int o_Hl, o_Wl, o_ph, o_pw, o_sh, o_sw, o_nph_w, o_c16;
  // ---- checks (all verdicts are produced inside the kernel: the last CTA to
  // finish reduces the per-CTA records and writes the reference VerifyOutcomes)
  int check;
  int64_t* fc_part;            // [n_tiles][m_tiles*128][2] {sum_k, extra} row partials (n_tiles > 1)
  unsigned int* tile_sem;      // FC, several N tiles: int8 [n_tiles][m_tiles][4] flags (a row failed its tile check); float [m_tiles] counters
  int64_t* cta_rec;            // [gridDim][kCtaRec] per-CTA {FC count, first key, lhs, rhs, FIC lhs, FIC rhs}
  unsigned long long* kacc;    // [0] FIC lhs, [1] FIC rhs (in-kernel), [2] CTA done ticket
  unsigned long long* rhs_ext;  // FIC rhs of the pristine input: read (rhs_mode 0) or stored (rhs_mode 1)
  int rhs_mode;                // 1: input-checksum warps compute the FIC rhs in this kernel (FR re-read),
                               // 2: AF -- the previous layer's epilogue produced it (af accumulator),
                               // 3: SM -- input-checksum warps read the staged A tiles (no re-read),
                               // 4: IC -- they accumulate the class sums of the input checksum
                               //    (ic_S; FIC's rhs then comes from ic at the verdict)
  int rhs_nsplit;              // image split of the rhs work items
  int rhs_deep;                // int8 FR: 16 image loads in flight per item (large inputs) instead of 8
  int g_ndig;                  // int8 FR: G digit planes dotted (2 when every third digit is zero, else 3)
  int conv_grid;               // CTAs running conv work units (blockIdx < conv_grid)
  int ic_ctas;                 // extra CTAs (blockIdx >= conv_grid) that only compute the FR
                               // input checksum on SMs the conv grid leaves idle (0: the conv
                               // CTAs' input-checksum warps do it)
  const int8_t* ficw8;         // FIC weight map G as balanced base-256 digits
                               // [phase][c16][Hl*Wl][3 digits][16 channels] (|G| < 2^23)
  // rhs_mode 3 (FIC-SM): the input-checksum warps take x from the A stages the
  // producer already staged (each M tile owns plane pixels [m0, m0 + 128) of
  // every strip) and G from a class table: G depends on a pixel only through
  // which filter rows / columns reach it, so G[phase][i][j] =
  // ficc8[phase][rowcls[a][i]][colcls[b][j]] -- a few KB instead of a map
  const int8_t* ficc8;         // [c16][3 digits][phase][nrc][ncc][16 channels]
  const uint8_t* rowcls;       // [nph_h][Hl] row class per phase row
  const uint8_t* colcls;       // [nph_w][Wl] column class per phase column
  int nrc, ncc;
  uint32_t fic_smem;           // bytes of the kernel's smem copy of {ficc8, rowcls, colcls} (0: none)
  uint32_t fic_tab_bytes;      // ficc8 part of it
  uint32_t ic_smem;            // IC: bytes of the CTA's per-channel output-sum accumulators (K int64; 0: off)
  void* outcome;               // abed_verify_outcome[3] {FC, FIC, IC}: FC and FIC written here
  // FIC-AF (fused_conv_epilog's next-layer input checksum tap, checksum.hpp:605-631,
  // cost_model "AF"): the epilogue accumulates the NEXT layer's FIC rhs
  // sum y * G_next from the int8 values it stores; nullptr = off
  const int8_t* af_ficw8;      // next layer's G digit planes [phase][c16][Hl*Wl][3][16]
  unsigned long long* af_acc;  // next layer's AF rhs accumulator (reset by its verdict)
  int64_t af_HlWl;             // next layer's pixels per image plane
  unsigned long long* ic_sum;  // [K] per-channel output sums (atomic, integer => deterministic)
  unsigned long long* cmp_count;  // OUT_I8_COMPARE mismatch count
  // ICBatch (ic_batch_checksum + conv_batch_checksum + ic_batch_verify,
  // checksum.hpp:350-421) fused: the packed input carries icb_d extra images
  // after the N real ones -- the balanced base-256 digit planes of the batch-sum
  // image sum_n x[n] -- written inside this kernel by the input-checksum warps
  // (and input-checksum CTAs); the producer loads an A strip that reaches them
  // only after every writer warp has signalled icb_ready.  The epilogue adds each
  // real output into icb_lhs[k][p][q] (int64 reduction) and stores the digit
  // rows' conv into icb_dig[j][k][p][q]; icb_scan_kernel compares afterwards.
  // IC input checksum in-kernel (rhs_mode 4): the FR pass adds each plane pixel's
  // batch sum into ic_S[phase][row class][column class][channel]; the verdict
  // turns the class sums into gen_input_checksum's ic[c,r,s] (checksum.hpp:248-266)
  int64_t* ic_S;
  const uint8_t* ic_rowcls;         // [nph_h][Hl] row class
  const uint8_t* ic_colcls;         // [nph_w][Wl] column class
  int ic_nrc, ic_ncc;
  int icb_d;                        // digit images (0 = ICBatch off)
  int64_t m_real;                   // N * Hl * Wl: GEMM rows of the real images
  unsigned long long* icb_lhs;      // [K*P*Q] sum_n ConvOut (reset by the scan)
  int32_t* icb_dig;                 // [icb_d][K*P*Q] conv of digit image j
  unsigned int* icb_ready;          // writer warps done (reset by the scan)
  unsigned int icb_writers;         // writer warps in this launch
  // ---- fault hook (ConvOut target): flip `fault_bit` of output element
  // (n,k,p,q) = fault_key in reference flat order before checks and epilog.
  int64_t fault_key;  // -1 = none
  int fault_bit;
  // ---- diagnostics: per-CTA clock timeline (kTraceSlots int64 per CTA) or nullptr
  // ---- float mode: fp16 / bf16 operands, f32 accumulators, f64 reductions and
  // absolute thresholds (checksum.hpp:474-595 float_verify semantics)
  int dtype;                   // 0 int8, 1 fp16, 2 bf16
  double tau_fc, tau_fic;
  double* facc;                // [0] FIC lhs, [1] FIC rhs (in-kernel)
  double* rhs_ext_f;           // FIC rhs of the pristine input (read: rhs_mode 0, stored: rhs_mode 1)
  const float* ficwf;          // G as f32 [phase][c16][Hl*Wl][8]
  int64_t* trace;
  int dbg;  // diagnostics: bit 0 = epilogue skips its work, bit 3 = no accumulator handshake
};
// trace slots: 0 globaltimer at entry, 1 clock at entry, 2 setup done, 3 first
// stage ready (MMA warp), 4 last MMA commit, 5 epilogue done, 6 units, 7 producer
// done, 8 first copy issued, 9 summed MMA-warp wait cycles on `full`, 10 summed
// epilogue-warp wait cycles on the accumulator; globaltimer stamps: 16 producer past
// griddepcontrol.wait, 17 first stage full (MMA warp), 18 last MMA commit, 19 epilogue done
constexpr int kTraceSlots = 24;
constexpr int kCtaRec = 6;  // int64 slots per CTA in ConvTcParams::cta_rec

// one plan's verdict reduction (verdict_kernel, conv_tc.cu)
struct VerdictJob {
  const int64_t* rec;  // [grid][kCtaRec] records of the last run
  int grid, P, Q, dtype, checks, rhs_mode;
  // FC with several N tiles: per-tile row partials [n_tiles][m_tiles*128][2] and
  // the per-M-tile flags the conv CTAs raise (consumed and reset here)
  const int64_t* fc_part;
  unsigned* tile_flag;
  int n_tiles, m_tiles, Hl, Wl;
  int64_t m_total;
  double tau_fc;
  unsigned long long* rhs_ext;
  unsigned long long* af_acc;  // rhs_mode 2: read, then reset for the next pass
  double* rhs_ext_f;
  double tau_fic;
  void* out;           // abed_verify_outcome[3] {FC, FIC, IC}
  const void* icb;     // ICBatch outcome of the last run (copied into out[2]) or nullptr
};
constexpr int kMaxVerdictJobs = 32;
// ICBatch verdict (icb_scan_kernel): per-block records {count, first key, lhs, rhs}
constexpr int kIcbScanBlocks = 296;
// one ICBatch plan's scan inputs; a pass scans every ICBatch plan in one launch
// (blockIdx.y = job) at its finalize
struct IcbScanJob {
  unsigned long long* lhs;  // [K][P][Q] batch sums of the outputs (consumed: zeroed by the scan)
  const int32_t* dig;       // [D][K][P][Q] conv of the batch-sum digit images
  int D, Q;
  int64_t kpq, PQ;
  int64_t* rec;             // [kIcbScanBlocks][4] per-block records
  unsigned int* ctl;        // {icb_ready, ticket}: reset by the last block
  void* out;                // abed_verify_outcome of the run
};
constexpr int kMaxIcbScanJobs = 32;
struct IcbScanBatch {
  IcbScanJob job[kMaxIcbScanJobs];
};
struct VerdictBatch {
  int n;
  VerdictJob job[kMaxVerdictJobs];
};

}  // namespace abed_dev
