// Device-side model state and the fused row kernels of the FADE predictor.
//
// Data layout in HBM (fp32, row-major, one row per stream b):
//   activations [B][ld] with ld = logical width (all widths are multiples of 4,
//   ModelConfig.device_check), except the FNR expansion whose width E is padded
//   to Ep = roundup(E, 64): the two expansion weights w_e1 / w_e2 are stored as
//   ONE interleaved matrix W12[H][2*Ep] whose 128-column block j holds
//   [w_e1[:, 64j:64j+64] | w_e2[:, 64j:64j+64]], so a 128-wide GEMM tile carries
//   matching a1/a2 columns and the GeGLU runs in the GEMM epilogue.
//   Padded columns are zero and stay zero (zero gradient => zero Adam step).
#pragma once
#include "common.cuh"
#include "gemm.cuh"

namespace fade {

// Ablation variants (model.py:39, 121-175) in the reference's VARIANTS order.
enum Variant { V_FULL = 0, V_DUAL, V_GLOBAL_ONLY, V_LOCAL_ONLY, V_MIXER_NOGATE, V_MIXER, V_COUNT };
struct VFlags {
  bool global;   // global stream + cache roll
  bool local;    // local conv stream
  bool router;   // sigmoid router mixing the two
  bool mixer;    // HGR coarse refiner (LN, W_down, per-stream W_U, W_up, skip)
  bool gate;     // the refiner's sigmoid gate (W_cgate)
  bool fnr;      // FNR expansion (W_e1/W_e2, W_f, output LN, skip)
};
__host__ __device__ inline VFlags vflags(int v) {
  VFlags f;
  f.global = v != V_LOCAL_ONLY;
  f.local = v != V_GLOBAL_ONLY;
  f.router = v != V_GLOBAL_ONLY && v != V_LOCAL_ONLY;
  f.mixer = v == V_FULL || v == V_MIXER || v == V_MIXER_NOGATE;
  f.gate = v == V_FULL || v == V_MIXER;
  f.fnr = v == V_FULL;
  return f;
}

struct Dims {
  int B, T, D, H, C, X, E, Ep, K;  // streams, ctx, embed, hidden, cache, mix, expand, padded, conv
};

// reference parameter order (model.py:76-105)
enum ParamId {
  P_EMB = 0, P_IN_LN_G, P_IN_LN_B, P_W_GATE, P_W_VAL, P_W_MEM, P_LAM_MEM, P_LOC_LN_G,
  P_LOC_LN_B, P_CONV_K, P_CONV_B, P_W_ROUTE, P_MIX_LN_G, P_MIX_LN_B, P_W_DOWN, P_W_MIX,
  P_W_UP, P_W_CGATE, P_LAM_MIX, P_REF_LN_G, P_REF_LN_B, P_W_E1, P_W_E2, P_W_F, P_OUT_LN_G,
  P_OUT_LN_B, P_LAM_OUT, P_W_HEAD, P_B_HEAD, P_COUNT
};

// Small parameters live contiguously in one arena in the order of the per-row
// reduction buffer ("rowred"), so one column-sum kernel produces their
// gradients and applies Adam in place.  Offsets (in floats) into that arena:
struct SmallLayout {
  int out_g, out_b, ref_g, ref_b, mix_g, mix_b, in_g, in_b;  // H each
  int loc_g, loc_b, conv_b;                                  // D each
  int conv_k;                                                // K*D*D
  int w_gate, w_val;                                         // D*D each
  int lam_out, lam_mix, lam_mem;                             // 1 each
  int rowred;                                                // width of the rowred buffer
  int trunk0, trunk1;   // [in_g, lam_out): the columns trunk_bwd sums per CTA (trunk_part)
  int b_head;                                                // 256, reduced from dlogits
  int total;
};

struct Tensor4 {     // parameter, Adam m, Adam v, gradient (test hook)
  float *p, *m, *v, *g;
};

struct StepState {   // device-resident, so one captured graph replays every step
  long long col;        // current column of the stream matrix (timestep)
  long long adam_t;     // Adam step count (optim.py:21 self.t)
  long long step_count; // Predictor.step_count
  long long loss_base;  // column whose loss goes to losses[0]
  AdamScalars adam;
  unsigned long long err_key;   // min over (step << 24 | stream << 3 | code); ~0 = none
  double alpha_sum, alpha_min, alpha_max;   // last predict's router stats
  // ring-buffer cache (ModelPtrs.ring_on): rolls counted since the cache was
  // last set; logical D-block j of every cache row lives at physical D-block
  // (j + ring) mod (C / D).  trunk_fwd writes the new block at D-block
  // `ring`, the forward W_mem GEMM reads with ring + 1 (ring_bias), and
  // mix_fwd (the next kernel) counts the roll.
  long long ring;
};

struct Acts {        // saved activations and gradient scratch, all [B][ld]
  // forward
  float *x, *x_hat, *x_inv, *gpre, *vpre, *loc, *loc_hat, *loc_inv, *conv_pre, *h_l;
  float *cache;                 // [B][C] rolling cache (ring buffer when ring_on, else rolled
                                //  in place each predict)
  float *ws_mem, *upre, *h_g, *alpha, *h_mix, *z_hat, *z_inv, *z;   // router pre-activation: sk[S_RPRE]
  float *zd, *u, *inner, *gate, *h_c, *z2_hat, *z2_inv, *z2;
  // TF32-rounded copies of x and h_mix for their GEMMs (route / W_route
  // update, cgate / W_cgate update): the fp32 originals also feed residuals
  float *x_tc, *hm_tc;
  float *a12, *wide, *ws_f, *n_hat, *n_inv, *nrm, *h, *logits;
  double *probs;                // [B][256] (predict API only)
  unsigned *cum;                // [2][B][kCumLd] CSPP slots
  double *nll;                  // [B]
  float *alpha_row;             // [B][3] per-row router stats (sum, min, max)
  // backward
  float *dlogits, *dhc, *dnpre, *da12, *ws_dz2, *dinner, *dcpre;
  float *dzd, *drpre, *dupre, *dh_l, *dx_part;
  float *tb_dx, *tb_dls;        // [B][H] trunk backward at large B: dx and dloc rows
  float *rowred;                // [B][rowred]
  float *trunk_part;            // [trunk_grid][trunk1 - trunk0] per-CTA sums of trunk_bwd
  long long* emb_acc;           // [256][D] embedding gradient, fixed point (emb_to_fixed)
};

// Split-K partial planes of the narrow GEMMs: the GEMM writes S slices of
// [B][N] and the consuming row kernel reduces them in a fixed order
// (split_sum), so a 8-40-tile GEMM still spreads over ~128-148 SMs.
enum SplitId { S_ZD, S_INNER, S_CPRE, S_LOGITS, S_DH, S_DU, S_DHMC, S_DZ, S_DXR, S_DBLOCK, S_RPRE,
               S_COUNT };
struct SplitBuf {
  float* ws;
  int S;
};

struct ModelPtrs {   // everything a row kernel may need, passed by value
  Dims d;
  int variant;         // Variant
  SmallLayout sl;
  Tensor4 w[P_COUNT];  // for small params these point into the small arena
  float* small_p; float* small_m; float* small_v; float* small_g;
  Acts a;
  StepState* st;
  int splits_mem, splits_f, splits_dz2;
  SplitBuf sk[S_COUNT];
  double lr, beta1, beta2, adam_eps;   // Adam hyperparameters (config.py:29-32)
  // executors only: device event tape [steps][kTapeSlots] indexed by
  // col - loss_base (null: not recorded)
  unsigned long long* tape;
  // 1: the rolling cache is a ring buffer (D and B multiples of the 32-float
  // GEMM k-tile): predict writes one block in place instead of moving (C - D)
  // floats per row (ref nn/ops.py:219-231 roll_cache semantics unchanged).
  // Layout then block-major, cache[(kb * B + b) * 32 + e] for physical
  // 32-column block kb, so the W_mem GEMMs read whole contiguous tiles.
  int ring_on;
  // trunk_bwd grid: min(B, 4 per SM); each CTA loops over rows b = cta,
  // cta + grid, ... and writes one partial row of its small-parameter sums
  int trunk_grid;
  // rows of the rowred matrix small_adam sums (rowred_rows): B, or B / 4 when
  // the warp-per-row backward kernels write one combined row per CTA
  int rr_rows;
  int dbg;   // experiments build only (FADE_DBG_TRUNK): bit 0 drops the embedding-gradient atomics
};

// The ring-buffer cache is an experiments-build option (engine.cu, FADE_RING):
// the shipped kernels compile its branches out.
__device__ __forceinline__ bool ring_cache(const ModelPtrs& M) {
#ifdef FADE_EXPERIMENTS
  return M.ring_on != 0;
#else
  (void)M;
  return false;
#endif
}
__device__ __forceinline__ unsigned long long* tape_at(const ModelPtrs& M, int slot) {
  return M.tape + kTapeSlots * (M.st->col - M.st->loss_base) + slot;
}

// warp-per-row variants (row_warp.cu); false: geometry not covered (H % 128)
bool launch_mix_fwd_w(const ModelPtrs& M, cudaStream_t s);
bool launch_coarse_fwd_w(const ModelPtrs& M, cudaStream_t s);
bool launch_out_fwd_w(const ModelPtrs& M, cudaStream_t s);
bool launch_out_bwd_w(const ModelPtrs& M, cudaStream_t s);
bool launch_coarse_bwd_w(const ModelPtrs& M, cudaStream_t s);
bool launch_mix_bwd_w(const ModelPtrs& M, cudaStream_t s);
bool launch_trunk_fwd_w(const ModelPtrs& M, const uint8_t* src, long long ld_src, int use_col,
                        cudaStream_t s);
bool launch_trunk_bwd_w(const ModelPtrs& M, const uint8_t* src, long long ld_src, int use_col,
                        cudaStream_t s);
// large-B trunk backward (row_warp.cu): true when launch_trunk_bwd runs the
// warp-per-row input-gradient kernel + the in/loc LayerNorm gradient kernel,
// and the caller runs launch_trunk_grads_conv (conv / GeGLU weight gradients,
// ready after the dx_r GEMM) on a second stream before small_adam
bool trunk_bwd_split(const ModelPtrs& M);
int rowred_rows(int B, int H);
void launch_trunk_grads_conv(const ModelPtrs& M, cudaStream_t s);
bool row_warp_enabled(int B, int which);   // which: 0 mix_fwd .. 5 mix_bwd

// row kernels (model_kernels.cu)
void launch_trunk_fwd(const ModelPtrs& M, const uint8_t* src, long long ld_src, int use_col,
                      cudaStream_t s);
void launch_mix_fwd(const ModelPtrs& M, cudaStream_t s);
void launch_bmm_fwd(const ModelPtrs& M, cudaStream_t s);
void launch_coarse_fwd(const ModelPtrs& M, cudaStream_t s);
void launch_out_fwd(const ModelPtrs& M, cudaStream_t s);
// head: fp64 softmax -> quantiser -> cum slot; optional probs; optional
// cross-entropy with targets read from tgt (+ col) or decoded in place.
struct HeadArgs {
  int adam_prep;            // 1: this step trains -> t += 1 and Adam scalars (optim.py:26-30)
  int want_probs;
  int xent;                 // 1: emit dlogits + nll
  const uint8_t* tgt;       // target bytes (row b at tgt + b*ld_tgt + col) or null
  long long ld_tgt;
  int tgt_use_col;
  // decoder (decompression: decode the symbol of each stream from this table)
  int decode;
  uint8_t* out;             // decoded byte -> out[b*ld_out + col]
  long long ld_out;
  const uint8_t* payload;
  const long long* off;
  const long long* dlen;
  long long* dpos;
  unsigned long long* dcode;
  unsigned long long* drng;
  int skip_quant;           // 1: the quantiser runs on the coder stream (k_head_quant)
};
void launch_head(const ModelPtrs& M, const HeadArgs& h, cudaStream_t s);
void launch_head_quant(const ModelPtrs& M, const long long* colp, cudaStream_t s);
void launch_out_bwd(const ModelPtrs& M, cudaStream_t s);
void launch_coarse_bwd(const ModelPtrs& M, cudaStream_t s);
void launch_bmm_bwd(const ModelPtrs& M, int grad_only, int mode, cudaStream_t s);
void launch_mix_bwd(const ModelPtrs& M, cudaStream_t s);
void launch_trunk_bwd(const ModelPtrs& M, const uint8_t* src, long long ld_src, int use_col,
                      cudaStream_t s);
// small-parameter + embedding Adam and the step loss; advance = 1 also moves
// the step state to the next column (the last kernel of a trained step)
// alpha_tape (optional): per-step router statistics (mean, min, max) at
// [3 * (col - loss_base)], the metrics tape of pipeline.py:162-185
void launch_small_adam(const ModelPtrs& M, int grad_only, double* losses, double* alpha_tape,
                       int advance, cudaStream_t s);

// Embedding-gradient accumulator: 2^-48 fixed point in int64.  Integer
// addition is associative, so atomics give a bit-reproducible sum (encoder
// and decoder replay the same trajectory); 2^-48 resolution is far below the
// fp32 rounding of the gradient values and |sum| < 2^15 leaves ample range.
__device__ __forceinline__ long long emb_to_fixed(float g) {
  return __double2ll_rn((double)g * 0x1p48);
}
__device__ __forceinline__ float emb_from_fixed(long long v) {
  return (float)((double)v * 0x1p-48);
}

}  // namespace fade
