/*
 * fade_b200.h -- C ABI of the B200-native FADE compression hot path.
 *
 * One shared library (paper_2604_07239_b200/_lib/libfade_b200.so, sm_100a)
 * replaces the reference's CPU path behind its own interfaces:
 *
 *  1. The kernel table.  The reference selects five integer kernels at import
 *     time (pkg/src/dszip/kernels.py:236-273, `BACKENDS[name]`, chosen by
 *     DSZIP_BACKEND).  fade_quantize_rows / fade_encode_step / fade_flush /
 *     fade_prime / fade_decode_step are drop-in entries for that table with
 *     the same argument meaning (int64 arrays, rows [r0, r1), in-place state,
 *     return -1 or the first failing row) -- but the arrays are DEVICE
 *     pointers and `stream` is a cudaStream_t.  These calls synchronise the
 *     stream because the return value is the reference's error protocol.
 *  2. The predictor.  fade_model_* replace pkg/src/dszip/model.py:44-259
 *     (Predictor.__init__/predict/train_step/forward_debug/loss_grads/
 *     save_state/load_state).  Host pointers; the model owns its device state.
 *  3. The executors.  fade_compress / fade_decompress run the whole per-step
 *     loop of pkg/src/dszip/pipeline.py:197-396 on the device (model stream +
 *     coder stream, CUDA graphs); the host only moves the input in and the
 *     bitstreams out.
 *
 * No function throws; every one returns a status (FADE_OK == 0) and leaves a
 * message in fade_last_error().  Data-dependent failures additionally fill a
 * fade_error_t record (kind, stream, step, why) mirroring CorruptionError /
 * ModelDivergenceError (pkg/src/dszip/errors.py:34-60).
 */
#ifndef FADE_B200_H
#define FADE_B200_H

#include <stdint.h>

#if defined(__GNUC__)
#define FADE_API __attribute__((visibility("default")))
#else
#define FADE_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

enum {
  FADE_OK = 0,
  FADE_ERR_CUDA = 1,      /* CUDA runtime/driver failure                      */
  FADE_ERR_USAGE = 2,     /* bad argument / unsupported geometry              */
  FADE_ERR_CORRUPT = 3,   /* decoder: invalid code (why 1) or truncated (2)   */
  FADE_ERR_DIVERGED = 4,  /* non-finite logits or loss                        */
  FADE_ERR_QUANT = 5,     /* a probability row is not a distribution          */
  FADE_ERR_ZERO_FREQ = 6, /* encoder: symbol with zero frequency              */
  FADE_ERR_STATE = 7      /* call order violated (e.g. train without predict) */
};

typedef struct {
  int32_t kind;   /* FADE_ERR_* */
  int32_t why;    /* decoder: 1 invalid code value, 2 truncated stream */
  int64_t stream; /* first failing stream (lowest index at the first failing step) */
  int64_t step;   /* coder timestep (column of the stream matrix) */
} fade_error_t;

FADE_API const char* fade_last_error(void);
FADE_API int fade_abi_version(void);
FADE_API int fade_device_count(void);
/* Compute capability and name of `device` (the per-shard fingerprint of the
 * v2 container records which GPU architecture wrote each shard). */
FADE_API int fade_device_arch(int device, int* major, int* minor, char* name, int name_len);

/* ---- 1. kernel table: kernels.py:48-233 (device pointers) ----------------- */

/* kernels.py:48-85 _quantize_rows: probs f64[R,256] -> freq i64[R,256]. */
FADE_API int64_t fade_quantize_rows(const double* probs, int64_t* freq, int64_t r0, int64_t r1,
                           void* stream);
/* kernels.py:123-155 _encode_step.  cum i64 rows of `cum_ld` (>=257) entries,
 * buf u8 rows of `buf_ld` bytes (the caller guarantees capacity, as
 * BatchEncoder._ensure_capacity does in coder.py:65-73). */
FADE_API int64_t fade_encode_step(const int64_t* cum, int64_t cum_ld, const int64_t* syms,
                         int64_t* low, int64_t* rng, int64_t* cache, int64_t* ncache,
                         uint8_t* buf, int64_t buf_ld, int64_t* blen, int64_t r0,
                         int64_t r1, void* stream);
/* kernels.py:158-183 _flush */
FADE_API int64_t fade_flush(int64_t* low, int64_t* cache, int64_t* ncache, uint8_t* buf,
                   int64_t buf_ld, int64_t* blen, int64_t r0, int64_t r1, void* stream);
/* kernels.py:186-197 _prime */
FADE_API int64_t fade_prime(const uint8_t* payload, const int64_t* off, const int64_t* dlen,
                   int64_t* pos, int64_t* code, int64_t* rng, int64_t r0, int64_t r1,
                   void* stream);
/* kernels.py:200-233 _decode_step; *why receives 1 (invalid code) or 2 (truncated). */
FADE_API int64_t fade_decode_step(const int64_t* cum, int64_t cum_ld, const uint8_t* payload,
                         const int64_t* off, const int64_t* dlen, int64_t* pos,
                         int64_t* code, int64_t* rng, int64_t* out, int64_t r0, int64_t r1,
                         int64_t* why, void* stream);

/* ---- 2. predictor: model.py:44-259 --------------------------------------- */

typedef struct {
  int32_t ctx_len, embed_dim, cache_dim, mix_dim, expand_dim, batch, alphabet, conv_kernel;
  double lr, beta1, beta2, adam_eps;
  /* ablation variant (model.py:39): 0 full, 1 dual, 2 global_only, 3 local_only,
   * 4 mixer_nogate, 5 mixer */
  int32_t variant;
} fade_config_t;

typedef struct fade_model fade_model_t;

/* Allocates all device state (parameters zeroed; upload the seeded init with
 * fade_model_set_tensor -- model.py:62-105 draws it with numpy on the host). */
FADE_API int fade_model_create(const fade_config_t* cfg, int device, fade_model_t** out);
FADE_API int fade_model_destroy(fade_model_t* m);

/* Tensor transfer in the reference's layout and PARAM order (model.py:76-105).
 * kind: 0 parameter, 1 Adam m, 2 Adam v, 3 last gradient (after loss_grads).
 * index: 0..28 in the reference's parameter order.  n = element count. */
FADE_API int fade_model_set_tensor(fade_model_t* m, int kind, int index, const float* host, int64_t n);
FADE_API int fade_model_get_tensor(fade_model_t* m, int kind, int index, float* host, int64_t n);
FADE_API int fade_model_set_cache(fade_model_t* m, const float* host);   /* f32[B, cache_dim] */
FADE_API int fade_model_get_cache(fade_model_t* m, float* host);
FADE_API int fade_model_set_counters(fade_model_t* m, int64_t adam_t, int64_t step_count);
FADE_API int fade_model_get_counters(fade_model_t* m, int64_t* adam_t, int64_t* step_count);

/* Predictor.predict (model.py:183-201): ctx u8[B, ctx_len] host.  Writes
 * probs f64[B,256] (may be NULL) and alpha (mean,min,max) (may be NULL). */
FADE_API int fade_model_predict(fade_model_t* m, const uint8_t* ctx, double* probs, double* alpha,
                       fade_error_t* err);
/* Predictor.train_step (model.py:203-215): targets u8[B]. */
FADE_API int fade_model_train_step(fade_model_t* m, const uint8_t* targets, double* loss,
                          fade_error_t* err);
/* Predictor.forward_debug (model.py:217-220): no state change.  part is one of
 * global, local, alpha, mix, mixer_inner, coarse, hidden, logits; out f32[B, width]. */
FADE_API int fade_model_forward_debug(fade_model_t* m, const uint8_t* ctx, const char* part, float* out);
/* Predictor.loss_grads (model.py:228-237): gradients readable with kind 3. */
FADE_API int fade_model_loss_grads(fade_model_t* m, const uint8_t* ctx, const uint8_t* targets,
                          double* loss);

/* ---- 3. executors: pipeline.py:197-396 ----------------------------------- */

/* Compress a B x L stream matrix (row b = stream b, pipeline.py:35-64).
 * `data` is host memory (on_device = 0) or device memory (on_device = 1).
 * The first `warm` columns are uniform-coded with no model call
 * (pipeline.py:193,212-213).  m may be NULL when L <= warm; the call then
 * runs on `device` (with a model, on the model's device).  Every call leaves
 * the calling thread's current CUDA device as it found it.
 * pipelined = 1 runs the coder on its own CUDA stream, double-buffered against
 * the model (the CSPP of pipeline.py:229-299); 0 is the serial order.  Both
 * produce identical bytes.  Outputs (host, each may be NULL): lengths[B];
 * losses[L-warm]; alpha[3*(L-warm)] per-step router mean/min/max for the
 * metrics tape (pipeline.py:162-185); tape[5*(L-warm)] the device event tape
 * (%globaltimer ns per model step: table fill begins, table full, drain
 * begins, drain done, step done -- the PingPongBuffer slot transitions of
 * pipeline.py:86-149 as the device ran them).  Fetch the bytes with
 * fade_coder_fetch.  A divergence reports err->step = Predictor.step_count at
 * the failing column (model.py:190-193,208-209: column - warm for a fresh
 * model); a coder error reports the column. */
typedef struct fade_coder fade_coder_t;
FADE_API int fade_compress(fade_model_t* m, int device, int batch, const uint8_t* data, int64_t L,
                  int64_t warm, int on_device, int pipelined, int64_t* lengths, double* losses,
                  double* alpha, uint64_t* tape, fade_coder_t** coder, fade_error_t* err);
/* Concatenated stream bytes (payload order of container.py:99-110). */
FADE_API int fade_coder_fetch(fade_coder_t* c, uint8_t* payload, int64_t nbytes);
FADE_API int fade_coder_destroy(fade_coder_t* c);

/* Decompress (pipeline.py:310-396): payload host bytes, lengths[B] host.
 * Writes the B x L matrix to out (host), losses[L-warm], alpha[3*(L-warm)]
 * and tape[5*(L-warm)] (each may be NULL; tape slots 2-3 stamp the decoder
 * inside the head kernel).  `device` as for fade_compress. */
FADE_API int fade_decompress(fade_model_t* m, int device, int batch, const uint8_t* payload,
                    int64_t nbytes, const int64_t* lengths, int64_t L, int64_t warm,
                    uint8_t* out, double* losses, double* alpha, uint64_t* tape,
                    fade_error_t* err);

/* ---- measurement hooks (bench.py) ------------------------------------------ */

/* The model's launch stream (cudaStream_t), so callers can time on it. */
FADE_API int fade_model_stream(fade_model_t* m, void** stream);

/* Time `iters` back-to-back launches of one step component in isolation on the
 * model stream (state from the last step): 0 = FNR expand GEMM (e12, GeGLU
 * epilogue), 1 = W12 gradient GEMM with fused Adam, 2 = W_mem gradient + Adam
 * group, 3 = per-stream memory backward + Adam (bmm_bwd), 4 = FNR project GEMM
 * (split-K).  Writes the mean ms per launch and the algorithmic bytes and
 * FLOPs of one launch. */
FADE_API int fade_bench_probe(fade_model_t* m, int which, int iters, double* ms, double* bytes,
                              double* flops);

/* Run `steps` model timesteps of compression starting at column `start` of a
 * device-resident B x L matrix, without host synchronisation; the coder keeps
 * its state in `coder` (created on first use).  Returns the number of kernel
 * launches issued per timestep in *launches (may be NULL). */
FADE_API int fade_bench_compress_steps(fade_model_t* m, const uint8_t* data_dev, int64_t L,
                              int64_t start, int64_t steps, fade_coder_t** coder,
                              int* launches, void* stream);

/* ---- test hooks (tests/test_gpu_gemm.py) ------------------------------------ */

/* tcgen05 TF32 GEMM on device pointers: C[M,N] = A.B; a_trans=1 means A is
 * stored [K][M]; b_trans=1 means B is stored [N][K]; splits>1 writes partial
 * slices at C + s*M*ldc.  bn is the tile width (64, 128 or 256); pair = 2
 * runs CTA pairs (tcgen05 cta_group::2, 256-row tiles; bn 128 or 256); pair | 4
 * selects the persistent warp-specialised kernel (gemm_ws.cuh). */
FADE_API int fade_debug_gemm(const float* A, long long lda, int a_trans, const float* B,
                             long long ldb, int b_trans, float* C, long long ldc, int M, int N,
                             int K, int splits, int bn, int pair, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* FADE_B200_H */
