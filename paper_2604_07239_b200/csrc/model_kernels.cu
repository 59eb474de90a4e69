// Fused row kernels of the FADE predictor (one CTA per stream row).
//
// Forward follows pkg/src/dszip/model.py:109-179 and the op definitions of
// pkg/src/dszip/nn/ops.py; backward restates the autograd closures of the same
// ops.  Every reduction is a fixed-order tree (no atomics on values), so the
// encoder and the decoder regenerate bit-identical probabilities.
#include "coder.cuh"
#include "model.cuh"

namespace fade {

// warp-per-row kernels (row_warp.cu) for H % 128 == 0; experiments build:
// FADE_ROW_WARP=0 keeps the CTA-per-row kernels below
// Measured per B (timestep, same box): B = 512 336 -> 364 us, 1024 530 ->
// 547 us (one warp per row is too little parallelism per row when the grid is
// small), 2048 883 -> 844 us, 4096 1631 -> 1547 us; so B >= 2048 only.
bool row_warp_enabled(int B, int which) {
  static const int forced = knob("FADE_ROW_WARP") ? atoi(knob("FADE_ROW_WARP")) : -1;
  if (forced >= 0) return (forced >> which) & 1;   // experiments: a bit per kernel
  return B >= 2048;
}

constexpr int kRowMax = 512;
constexpr int kBmmThreads = 128;
constexpr int kBmmRows = 16;      // W_U rows per k_bmm_bwd CTA (its 25 KB of smem fits beside
                                   // the two W_f update CTAs that share the SMs at that time)
// The trunk kernels run 256 threads x 2 elements at <= 64 registers so four
// CTAs fit per SM: all B = 512 rows are resident in ONE wave (512-thread CTAs
// at 64 registers fit two per SM -> two serial waves of a latency-bound row).
constexpr int kTrunkThreads = 256;

// One CTA per stream row with one thread per row element (H = 512 -> 512
// threads): B = 512 rows alone give only ~3.5 CTAs per SM, so the parallelism
// has to come from inside the row to keep enough loads in flight.
static int row_threads(int width) {
  const int t = (width + 31) / 32 * 32;
  return t < 128 ? 128 : (t > kRowMax ? kRowMax : t);
}

// LayerNorm statistics of a row held in shared memory (ops.py:94-101):
// mu = mean(x); var = mean((x-mu)^2); inv = 1/sqrt(var + eps)
__device__ __forceinline__ void ln_stats(const float* xs, int n, float* red, float* mu_out,
                                         float* inv_out) {
  float s = 0.f;
  for (int j = threadIdx.x; j < n; j += blockDim.x) s += xs[j];
  const float mu = block_sum_rt(s, red) / (float)n;
  float q = 0.f;
  for (int j = threadIdx.x; j < n; j += blockDim.x) {
    const float c = xs[j] - mu;
    q += c * c;
  }
  const float var = block_sum_rt(q, red) / (float)n;
  *mu_out = mu;
  *inv_out = __fdiv_rn(1.0f, __fsqrt_rn(var + kLnEps));
}

// Fixed-order reduction of S split-K partial planes at element idx: four
// independent accumulators (slices s = k mod 4) keep the loads in flight.
template <int kSplitBatch = 4>
__device__ __forceinline__ float split_sum(const float* __restrict__ ws, long long plane,
                                           long long idx, int S) {
  // loads issued kSplitBatch planes at a time (one L2 round trip per batch),
  // then added in plane order: the same additions in the same order as a
  // plain `a[s & 3] += ws[s]` loop, whatever the batch (kernels capped at 32
  // registers keep 4; the head reduces its logit slices 8 at a time)
  float a[4] = {0.f, 0.f, 0.f, 0.f};
  if constexpr (kSplitBatch == 4) {
    // (the unrolled-by-4 loop resolves a[s & 3] to registers; measured faster
    // than a hand-split main/remainder loop)
#pragma unroll 4
    for (int s = 0; s < S; ++s) a[s & 3] += ws[s * plane + idx];
    return (a[0] + a[1]) + (a[2] + a[3]);
  }
  for (int s0 = 0; s0 < S; s0 += kSplitBatch) {
    float v[kSplitBatch];
#pragma unroll
    for (int k = 0; k < kSplitBatch; ++k)
      if (s0 + k < S) v[k] = ws[(s0 + k) * plane + idx];
#pragma unroll
    for (int k = 0; k < kSplitBatch; ++k)
      if (s0 + k < S) a[k & 3] += v[k];
  }
  return (a[0] + a[1]) + (a[2] + a[3]);
}
// Row [rH, rH + n) of S split-K planes reduced into dst (smem), bit-identical
// to split_sum: thread group g (of 4) sums the planes s = g mod 4 in order with
// float4 loads -- every thread of the CTA keeps loads in flight -- and the
// four partial rows combine as (p0 + p1) + (p2 + p3).  part: [4][n] smem.
__device__ __forceinline__ void split_row(float* dst, float* part, const float* __restrict__ ws,
                                          long long plane, long long rH, int n, int S) {
  const int n4 = n / 4;      // n % 4 == 0 (ModelConfig.device_check)
  for (int idx = threadIdx.x; idx < 4 * n4; idx += blockDim.x) {
    const int g = idx / n4, j4 = idx - g * n4;
    float4 a = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll 4
    for (int s = g; s < S; s += 4) {
      const float4 v = *(const float4*)(ws + s * plane + rH + 4 * j4);
      a.x += v.x;
      a.y += v.y;
      a.z += v.z;
      a.w += v.w;
    }
    *(float4*)(part + g * n + 4 * j4) = a;
  }
  __syncthreads();
  for (int j = threadIdx.x; j < n; j += blockDim.x)
    dst[j] = (part[j] + part[n + j]) + (part[2 * n + j] + part[3 * n + j]);
  __syncthreads();
}

// element idx of a narrow GEMM's output [B][N] (plane = B*N), reduced over its slices
template <int kSplitBatch = 4>
__device__ __forceinline__ float sk_sum(const SplitBuf& k, long long plane, long long idx) {
  return split_sum<kSplitBatch>(k.ws, plane, idx, k.S);
}

// LayerNorm backward over one row (ops.py:103-113): returns dx into dxs (smem or
// regs written by caller).  g = upstream grad (smem), xhat (global row), gain.
__device__ __forceinline__ void ln_bwd_means(const float* gs, const float* xhat_row,
                                             const float* gain, int n, float* red, float* m1,
                                             float* m2) {
  float s1 = 0.f, s2 = 0.f;
  for (int j = threadIdx.x; j < n; j += blockDim.x) {
    const float gg = gs[j] * gain[j];
    s1 += gg;
    s2 += gg * xhat_row[j];
  }
  *m1 = block_sum_rt(s1, red) / (float)n;
  *m2 = block_sum_rt(s2, red) / (float)n;
}

// ---------------------------------------------------------------------------
// trunk + local stream forward (model.py:118-137)
// DT/TT/KT > 0: compile-time embed width, context length, conv taps (the
// default geometry), so index math folds to shifts and the tap loops unroll;
// 0 = runtime geometry
template <int DT, int TT, int KT>
__global__ void __launch_bounds__(kTrunkThreads, 4) k_trunk_fwd(ModelPtrs M, const uint8_t* src,
                                                       long long ld_src, int use_col) {
  pdl_enter();
  Dims d = M.d;
  if (DT) { d.D = DT; d.T = TT; d.K = KT; d.H = DT * TT; }
  const int tid = threadIdx.x;
  extern __shared__ float sm[];
  float* es = sm;                         // raw embedding row [H]
  float* xs = es + d.H;                   // x row [H]
  float* locs = xs + d.H;                 // LN_D(emb) row [H]
  float* wg = locs + d.H;                 // [D*D]
  float* wv = wg + d.D * d.D;             // [D*D]
  float* ck = wv + d.D * d.D;             // [K*D*D]
  float* blk = ck + d.K * d.D * d.D;      // [D]
  float* tmu = blk + d.D;                 // [T]
  float* tinv = tmu + d.T;                // [T]
  float* red = tinv + d.T;                // [32]
  int* ctx = (int*)(red + 32);            // [T]
  // DT > 0: the cache tail [D, C) staged for the in-place roll (16-B aligned)
  float* cstage = (float*)(((uintptr_t)(ctx + d.T) + 15) & ~(uintptr_t)15);

  const VFlags vf = vflags(M.variant);
  const long long c0 = use_col ? M.st->col - d.T : 0;
  if (M.tape && blockIdx.x == 0 && tid == 0) *tape_at(M, 0) = gtimer_ns();
  const int n4 = (d.C - d.D) / 4;        // float4 count the roll moves
  // ring buffer (block-major [C/32][B][32], model.cuh): the new block
  // overwrites the oldest one in place; nothing else moves (ref
  // ops.py:219-231 semantics).  Element o of the new block lands at
  // ring_elem(o); without the ring, at crow[C - D + o] after the roll.
  const bool ring = ring_cache(M);
  const int rnb = d.C / 32, rstep = d.D / 32;
  const int rb0 = ring ? (int)((M.st->ring * rstep) % rnb) : 0;
  // the weights are staged once per CTA; a CTA walks rows b = cta, cta +
  // grid, ... (grid = min(B, 4 per SM): at large B the 20 KB of weights are
  // not re-read for every row)
  if constexpr (DT > 0) {
    // weights into smem as float4: at the compiled geometry (D = 32, H = 512)
    // every small-arena offset is a multiple of 4 floats (make_small_layout)
    // (cp.async: no register round trip before the embedding gather; they
    // are first read after the LayerNorm, behind a wait_all + barrier)
    const float4* g4 = (const float4*)M.w[P_W_GATE].p;
    const float4* v4 = (const float4*)M.w[P_W_VAL].p;
    const float4* k4 = (const float4*)M.w[P_CONV_K].p;
    auto cp16 = [](float* dst, const float4* src) {
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(
                       (uint32_t)__cvta_generic_to_shared(dst)),
                   "l"(src)
                   : "memory");
    };
    for (int j = tid; j < d.D * d.D / 4; j += blockDim.x) {
      cp16(wg + 4 * j, g4 + j);
      cp16(wv + 4 * j, v4 + j);
    }
    for (int j = tid; j < d.K * d.D * d.D / 4; j += blockDim.x) cp16(ck + 4 * j, k4 + j);
    asm volatile("cp.async.commit_group;" ::: "memory");
  } else {
    for (int j = tid; j < d.D * d.D; j += blockDim.x) {
      wg[j] = M.w[P_W_GATE].p[j];
      wv[j] = M.w[P_W_VAL].p[j];
    }
    for (int j = tid; j < d.K * d.D * d.D; j += blockDim.x) ck[j] = M.w[P_CONV_K].p[j];
  }
  for (int b = blockIdx.x; b < d.B; b += gridDim.x) {
  float* crow = M.a.cache + (long long)b * d.C;
  auto ring_elem = [&](int o) -> float* {
    return M.a.cache + (((long long)((rb0 + (o >> 5)) % rnb) * d.B + b) << 5) + (o & 31);
  };
  if constexpr (DT > 0) {
    // the roll's reads depend on nothing this kernel computes: start them
    // first (cp.async into smem) so they land under the LayerNorm/GeGLU work
    if (vf.global && !ring) {
      for (int q = tid; q < n4; q += blockDim.x)
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(
                         (uint32_t)__cvta_generic_to_shared(cstage + 4 * q)),
                     "l"(crow + d.D + 4 * q)
                     : "memory");
      asm volatile("cp.async.commit_group;" ::: "memory");
    }
  }
  for (int t = tid; t < d.T; t += blockDim.x) ctx[t] = src[(long long)b * ld_src + c0 + t];
  __syncthreads();

  // embedding gather + input LayerNorm over the flattened window
  const float* E = M.w[P_EMB].p;
  for (int j = tid; j < d.H; j += blockDim.x) es[j] = E[ctx[j / d.D] * d.D + (j % d.D)];
  __syncthreads();
  float mu, inv;
  ln_stats(es, d.H, red, &mu, &inv);
  const float* g_in = M.w[P_IN_LN_G].p;
  const float* b_in = M.w[P_IN_LN_B].p;
  const long long rH = (long long)b * d.H;
  for (int j = tid; j < d.H; j += blockDim.x) {
    const float xh = (es[j] - mu) * inv;
    const float xv = xh * g_in[j] + b_in[j];
    xs[j] = xv;
    M.a.x_hat[rH + j] = xh;
    M.a.x[rH + j] = xv;
    M.a.x_tc[rH + j] = tf32_rne(xv);
  }
  if (tid == 0) M.a.x_inv[b] = inv;
  if constexpr (DT > 0) asm volatile("cp.async.wait_all;" ::: "memory");   // weights (and roll reads) landed
  __syncthreads();

  // GeGLU block of the newest symbol: gelu(x_t W_gate) * (x_t W_val)
  const float* xt = xs + (d.H - d.D);
  if constexpr (DT > 0) {
    if (vf.global) {
      // warp w sums inputs i in [4w, 4w + 4) for all 32 outputs (lane = o;
      // conflict-free weight rows, broadcast x_t), then a fixed-order sum of
      // the 8 warp partials; the staged cache tail is written back meanwhile
      static_assert(kTrunkThreads / 32 * 4 == DT, "GeGLU split");
      float* pg = locs;                    // [8][32] partials (locs is free until the local LN)
      float* pv = locs + 256;
      const int w = tid >> 5, o = tid & 31;
      float g = 0.f, v = 0.f;
#pragma unroll
      for (int i = 4 * w; i < 4 * w + 4; ++i) {
        g += xt[i] * wg[i * DT + o];
        v += xt[i] * wv[i * DT + o];
      }
      pg[w * 32 + o] = g;
      pv[w * 32 + o] = v;
      asm volatile("cp.async.wait_all;" ::: "memory");
      __syncthreads();     // partials visible; every thread's cache reads landed
      if (tid < DT) {
        float gs = 0.f, vs = 0.f;
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          gs += pg[k * 32 + tid];
          vs += pv[k * 32 + tid];
        }
        M.a.gpre[(long long)b * DT + tid] = gs;
        M.a.vpre[(long long)b * DT + tid] = vs;
        *(ring ? ring_elem(tid) : crow + d.C - DT + tid) = tf32_rne(gelu_f(gs) * vs);
      }
      if (!ring)
        for (int q = tid; q < n4; q += blockDim.x) *(float4*)(crow + 4 * q) = *(const float4*)(cstage + 4 * q);
      __syncthreads();     // locs partials consumed
    }
  } else if (vf.global) {
  for (int o = tid; o < d.D; o += blockDim.x) {
    float g = 0.f, v = 0.f;
    for (int i = 0; i < d.D; ++i) {
      g += xt[i] * wg[i * d.D + o];
      v += xt[i] * wv[i * d.D + o];
    }
    M.a.gpre[(long long)b * d.D + o] = g;
    M.a.vpre[(long long)b * d.D + o] = v;
    blk[o] = tf32_rne(gelu_f(g) * v);
  }
  // roll the cache in place: new[j] = old[j + D]; new[C-D+o] = block[o]
  if (ring) {
    __syncthreads();
    for (int o = tid; o < d.D; o += blockDim.x) *ring_elem(o) = blk[o];
  } else {
    constexpr int U = 4;
    for (int base = 0; base < n4; base += U * (int)blockDim.x) {
      float4 r[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int q = base + u * (int)blockDim.x + tid;
        if (q < n4) r[u] = *(const float4*)(crow + d.D + 4 * q);
      }
      __syncthreads();
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int q = base + u * (int)blockDim.x + tid;
        if (q < n4) *(float4*)(crow + 4 * q) = r[u];
      }
      __syncthreads();
    }
    __syncthreads();
    for (int o = tid; o < d.D; o += blockDim.x) crow[d.C - d.D + o] = blk[o];
  }
  }   // global stream
  if (vf.local) {

  // local stream: per-symbol LayerNorm over D (ops.py:94-101 on (B,T,D))
  if constexpr (DT > 0) {
    // warp w normalises symbols t = w, w + 8 (lane = e): shuffle trees
    // instead of 32-long serial sums on 16 threads
    const int w = tid >> 5, e = tid & 31;
#pragma unroll
    for (int t = w; t < TT; t += kTrunkThreads / 32) {
      const float x = es[t * DT + e];
      const float m = warp_sum(x) / (float)DT;
      const float c = x - m;
      const float var = warp_sum(c * c) / (float)DT;
      if (e == 0) {
        tmu[t] = m;
        tinv[t] = __fdiv_rn(1.0f, __fsqrt_rn(var + kLnEps));
        M.a.loc_inv[(long long)b * TT + t] = tinv[t];
      }
    }
  } else
  for (int t = tid; t < d.T; t += blockDim.x) {
    float s = 0.f;
    for (int e = 0; e < d.D; ++e) s += es[t * d.D + e];
    const float m = s / (float)d.D;
    float q = 0.f;
    for (int e = 0; e < d.D; ++e) {
      const float c = es[t * d.D + e] - m;
      q += c * c;
    }
    tmu[t] = m;
    tinv[t] = __fdiv_rn(1.0f, __fsqrt_rn(q / (float)d.D + kLnEps));
    M.a.loc_inv[(long long)b * d.T + t] = tinv[t];
  }
  __syncthreads();
  const float* lg = M.w[P_LOC_LN_G].p;
  const float* lb = M.w[P_LOC_LN_B].p;
  for (int j = tid; j < d.H; j += blockDim.x) {
    const int t = j / d.D, e = j % d.D;
    const float lh = (es[j] - tmu[t]) * tinv[t];
    const float lv = lh * lg[e] + lb[e];
    locs[j] = lv;
    M.a.loc_hat[rH + j] = lh;
    M.a.loc[rH + j] = lv;
  }
  __syncthreads();
  // same-padded conv, taps in ascending order (ops.py:57-72), then gelu
  const float* cb = M.w[P_CONV_B].p;
  const int pad = d.K / 2;
  if constexpr (DT > 0) {
    // 256 threads = (co, t0) with t0 < TT/2; each thread also computes
    // t1 = t0 + TT/2 with the same taps: every kernel weight load feeds two
    // outputs, the inputs come in as float4 warp broadcasts (same t per warp)
    static_assert(DT == 32 && TT == 16 && kTrunkThreads == DT * TT / 2, "conv thread map");
    const int co = tid % DT, t0 = tid / DT, t1 = t0 + TT / 2;
    float acc0 = cb[co], acc1 = acc0;
#pragma unroll
    for (int tap = 0; tap < KT; ++tap) {
      const int s0 = t0 + tap - KT / 2, s1 = t1 + tap - KT / 2;
      const bool v0 = s0 >= 0, v1 = s1 < TT;        // s0 < TT and s1 >= 0 always hold
      const float4* l0 = (const float4*)(locs + (v0 ? s0 : 0) * DT);
      const float4* l1 = (const float4*)(locs + (v1 ? s1 : 0) * DT);
      const float* kc = ck + tap * DT * DT + co;
      float p0 = 0.f, p1 = 0.f;
#pragma unroll
      for (int c4 = 0; c4 < DT / 4; ++c4) {
        const float4 a = l0[c4], bq = l1[c4];
        const float k0 = kc[(4 * c4) * DT], k1 = kc[(4 * c4 + 1) * DT];
        const float k2 = kc[(4 * c4 + 2) * DT], k3 = kc[(4 * c4 + 3) * DT];
        p0 += a.x * k0; p0 += a.y * k1; p0 += a.z * k2; p0 += a.w * k3;
        p1 += bq.x * k0; p1 += bq.y * k1; p1 += bq.z * k2; p1 += bq.w * k3;
      }
      if (v0) acc0 += p0;
      if (v1) acc1 += p1;
    }
    M.a.conv_pre[rH + t0 * DT + co] = acc0;
    M.a.h_l[rH + t0 * DT + co] = gelu_f(acc0);
    M.a.conv_pre[rH + t1 * DT + co] = acc1;
    M.a.h_l[rH + t1 * DT + co] = gelu_f(acc1);
  } else {
  for (int j = tid; j < d.H; j += blockDim.x) {
    const int t = j / d.D, co = j % d.D;
    float acc = cb[co];
    for (int tap = 0; tap < d.K; ++tap) {
      const int s = t + tap - pad;
      if (s < 0 || s >= d.T) continue;
      float part = 0.f;
      const float* lrow = locs + s * d.D;
      const float* kc = ck + tap * d.D * d.D + co;
      for (int ci = 0; ci < d.D; ++ci) part += lrow[ci] * kc[ci * d.D];
      acc += part;
    }
    M.a.conv_pre[rH + j] = acc;
    M.a.h_l[rH + j] = gelu_f(acc);
  }
  }
  }   // local stream
  __syncthreads();   // the next row reuses every smem row buffer
  }   // rows of this CTA
}

void launch_trunk_fwd(const ModelPtrs& M, const uint8_t* src, long long ld_src, int use_col,
                      cudaStream_t s) {
  const Dims& d = M.d;
  if (row_warp_enabled(d.B, 6) && launch_trunk_fwd_w(M, src, ld_src, use_col, s)) return;
  const size_t smem = sizeof(float) * (3 * d.H + (2 + d.K) * d.D * d.D + d.D + 2 * d.T + 32) +
                      sizeof(int) * d.T;
  // + the staged cache tail when the cache rolls (a ring buffer moves nothing)
  const size_t smem_dt = smem + 16 + (M.ring_on ? 0 : sizeof(float) * (d.C - d.D));
  if (d.D == 32 && d.T == 16 && d.K == 3 && smem_dt <= 56 * 1024) {
    static const cudaError_t attr = cudaFuncSetAttribute(
        k_trunk_fwd<32, 16, 3>, cudaFuncAttributeMaxDynamicSharedMemorySize, 56 * 1024);
    (void)attr;
    launch_pdl(k_trunk_fwd<32, 16, 3>, dim3(M.trunk_grid), dim3(kTrunkThreads), smem_dt, s, M, src,
               ld_src, use_col);
  } else {
    launch_pdl(k_trunk_fwd<0, 0, 0>, dim3(M.trunk_grid), dim3(kTrunkThreads), smem, s, M, src, ld_src,
               use_col);
  }
}

// ---------------------------------------------------------------------------
// global stream finish + router + mixer LayerNorm (model.py:128-153)
__global__ void __launch_bounds__(kRowMax, 4) k_mix_fwd(ModelPtrs M) {
  pdl_enter();
  const Dims d = M.d;
  const int b = blockIdx.x, tid = threadIdx.x;
  extern __shared__ float sm[];
  float* hm = sm;            // h_mix row
  float* red = hm + d.H;
  float* ups = red + 32;     // [H] reduced W_mem pre-activation
  float* part = ups + d.H;   // [4][H]
  const long long rH = (long long)b * d.H;
  const long long plane = (long long)d.B * d.H;
  const float lam = M.w[P_LAM_MEM].p[0];
  const VFlags vf = vflags(M.variant);
  // count this step's roll of the ring-buffer cache: trunk_fwd wrote the new
  // block at the old position and the forward W_mem GEMM (ring_bias 1) has
  // read; no other kernel of this grid reads the position
  if (ring_cache(M) && b == 0 && tid == 0) M.st->ring += 1;
  if (vf.global) split_row(ups, part, M.a.ws_mem, plane, rH, d.H, M.splits_mem);
  float asum = 0.f, amin = 3.4e38f, amax = -3.4e38f;
  for (int j = tid; j < d.H; j += blockDim.x) {
    float hg = 0.f, hmx;
    if (vf.global) {
      const float up = ups[j];
      hg = gelu_f(up) + M.a.x[rH + j] * lam;
      M.a.upre[rH + j] = up;
      M.a.h_g[rH + j] = hg;
    }
    if (vf.router) {
      const float al = sigmoid_f(sk_sum(M.sk[S_RPRE], plane, rH + j));
      hmx = al * hg + (1.0f - al) * M.a.h_l[rH + j];
      M.a.alpha[rH + j] = al;
      asum += al;
      amin = fminf(amin, al);
      amax = fmaxf(amax, al);
    } else {
      hmx = vf.global ? hg : M.a.h_l[rH + j];   // single-stream variants
    }
    M.a.h_mix[rH + j] = hmx;
    M.a.hm_tc[rH + j] = tf32_rne(hmx);
    hm[j] = hmx;
  }
  __syncthreads();
  // router statistics for the metrics tape (model.py:197-199)
  if (vf.router) {
    const float s = block_sum_rt(asum, red);
    float mn = warp_max(-amin), mx = warp_max(amax);
    __shared__ float rmn[32], rmx[32];
    if ((tid & 31) == 0) { rmn[tid >> 5] = mn; rmx[tid >> 5] = mx; }
    __syncthreads();
    if (tid == 0) {
      float a = rmn[0], c = rmx[0];
      for (int w = 1; w < (int)(blockDim.x >> 5); ++w) { a = fmaxf(a, rmn[w]); c = fmaxf(c, rmx[w]); }
      M.a.alpha_row[3 * b + 0] = s;
      M.a.alpha_row[3 * b + 1] = -a;
      M.a.alpha_row[3 * b + 2] = c;
    }
  }
  if (!vf.mixer) return;
  float mu, inv;
  ln_stats(hm, d.H, red, &mu, &inv);
  const float* g = M.w[P_MIX_LN_G].p;
  const float* bb = M.w[P_MIX_LN_B].p;
  for (int j = tid; j < d.H; j += blockDim.x) {
    const float zh = (hm[j] - mu) * inv;
    M.a.z_hat[rH + j] = zh;
    M.a.z[rH + j] = tf32_rne(zh * g[j] + bb[j]);
  }
  if (tid == 0) M.a.z_inv[b] = inv;
}

void launch_mix_fwd(const ModelPtrs& M, cudaStream_t s) {
  if (row_warp_enabled(M.d.B, 0) && launch_mix_fwd_w(M, s)) return;
  launch_pdl(k_mix_fwd, dim3(M.d.B), dim3(row_threads(M.d.H)), sizeof(float) * (6 * M.d.H + 32), s,
             M);
}

// per-stream persistent memory: u[b] = zd[b] @ W_U[b]  (ops.py:44-54)
// One CTA per stream: lanes cover 4 consecutive columns (float4, a warp reads
// whole 512-byte rows of W_U), the 8 warps each sum a contiguous 1/8 of the
// rows with 8 row loads in flight -- the 33.5 MB W_U read is HBM-bound --
// and the warp partials combine in a fixed order.
constexpr int kBmmFwdWarps = 8;
__global__ void __launch_bounds__(32 * kBmmFwdWarps, 4) k_bmm_fwd(ModelPtrs M) {
  pdl_enter();
  const int X = M.d.X, b = blockIdx.x;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  extern __shared__ float zs[];                 // [X] zd row, then [8][X] partial rows
  float* part = zs + X;
  const long long plane = (long long)M.d.B * X;
  for (int i = threadIdx.x; i < X; i += blockDim.x) {
    const float v = sk_sum(M.sk[S_ZD], plane, (long long)b * X + i);
    zs[i] = v;
    M.a.zd[(long long)b * X + i] = v;             // kept for the W_U gradient
  }
  __syncthreads();
  const int per = (X + kBmmFwdWarps - 1) / kBmmFwdWarps;
  const int i0 = w * per, i1 = min(X, i0 + per);
  const int X4 = X / 4;                           // X % 4 == 0 (ModelConfig.device_check)
  const float4* W = (const float4*)(M.w[P_W_MIX].p + (long long)b * X * X);
  for (int j4 = lane; j4 < X4; j4 += 32) {
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll 8
    for (int i = i0; i < i1; ++i) {
      const float z = zs[i];
      const float4 w4 = W[(long long)i * X4 + j4];
      acc.x += z * w4.x;
      acc.y += z * w4.y;
      acc.z += z * w4.z;
      acc.w += z * w4.w;
    }
    *(float4*)(part + w * X + 4 * j4) = acc;
  }
  __syncthreads();
  for (int o = threadIdx.x; o < X; o += blockDim.x) {
    float u = 0.f;
#pragma unroll
    for (int k = 0; k < kBmmFwdWarps; ++k) u += part[k * X + o];
    M.a.u[(long long)b * X + o] = tf32_rne(u);
  }
}

void launch_bmm_fwd(const ModelPtrs& M, cudaStream_t s) {
  launch_pdl(k_bmm_fwd, dim3(M.d.B), dim3(32 * kBmmFwdWarps),
             sizeof(float) * M.d.X * (1 + kBmmFwdWarps), s, M);
}

// self-gated coarse refiner + FNR LayerNorm (model.py:156-167)
__global__ void __launch_bounds__(kRowMax, 4) k_coarse_fwd(ModelPtrs M) {
  pdl_enter();
  const Dims d = M.d;
  const int b = blockIdx.x, tid = threadIdx.x;
  extern __shared__ float sm[];
  float* hc = sm;
  float* red = hc + d.H;
  const long long rH = (long long)b * d.H;
  const float lam = M.w[P_LAM_MIX].p[0];
  const long long plane = (long long)d.B * d.H;
  const VFlags vf = vflags(M.variant);
  for (int j = tid; j < d.H; j += blockDim.x) {
    // mixer_nogate: inner + skip (inner * 1 is exact)
    const float gt = vf.gate ? sigmoid_f(sk_sum(M.sk[S_CPRE], plane, rH + j)) : 1.0f;
    const float in = sk_sum(M.sk[S_INNER], plane, rH + j);
    const float v = in * gt + M.a.h_mix[rH + j] * lam;
    M.a.inner[rH + j] = in;
    M.a.gate[rH + j] = gt;
    M.a.h_c[rH + j] = v;
    hc[j] = v;
  }
  if (!vf.fnr) return;
  __syncthreads();
  float mu, inv;
  ln_stats(hc, d.H, red, &mu, &inv);
  const float* g = M.w[P_REF_LN_G].p;
  const float* bb = M.w[P_REF_LN_B].p;
  for (int j = tid; j < d.H; j += blockDim.x) {
    const float zh = (hc[j] - mu) * inv;
    M.a.z2_hat[rH + j] = zh;
    M.a.z2[rH + j] = tf32_rne(zh * g[j] + bb[j]);
  }
  if (tid == 0) M.a.z2_inv[b] = inv;
}

void launch_coarse_fwd(const ModelPtrs& M, cudaStream_t s) {
  if (row_warp_enabled(M.d.B, 1) && launch_coarse_fwd_w(M, s)) return;
  launch_pdl(k_coarse_fwd, dim3(M.d.B), dim3(row_threads(M.d.H)), sizeof(float) * (M.d.H + 32), s, M);
}

// FNR output: split-K reduce, LayerNorm, gelu, residual (model.py:170-172)
__global__ void __launch_bounds__(kRowMax, 4) k_out_fwd(ModelPtrs M) {
  pdl_enter();
  const Dims d = M.d;
  const int b = blockIdx.x, tid = threadIdx.x;
  extern __shared__ float sm[];
  float* np_ = sm;
  float* red = np_ + d.H;
  float* part = red + 32;                 // [4][H]
  const long long rH = (long long)b * d.H;
  const long long plane = (long long)d.B * d.H;
  split_row(np_, part, M.a.ws_f, plane, rH, d.H, M.splits_f);
  float mu, inv;
  ln_stats(np_, d.H, red, &mu, &inv);
  const float* g = M.w[P_OUT_LN_G].p;
  const float* bb = M.w[P_OUT_LN_B].p;
  const float lam = M.w[P_LAM_OUT].p[0];
  for (int j = tid; j < d.H; j += blockDim.x) {
    const float nh = (np_[j] - mu) * inv;
    const float nv = nh * g[j] + bb[j];
    M.a.n_hat[rH + j] = nh;
    M.a.nrm[rH + j] = nv;
    M.a.h[rH + j] = tf32_rne(gelu_f(nv) + M.a.h_c[rH + j] * lam);
  }
  if (tid == 0) M.a.n_inv[b] = inv;
}

void launch_out_fwd(const ModelPtrs& M, cudaStream_t s) {
  if (row_warp_enabled(M.d.B, 2) && launch_out_fwd_w(M, s)) return;
  launch_pdl(k_out_fwd, dim3(M.d.B), dim3(row_threads(M.d.H)), sizeof(float) * (5 * M.d.H + 32), s,
             M);
}

// ---------------------------------------------------------------------------
// head: fp64 softmax (ops.py:246-255) -> quantiser (kernels.py:48-85) ->
// cumulative table (coder.py:37-43) -> [decode] -> softmax-xent (ops.py:258-279)
__device__ __forceinline__ void record_error(StepState* st, long long step, long long stream,
                                             int code) {
  // lowest step first, then lowest stream; code 1/2 corrupt(why), 3 diverged,
  // 4 quantiser, 5 non-finite loss
  const unsigned long long key = ((unsigned long long)step << 24) |
                                 ((unsigned long long)stream << 3) | (unsigned long long)code;
  atomicMin((unsigned long long*)&st->err_key, key);
}

__device__ __forceinline__ double block_sum_d256(double v, double* red) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  v = warp_sum_d(v);
  if (lane == 0) red[w] = v;
  __syncthreads();
  double t = lane < 8 ? red[lane] : 0.0;
#pragma unroll
  for (int o = 4; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
  t = __shfl_sync(0xffffffffu, t, 0);
  __syncthreads();
  return t;
}

__device__ void adam_prep_dev(StepState* st, double lr, double b1, double b2, double eps);

// After a divergence or quantiser failure the graph keeps replaying the
// remaining timesteps (the host reads the error once, at the end), so the
// failing row's table slot gets the uniform table (coder.py:46-49): the
// encoder downstream then codes a well-formed interval instead of reading a
// stale or zero-width slot.  The run's result is the recorded error.
__device__ __forceinline__ void write_uniform_cum(unsigned* cum) {
  const int i = threadIdx.x;
  cum[i] = (unsigned)i * 256u;
  if (i == kAlphabet - 1) cum[kAlphabet] = kTotal;
}

// fp64 softmax of one 256-logit row, thread i = symbol i: row max in float
// (exact), z = logit - max in f64, p = exp(z) / sum.  The head kernel and the
// coder-stream quantiser (k_head_quant) both use this exact sequence, so the
// encoder's tables equal the decoder's bit for bit.
__device__ __forceinline__ double row_softmax(float lg, float* fred, double* dred, double* zo,
                                              double* so) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  float mx = warp_max(lg);
  if (lane == 0) fred[w] = mx;
  __syncthreads();
  mx = fred[0];
  for (int k = 1; k < 8; ++k) mx = fmaxf(mx, fred[k]);
  const double z = (double)lg - (double)mx;
  const double e = exp(z);
  const double s = block_sum_d256(e, dred);
  *zo = z;
  *so = s;
  return e / s;
}

__global__ void __launch_bounds__(256) k_head(ModelPtrs M, HeadArgs H) {
  pdl_enter();
  __shared__ QuantSmem qs;
  __shared__ double dred[8];
  __shared__ unsigned cum_s[kAlphabet + 1];
  __shared__ int wsum[8];
  __shared__ int sym_s;
  __shared__ int bad_s;
  const int b = blockIdx.x, i = threadIdx.x;
  StepState* st = M.st;
  const long long col = st->col;
  if (i == 0) bad_s = 0;
  const float lg = sk_sum<8>(M.sk[S_LOGITS], (long long)M.d.B * kAlphabet, (long long)b * kAlphabet + i);
  M.a.logits[(long long)b * kAlphabet + i] = lg;
  __syncthreads();
  if (!isfinite(lg)) atomicOr(&bad_s, 1);
  __syncthreads();
  if (H.adam_prep && b == 0 && i == 0)
    adam_prep_dev(st, M.lr, M.beta1, M.beta2, M.adam_eps);
  if (bad_s) {
    if (i == 0) record_error(st, col, b, 3);
    if (!H.skip_quant) write_uniform_cum(M.a.cum + ((col & 1) * (long long)M.d.B + b) * kCumLd);
    return;
  }
  __shared__ float fred[8];
  double z, s;
  const double p = row_softmax(lg, fred, dred, &z, &s);
  if (H.want_probs) M.a.probs[(long long)b * kAlphabet + i] = p;
  if (!H.skip_quant) {
    bool qbad;
    const int f = quantize_sym(p, qs, &qbad);
    unsigned* cum = M.a.cum + ((col & 1) * (long long)M.d.B + b) * kCumLd;
    if (qbad) {
      if (i == 0) record_error(st, col, b, 4);
      write_uniform_cum(cum);
      return;
    }
    const int c = block_excl_scan256(f, wsum);
    cum[i] = (unsigned)c;
    cum_s[i] = (unsigned)c;
    if (i == kAlphabet - 1) {
      cum[kAlphabet] = kTotal;
      cum_s[kAlphabet] = kTotal;
    }
    __syncthreads();
    if (M.tape && i == 0) atomicMax(tape_at(M, 1), gtimer_ns());
  }
  if (!H.xent) return;
  int tgt;
  if (H.decode) {
    if (i == 0) {
      DecLane ln{H.dcode[b], H.drng[b], H.dpos[b]};
      int sy = 0;
      const int why = dec_symbol(ln, cum_s, H.payload + H.off[b], H.dlen[b], &sy);
      if (why) {
        record_error(st, col, b, why);
        sy = 0;
      } else {
        H.dcode[b] = ln.code;
        H.drng[b] = ln.rng;
        H.dpos[b] = ln.pos;
      }
      H.out[(long long)b * H.ld_out + col] = (uint8_t)sy;
      sym_s = sy;
      if (M.tape) {
        // the decoder drains the table inside this kernel
        if (b == 0) *tape_at(M, 2) = gtimer_ns();
        atomicMax(tape_at(M, 3), gtimer_ns());
      }
    }
    __syncthreads();
    tgt = sym_s;
  } else {
    tgt = H.tgt[(long long)b * H.ld_tgt + (H.tgt_use_col ? col : 0)];
  }
  // softmax_xent in f64: logp = z - log(sum exp z); grad = (p - onehot) / B
  const double lse = log(s);
  const double logp = z - lse;
  double dgrad = exp(logp);
  if (i == tgt) {
    M.a.nll[b] = -logp;
    dgrad -= 1.0;
  }
  dgrad *= 1.0 / (double)M.d.B;
  M.a.dlogits[(long long)b * kAlphabet + i] = (float)dgrad;
}

void launch_head(const ModelPtrs& M, const HeadArgs& h, cudaStream_t s) {
  launch_pdl(k_head, dim3(M.d.B), dim3(256), 0, s, M, h);
}

// Compression's quantiser + cumulative table on the coder stream (CSPP): the
// head kernel (skip_quant) emits the logits and the loss gradient only, so
// the backward starts without waiting for the quantiser; this kernel
// recomputes the row's softmax from the logits with the head's own sequence
// and writes the table slot of the coder's column (*colp) for k_encode_col.
__global__ void __launch_bounds__(256) k_head_quant(ModelPtrs M, const long long* colp) {
  pdl_enter();
  __shared__ QuantSmem qs;
  __shared__ double dred[8];
  __shared__ float fred[8];
  __shared__ int wsum[8];
  __shared__ int bad_s;
  const int b = blockIdx.x, i = threadIdx.x;
  const long long col = *colp;
  if (i == 0) bad_s = 0;
  const float lg = M.a.logits[(long long)b * kAlphabet + i];
  __syncthreads();
  if (!isfinite(lg)) atomicOr(&bad_s, 1);
  __syncthreads();
  unsigned* cum = M.a.cum + ((col & 1) * (long long)M.d.B + b) * kCumLd;
  if (bad_s) {            // the head kernel has recorded the divergence
    write_uniform_cum(cum);
    return;
  }
  double z, s;
  const double p = row_softmax(lg, fred, dred, &z, &s);
  bool qbad;
  const int f = quantize_sym(p, qs, &qbad);
  if (qbad) {
    if (i == 0) record_error(M.st, col, b, 4);
    write_uniform_cum(cum);
    return;
  }
  const int c = block_excl_scan256(f, wsum);
  cum[i] = (unsigned)c;
  if (i == kAlphabet - 1) cum[kAlphabet] = kTotal;
  if (M.tape && i == 0) atomicMax(M.tape + kTapeSlots * (col - M.st->loss_base) + 1, gtimer_ns());
}

void launch_head_quant(const ModelPtrs& M, const long long* colp, cudaStream_t s) {
  launch_pdl(k_head_quant, dim3(M.d.B), dim3(256), 0, s, M, colp);
}

// Adam bias-correction scalars from the device step counter (optim.py:26-30);
// run by one thread of the head kernel of every training step
__device__ void adam_prep_dev(StepState* st, double lr, double b1, double b2, double eps) {
  const long long t = ++st->adam_t;
  const double c1 = 1.0 - pow(b1, (double)t);
  const double c2 = 1.0 - pow(b2, (double)t);
  AdamScalars a;
  a.beta1 = (float)b1;
  a.beta2 = (float)b2;
  a.one_m_b1 = (float)(1.0 - b1);
  a.one_m_b2 = (float)(1.0 - b2);
  a.eps = (float)eps;
  a.step_size = (float)(lr / c1);
  a.inv_sqrt_c2 = 1.0 / sqrt(c2);
  st->adam = a;
}


__device__ __forceinline__ void adam_update(const AdamScalars& a, float g, float* p, float* m,
                                            float* v) {
  const float m1 = fadd_ftz(fmul_ftz(*m, a.beta1), fmul_ftz(a.one_m_b1, g));
  const float v1 = fadd_ftz(fmul_ftz(*v, a.beta2), fmul_ftz(a.one_m_b2, fmul_ftz(g, g)));
  float sc = (float)__dmul_rn((double)fsqrt_fastpath(v1), a.inv_sqrt_c2);
  sc = __fadd_rn(sc, a.eps);
  sc = __fmul_rn(fdiv_fastpath(m1, sc), a.step_size);
  *m = m1;
  *v = v1;
  *p = __fsub_rn(*p, sc);
}

// ---------------------------------------------------------------------------
// backward row kernels

// h = gelu(LN(npre)) + lam_out * h_c   (model.py:170-172 backward)
__global__ void __launch_bounds__(kRowMax, 4) k_out_bwd(ModelPtrs M) {
  pdl_enter();
  const Dims d = M.d;
  const int b = blockIdx.x, tid = threadIdx.x;
  extern __shared__ float sm[];
  float* dn = sm;
  float* red = dn + d.H;
  const long long rH = (long long)b * d.H;
  float* rr = M.a.rowred + (long long)b * M.sl.rowred;
  const float lam = M.w[P_LAM_OUT].p[0];
  float lsum = 0.f;
  const long long plane = (long long)d.B * d.H;
  for (int j = tid; j < d.H; j += blockDim.x) {
    const float dh = sk_sum(M.sk[S_DH], plane, rH + j);
    const float v = dh * gelu_grad_f(M.a.nrm[rH + j]);
    dn[j] = v;
    rr[M.sl.out_g + j] = v * M.a.n_hat[rH + j];
    rr[M.sl.out_b + j] = v;
    lsum += dh * M.a.h_c[rH + j];
    M.a.dhc[rH + j] = dh * lam;
  }
  __syncthreads();
  const float ls = block_sum_rt(lsum, red);
  if (tid == 0) rr[M.sl.lam_out] = ls;
  float m1, m2;
  const float* g = M.w[P_OUT_LN_G].p;
  ln_bwd_means(dn, M.a.n_hat + rH, g, d.H, red, &m1, &m2);
  const float inv = M.a.n_inv[b];
  for (int j = tid; j < d.H; j += blockDim.x)
    M.a.dnpre[rH + j] = (dn[j] * g[j] - m1 - M.a.n_hat[rH + j] * m2) * inv;
}

void launch_out_bwd(const ModelPtrs& M, cudaStream_t s) {
  if (row_warp_enabled(M.d.B, 3) && launch_out_bwd_w(M, s)) return;
  launch_pdl(k_out_bwd, dim3(M.d.B), dim3(row_threads(M.d.H)), sizeof(float) * (M.d.H + 32), s, M);
}

// z2 = LN(h_c); h_c = inner * sigmoid(cpre) + lam_mix * h_mix   (backward)
__global__ void __launch_bounds__(kRowMax, 4) k_coarse_bwd(ModelPtrs M) {
  pdl_enter();
  const Dims d = M.d;
  const int b = blockIdx.x, tid = threadIdx.x;
  extern __shared__ float sm[];
  float* dz = sm;
  float* red = dz + d.H;
  float* part = red + 32;    // [4][H]
  const long long rH = (long long)b * d.H;
  const long long plane = (long long)d.B * d.H;
  float* rr = M.a.rowred + (long long)b * M.sl.rowred;
  const VFlags vf = vflags(M.variant);
  float m1 = 0.f, m2 = 0.f, inv = 0.f;
  const float* g = M.w[P_REF_LN_G].p;
  if (vf.fnr) {
    split_row(dz, part, M.a.ws_dz2, plane, rH, d.H, M.splits_dz2);
    for (int j = tid; j < d.H; j += blockDim.x) {
      const float acc = dz[j];
      rr[M.sl.ref_g + j] = acc * M.a.z2_hat[rH + j];
      rr[M.sl.ref_b + j] = acc;
    }
    ln_bwd_means(dz, M.a.z2_hat + rH, g, d.H, red, &m1, &m2);
    inv = M.a.z2_inv[b];
  }
  float lsum = 0.f;
  for (int j = tid; j < d.H; j += blockDim.x) {
    // without the FNR, h = h_coarse and dh arrives straight from the head GEMM
    const float dhc = vf.fnr ? M.a.dhc[rH + j] + (dz[j] * g[j] - m1 - M.a.z2_hat[rH + j] * m2) * inv
                             : sk_sum(M.sk[S_DH], plane, rH + j);
    const float gt = M.a.gate[rH + j];
    M.a.dhc[rH + j] = dhc;
    M.a.dinner[rH + j] = dhc * gt;
    if (vf.gate) M.a.dcpre[rH + j] = dhc * M.a.inner[rH + j] * gt * (1.0f - gt);
    lsum += dhc * M.a.h_mix[rH + j];
  }
  const float ls = block_sum_rt(lsum, red);
  if (tid == 0) rr[M.sl.lam_mix] = ls;
}

void launch_coarse_bwd(const ModelPtrs& M, cudaStream_t s) {
  if (row_warp_enabled(M.d.B, 4) && launch_coarse_bwd_w(M, s)) return;
  launch_pdl(k_coarse_bwd, dim3(M.d.B), dim3(row_threads(M.d.H)), sizeof(float) * (5 * M.d.H + 32),
             s, M);
}

// per-stream memory backward + its Adam step in one streaming pass
// (ops.py:48-52 for the gradients, optim.py:25-44 for the update)
// mode bit 0: input gradient dzd (reads W_U once -- the model stream's part);
// mode bit 1: W_U gradient + Adam (the 24 B/param RMW -- run on the side
// stream after the input gradient has read the old W_U)
__device__ __forceinline__ void bulk_load(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void bulk_store(void* dst, const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst),
               "r"(smem_u32(src)), "r"(bytes)
               : "memory");
}

// smem of the bulk-copy fast path: du [128], zd [32], barrier (< 1 KB), then
// the p/m/v tiles at byte 1024
constexpr int kBmmTileBytes = kBmmRows * 128 * 4;     // kBmmRows rows x X = 128 floats
constexpr int kBmmFastSmem = 1024 + 3 * kBmmTileBytes;

// FAST: the default-geometry training path (X = 128, fused W_U Adam), compiled
// on its own at <= 64 registers so eight CTAs share an SM (-2.5 us per
// timestep against five); the generic path keeps its own allocation
template <bool FAST>
__global__ void __launch_bounds__(kBmmThreads, FAST ? 8 : 1) k_bmm_bwd(ModelPtrs M, int grad_only, int mode) {
  const int X = M.d.X, b = blockIdx.x;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  extern __shared__ float sm[];
  float* dus = sm;          // [X]
  float* zds = sm + X;      // [X]
  const int i0 = blockIdx.y * kBmmRows, i1 = min(X, i0 + kBmmRows);
  const long long base = (long long)b * X * X;
  const bool do_dx = mode & 1, do_upd = mode & 2;
  if constexpr (FAST) {
    // default geometry, training path: this CTA's kBmmRows rows of W_U p, m, v
    // are three contiguous blocks, pulled into smem by bulk copies issued
    // BEFORE the dependency wait (no kernel of this step writes W_U before
    // us; the previous step's update finished at the graph boundary), so the
    // HBM reads overlap the tail of the du GEMM; updated in place, written
    // back by bulk copies
    // two halves, each with its own barrier: half 0 is updated and streamed
    // back while half 1 is still landing
    uint64_t* bar = (uint64_t*)(sm + X + kBmmRows);     // [2], after du [X] and zd [kBmmRows]
    float* tile = (float*)((char*)sm + 1024);           // [3][kBmmRows][X]: p, m, v
    constexpr int kHalf = kBmmRows / 2;
    const int nrows = i1 - i0;
    auto rows_of = [&](int h) { return max(0, min(kHalf, nrows - h * kHalf)); };
    const long long off = base + (long long)i0 * X;
    float* const gsrc[3] = {M.w[P_W_MIX].p + off, M.w[P_W_MIX].m + off, M.w[P_W_MIX].v + off};
    if (threadIdx.x == 0) {
      mbar_init(&bar[0], 1);
      mbar_init(&bar[1], 1);
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
      for (int h = 0; h < 2; ++h) {
        const uint32_t bytes = (uint32_t)rows_of(h) * X * 4;
        if (!bytes) continue;
        mbar_expect_tx(&bar[h], 3 * bytes);
        for (int t = 0; t < 3; ++t)
          bulk_load(tile + t * kBmmRows * X + h * kHalf * X, gsrc[t] + h * kHalf * X, bytes, &bar[h]);
      }
    }
    pdl_enter();
    for (int i = threadIdx.x; i < X; i += blockDim.x)
      dus[i] = sk_sum(M.sk[S_DU], (long long)M.d.B * X, (long long)b * X + i);
    for (int i = i0 + threadIdx.x; i < i1; i += blockDim.x) zds[i - i0] = M.a.zd[(long long)b * X + i];
    __syncthreads();
    const AdamScalars a = M.st->adam;
    const float4 du4 = *(const float4*)(dus + 4 * lane);
    constexpr int kWarps = kBmmThreads / 32;
    float4* tp = (float4*)tile;
    float4* tm = (float4*)(tile + kBmmRows * X);
    float4* tv = (float4*)(tile + 2 * kBmmRows * X);
    for (int h = 0; h < 2; ++h) {
      const int nr = rows_of(h);
      if (!nr) break;
      mbar_wait(&bar[h], 0);
      for (int r = h * kHalf + w; r < h * kHalf + nr; r += kWarps) {
        const int q = r * 32 + lane;
        float4 p = tp[q], mm = tm[q], v = tv[q];
        const float acc = du4.x * p.x + du4.y * p.y + du4.z * p.z + du4.w * p.w;
        const float zi = zds[r];
        adam_update(a, zi * du4.x, &p.x, &mm.x, &v.x);
        adam_update(a, zi * du4.y, &p.y, &mm.y, &v.y);
        adam_update(a, zi * du4.z, &p.z, &mm.z, &v.z);
        adam_update(a, zi * du4.w, &p.w, &mm.w, &v.w);
        tp[q] = p;
        tm[q] = mm;
        tv[q] = v;
        if (do_dx) {
          const float s = warp_sum(acc);
          if (lane == 0) M.a.dzd[(long long)b * X + i0 + r] = s;
        }
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncthreads();
      if (threadIdx.x == 0) {
        const uint32_t bytes = (uint32_t)nr * X * 4;
        for (int t = 0; t < 3; ++t)
          bulk_store(gsrc[t] + h * kHalf * X, tile + t * kBmmRows * X + h * kHalf * X, bytes);
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      }
    }
    if (threadIdx.x == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
    return;
  } else {
  pdl_enter();
  for (int i = threadIdx.x; i < X; i += blockDim.x)
    dus[i] = sk_sum(M.sk[S_DU], (long long)M.d.B * X, (long long)b * X + i);
  for (int i = i0 + threadIdx.x; i < i1; i += blockDim.x) zds[i - i0] = M.a.zd[(long long)b * X + i];
  __syncthreads();
  float4* __restrict__ Wp = (float4*)(M.w[P_W_MIX].p + base);
  float4* __restrict__ Wm = (float4*)(M.w[P_W_MIX].m + base);
  float4* __restrict__ Wv = (float4*)(M.w[P_W_MIX].v + base);
  float4* __restrict__ Wg = (float4*)(M.w[P_W_MIX].g + base);
  const AdamScalars a = M.st->adam;
  const int X4 = X / 4;      // X is a multiple of 4 (ModelConfig.device_check)
  (void)do_dx;
  // one warp per row i; lanes cover 4 consecutive columns each (float4), so
  // the read-modify-write of p, m, v is one coalesced 512-byte pass per row.
  // A CTA owns kBmmRows rows of one stream: 4x more CTAs than streams keeps
  // the HBM-bound RMW evenly spread over the 148 SMs.
  constexpr int kWarps = kBmmThreads / 32;
  if (X4 == 32 && do_upd && !grad_only) {
    // default geometry (X = 128: one float4 per lane per row), the training
    // path: a warp takes R rows at a time and issues all 3R loads before any
    // Adam arithmetic, so the HBM round trips overlap instead of serialising
    constexpr int R = 4;
    const float4 du4 = *(const float4*)(dus + 4 * lane);
    for (int kb = 0; i0 + w + kb * kWarps < i1; kb += R) {
      float4 P[R], Mm[R], V[R];
#pragma unroll
      for (int k = 0; k < R; ++k) {
        const int i = i0 + w + (kb + k) * kWarps;
        if (i < i1) {
          const long long q = (long long)i * 32 + lane;
          P[k] = Wp[q];
          Mm[k] = Wm[q];
          V[k] = Wv[q];
        }
      }
#pragma unroll
      for (int k = 0; k < R; ++k) {
        const int i = i0 + w + (kb + k) * kWarps;
        if (i >= i1) continue;
        float4 p = P[k];
        float acc = du4.x * p.x + du4.y * p.y + du4.z * p.z + du4.w * p.w;
        const float zi = zds[i - i0];
        adam_update(a, zi * du4.x, &p.x, &Mm[k].x, &V[k].x);
        adam_update(a, zi * du4.y, &p.y, &Mm[k].y, &V[k].y);
        adam_update(a, zi * du4.z, &p.z, &Mm[k].z, &V[k].z);
        adam_update(a, zi * du4.w, &p.w, &Mm[k].w, &V[k].w);
        const long long q = (long long)i * 32 + lane;
        Wp[q] = p;
        Wm[q] = Mm[k];
        Wv[q] = V[k];
        if (do_dx) {
          acc = warp_sum(acc);
          if (lane == 0) M.a.dzd[(long long)b * X + i] = acc;
        }
      }
    }
    return;
  }
#pragma unroll 4
  for (int i = i0 + w; i < i1; i += kBmmThreads / 32) {
    float acc = 0.f;
    const float zi = zds[i - i0];
    for (int j4 = lane; j4 < X4; j4 += 32) {
      const long long q = (long long)i * X4 + j4;
      float4 p = Wp[q];
      const float4 du4 = *(const float4*)(dus + 4 * j4);
      acc += du4.x * p.x + du4.y * p.y + du4.z * p.z + du4.w * p.w;
      const float4 g = make_float4(zi * du4.x, zi * du4.y, zi * du4.z, zi * du4.w);
      if (!do_upd) {
      } else if (grad_only) {
        Wg[q] = g;
      } else {
        float4 m = Wm[q], v = Wv[q];
        adam_update(a, g.x, &p.x, &m.x, &v.x);
        adam_update(a, g.y, &p.y, &m.y, &v.y);
        adam_update(a, g.z, &p.z, &m.z, &v.z);
        adam_update(a, g.w, &p.w, &m.w, &v.w);
        Wp[q] = p;
        Wm[q] = m;
        Wv[q] = v;
      }
    }
    if (do_dx) {
      acc = warp_sum(acc);
      if (lane == 0) M.a.dzd[(long long)b * X + i] = acc;
    }
  }
}  // generic path
}

void launch_bmm_bwd(const ModelPtrs& M, int grad_only, int mode, cudaStream_t s) {
  static const cudaError_t attr =
      cudaFuncSetAttribute(k_bmm_bwd<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, kBmmFastSmem);
  (void)attr;
  const bool fast = M.d.X == 128 && (mode & 2) && !grad_only;
  if (fast)
    launch_pdl(k_bmm_bwd<true>, dim3(M.d.B, cdiv(M.d.X, kBmmRows)), dim3(kBmmThreads),
               (size_t)kBmmFastSmem, s, M, grad_only, mode);
  else
    launch_pdl(k_bmm_bwd<false>, dim3(M.d.B, cdiv(M.d.X, kBmmRows)), dim3(kBmmThreads),
               sizeof(float) * (M.d.X + kBmmRows), s, M, grad_only, mode);
}

// mixer LayerNorm + router mix + global-stream gelu (model.py:128-153 backward)
__global__ void __launch_bounds__(kRowMax, 4) k_mix_bwd(ModelPtrs M) {
  pdl_enter();
  const Dims d = M.d;
  const int b = blockIdx.x, tid = threadIdx.x;
  extern __shared__ float sm[];
  float* dz = sm;
  float* red = dz + d.H;
  const long long rH = (long long)b * d.H;
  float* rr = M.a.rowred + (long long)b * M.sl.rowred;
  const long long plane = (long long)d.B * d.H;
  const VFlags vf = vflags(M.variant);
  float m1 = 0.f, m2 = 0.f, inv = 0.f;
  const float* g = M.w[P_MIX_LN_G].p;
  if (vf.mixer) {
    for (int j = tid; j < d.H; j += blockDim.x) {
      const float v = sk_sum(M.sk[S_DZ], plane, rH + j);
      dz[j] = v;
      rr[M.sl.mix_g + j] = v * M.a.z_hat[rH + j];
      rr[M.sl.mix_b + j] = v;
    }
    __syncthreads();
    ln_bwd_means(dz, M.a.z_hat + rH, g, d.H, red, &m1, &m2);
    inv = M.a.z_inv[b];
  }
  const float lam_mix = M.w[P_LAM_MIX].p[0];
  const float lam_mem = M.w[P_LAM_MEM].p[0];
  float lsum = 0.f;
  for (int j = tid; j < d.H; j += blockDim.x) {
    float dhm;
    if (vf.mixer) {
      const float dhmc = vf.gate ? sk_sum(M.sk[S_DHMC], plane, rH + j) : 0.f;
      dhm = M.a.dhc[rH + j] * lam_mix + dhmc + (dz[j] * g[j] - m1 - M.a.z_hat[rH + j] * m2) * inv;
    } else {
      dhm = sk_sum(M.sk[S_DH], plane, rH + j);   // h = h_mix
    }
    float dhg = dhm, dhl = dhm;
    if (vf.router) {
      const float al = M.a.alpha[rH + j];
      const float dal = dhm * (M.a.h_g[rH + j] - M.a.h_l[rH + j]);
      dhg = dhm * al;
      dhl = dhm * (1.0f - al);
      M.a.drpre[rH + j] = dal * al * (1.0f - al);
    }
    if (vf.local) M.a.dh_l[rH + j] = dhl;
    if (vf.global) {
      M.a.dupre[rH + j] = dhg * gelu_grad_f(M.a.upre[rH + j]);
      M.a.dx_part[rH + j] = dhg * lam_mem;
      lsum += dhg * M.a.x[rH + j];
    }
  }
  if (!vf.global) return;
  const float ls = block_sum_rt(lsum, red);
  if (tid == 0) rr[M.sl.lam_mem] = ls;
}

void launch_mix_bwd(const ModelPtrs& M, cudaStream_t s) {
  if (row_warp_enabled(M.d.B, 5) && launch_mix_bwd_w(M, s)) return;
  launch_pdl(k_mix_bwd, dim3(M.d.B), dim3(row_threads(M.d.H)), sizeof(float) * (M.d.H + 32), s, M);
}

// trunk + local stream backward (model.py:118-137 backward)
template <int DT, int TT, int KT>
__global__ void __launch_bounds__(kTrunkThreads, 4) k_trunk_bwd(ModelPtrs M, const uint8_t* src,
                                                       long long ld_src, int use_col) {
  pdl_enter();
  Dims d = M.d;
  if (DT) { d.D = DT; d.T = TT; d.K = KT; d.H = DT * TT; }
  const int tid = threadIdx.x;
  extern __shared__ float sm[];
  float* dxs = sm;                        // [H] dx, later dxf
  float* dcv = dxs + d.H;                 // [H] dconv
  float* locs = dcv + d.H;                // [H] LN_D(emb) (conv input)
  float* dls = locs + d.H;                // [H] dloc
  float* ck = dls + d.H;                  // [K*D][D+1]
  float* dg = ck + d.K * d.D * (d.D + 1); // [D] dgpre
  float* dv = dg + d.D;                   // [D] dvpre
  float* xt = dv + d.D;                   // [D]
  float* red = xt + d.D;                  // [32]
  float* xh = red + 32;                   // [H] x_hat (input LayerNorm)
  float* lhs = xh + d.H;                  // [H] loc_hat (per-symbol LayerNorm)
  float* lis = lhs + d.H;                 // [T] loc_inv
  int* ctx = (int*)(lis + ((d.T + 3) & ~3));   // [T] context symbols
  // per-CTA sums of this kernel's small-parameter gradient columns
  // [trunk0, trunk1) of the small arena (in_g ... w_val), accumulated over the
  // CTA's rows in row order and written once to trunk_part[blockIdx.x]; the
  // small-parameter kernel sums the gridDim.x partial rows in a fixed order
  // (one row per CTA -- B <= trunk grid -- writes its row straight to
  // trunk_part; several rows accumulate in shared memory first)
  const bool multi = d.B > (int)gridDim.x;
  const int t0 = M.sl.trunk0;
  float* acc = multi ? (float*)(ctx + ((d.T + 3) & ~3))
                     : M.a.trunk_part + (long long)blockIdx.x * (M.sl.trunk1 - t0);
  // rr[X + q] (a per-row column write of the CTA-per-row layout) becomes an
  // accumulate into this CTA's partial row; each column has one owner thread
#define RR_ADD(off, q, v) (multi ? (void)(acc[(off) - t0 + (q)] += (v)) : (void)(acc[(off) - t0 + (q)] = (v)))
  const float* Wg = M.w[P_W_GATE].p;
  const long long c0 = use_col ? M.st->col - d.T : 0;
  const float* Wv = M.w[P_W_VAL].p;
  // taps transposed to [tap][co][ci] with a padded row (D + 1) so both this
  // transposing store and the input-gradient loop below are bank-conflict free
  // (once per CTA: the rows below share them)
  const int ckp = d.D + 1;
  for (int j = tid; j < d.K * d.D * d.D; j += blockDim.x) {
    const int tap = j / (d.D * d.D), ci = (j / d.D) % d.D, co = j % d.D;
    ck[(tap * d.D + co) * ckp + ci] = M.w[P_CONV_K].p[j];
  }
  if (multi)
    for (int c = tid; c < M.sl.trunk1 - t0; c += blockDim.x) acc[c] = 0.f;
  const VFlags vf = vflags(M.variant);
  for (int b = blockIdx.x; b < d.B; b += gridDim.x) {
  const long long rH = (long long)b * d.H;
  // every global input of the row is loaded in this one round (the
  // LayerNorm phases below read x_hat / loc_hat / loc_inv from shared
  // memory instead of a dependent global round each)
  const float xinv = M.a.x_inv[b];
  for (int t = tid; t < d.T; t += blockDim.x) {
    ctx[t] = src[(long long)b * ld_src + c0 + t];
    if (vf.local) lis[t] = M.a.loc_inv[(long long)b * d.T + t];
  }
  if (vf.global) {
    for (int o = tid; o < d.D; o += blockDim.x) {
      const float gp = M.a.gpre[(long long)b * d.D + o];
      const float vp = M.a.vpre[(long long)b * d.D + o];
      const float db = sk_sum(M.sk[S_DBLOCK], (long long)d.B * d.D, (long long)b * d.D + o);
      dg[o] = db * vp * gelu_grad_f(gp);
      dv[o] = db * gelu_f(gp);
      xt[o] = M.a.x[rH + d.H - d.D + o];
    }
  }
  for (int j = tid; j < d.H; j += blockDim.x) {
    // dx: router (x W_route) + global skip (lam_mem x); zero in local_only
    float dx = 0.f;
    if (vf.router) dx = sk_sum(M.sk[S_DXR], (long long)d.B * d.H, rH + j);
    if (vf.global) dx = vf.router ? dx + M.a.dx_part[rH + j] : M.a.dx_part[rH + j];
    dxs[j] = dx;
    xh[j] = M.a.x_hat[rH + j];
    if (vf.local) {
      dcv[j] = M.a.dh_l[rH + j] * gelu_grad_f(M.a.conv_pre[rH + j]);
      locs[j] = M.a.loc[rH + j];
      lhs[j] = M.a.loc_hat[rH + j];
    }
  }
  __syncthreads();
  if (vf.global) {
    // W_gate / W_val gradients (outer products) and dx_t
    for (int q = tid; q < d.D * d.D; q += blockDim.x) {
      const int i = q / d.D, o = q % d.D;
      RR_ADD(M.sl.w_gate, q, xt[i] * dg[o]);
      RR_ADD(M.sl.w_val, q, xt[i] * dv[o]);
    }
    if constexpr (DT > 0) {
      // all 8 warps: warp w takes inputs i in [4w, 4w + 4), lane = output o
      // (coalesced weight rows), xor-tree sums -- instead of 32 threads each
      // walking 64 dependent loads while 7 warps wait at the barrier
      static_assert(kTrunkThreads / 32 * 4 == DT, "dx_t split");
      const int w = tid >> 5, o = tid & 31;
#pragma unroll
      for (int i = 4 * w; i < 4 * w + 4; ++i) {
        const float a1 = warp_sum(dg[o] * Wg[i * DT + o]);
        const float a2 = warp_sum(dv[o] * Wv[i * DT + o]);
        if (o == 0) dxs[d.H - DT + i] += a1 + a2;
      }
    } else {
      for (int i = tid; i < d.D; i += blockDim.x) {
        float a1 = 0.f, a2 = 0.f;
        for (int o = 0; o < d.D; ++o) {
          a1 += dg[o] * Wg[i * d.D + o];
          a2 += dv[o] * Wv[i * d.D + o];
        }
        dxs[d.H - d.D + i] += a1 + a2;
      }
    }
    __syncthreads();
  }
  // input LayerNorm backward
  const float* gin = M.w[P_IN_LN_G].p;
  for (int j = tid; j < d.H; j += blockDim.x) {
    RR_ADD(M.sl.in_g, j, dxs[j] * xh[j]);
    RR_ADD(M.sl.in_b, j, dxs[j]);
  }
  float m1, m2;
  ln_bwd_means(dxs, xh, gin, d.H, red, &m1, &m2);
  for (int j = tid; j < d.H; j += blockDim.x)
    dxs[j] = (dxs[j] * gin[j] - m1 - xh[j] * m2) * xinv;   // dxf
  if (vf.local) {
  // conv gradients: bias, taps, input (ops.py:74-88)
  const int pad = d.K / 2;
  for (int co = tid; co < d.D; co += blockDim.x) {
    float s = 0.f;
    for (int t = 0; t < d.T; ++t) s += dcv[t * d.D + co];
    RR_ADD(M.sl.conv_b, co, s);
  }
  if constexpr (DT > 0) {
    // register-blocked: one (ci, co) pair per pass, its T inputs and T output
    // gradients loaded once and reused by all K taps
    for (int q = tid; q < DT * DT; q += blockDim.x) {
      const int ci = q / DT, co = q % DT;
      float l[TT], g[TT];
#pragma unroll
      for (int t = 0; t < TT; ++t) {
        l[t] = locs[t * DT + ci];
        g[t] = dcv[t * DT + co];
      }
#pragma unroll
      for (int tap = 0; tap < KT; ++tap) {
        float a = 0.f;
#pragma unroll
        for (int t = 0; t < TT; ++t) {
          const int sidx = t + tap - KT / 2;
          if (sidx >= 0 && sidx < TT) a += l[sidx] * g[t];
        }
        RR_ADD(M.sl.conv_k, tap * DT * DT + q, a);
      }
    }
  } else {
    for (int q = tid; q < d.K * d.D * d.D; q += blockDim.x) {
      const int tap = q / (d.D * d.D), ci = (q / d.D) % d.D, co = q % d.D;
      float s = 0.f;
      for (int t = 0; t < d.T; ++t) {
        const int sidx = t + tap - pad;
        if (sidx >= 0 && sidx < d.T) s += locs[sidx * d.D + ci] * dcv[t * d.D + co];
      }
      RR_ADD(M.sl.conv_k, q, s);
    }
  }
  if constexpr (DT > 0) {
    // input gradient, two positions per thread sharing each tap weight load
    // (s0 and s0 + TT/2, same ci); dconv rows come in as float4 broadcasts
    const int ci = tid % DT, s0 = tid / DT, s1 = s0 + TT / 2;
    float acc0 = 0.f, acc1 = 0.f;
#pragma unroll
    for (int tap = 0; tap < KT; ++tap) {
      const int t0 = s0 - tap + KT / 2, t1 = s1 - tap + KT / 2;
      const bool v0 = t0 >= 0, v1 = t1 < TT;          // t0 < TT and t1 >= 0 always hold
      const float4* g0 = (const float4*)(dcv + (v0 ? t0 : 0) * DT);
      const float4* g1 = (const float4*)(dcv + (v1 ? t1 : 0) * DT);
      const float* kk = ck + tap * DT * ckp + ci;
      float p0 = 0.f, p1 = 0.f;
#pragma unroll
      for (int c4 = 0; c4 < DT / 4; ++c4) {
        const float4 a = g0[c4], bq = g1[c4];
        const float k0 = kk[(4 * c4) * ckp], k1 = kk[(4 * c4 + 1) * ckp];
        const float k2 = kk[(4 * c4 + 2) * ckp], k3 = kk[(4 * c4 + 3) * ckp];
        p0 += a.x * k0; p0 += a.y * k1; p0 += a.z * k2; p0 += a.w * k3;
        p1 += bq.x * k0; p1 += bq.y * k1; p1 += bq.z * k2; p1 += bq.w * k3;
      }
      if (v0) acc0 += p0;
      if (v1) acc1 += p1;
    }
    dls[s0 * DT + ci] = acc0;
    dls[s1 * DT + ci] = acc1;
  } else {
    for (int j = tid; j < d.H; j += blockDim.x) {
      const int sidx = j / d.D, ci = j % d.D;
      float acc = 0.f;
      for (int tap = 0; tap < d.K; ++tap) {
        const int t = sidx - tap + pad;
        if (t < 0 || t >= d.T) continue;
        float part = 0.f;
        for (int co = 0; co < d.D; ++co) part += dcv[t * d.D + co] * ck[(tap * d.D + co) * ckp + ci];
        acc += part;
      }
      dls[j] = acc;
    }
  }
  __syncthreads();
  // per-symbol LayerNorm backward over D
  const float* lg = M.w[P_LOC_LN_G].p;
  if constexpr (DT > 0) {
    // warp w takes positions t = w, w + 8; lane = channel e (coalesced
    // loc_hat rows).  Per-t means by xor-tree sums; the per-channel gain and
    // bias gradients from 8 warp partials (dconv is dead now) in a fixed order
    const int w = tid >> 5, e = tid & 31;
    float* p1 = dcv;
    float* p2 = dcv + 8 * DT;
    float q1 = 0.f, q2 = 0.f;
#pragma unroll
    for (int t = w; t < TT; t += 8) {
      const float dl = dls[t * DT + e];
      const float lh = lhs[t * DT + e];
      q1 += dl * lh;
      q2 += dl;
      const float gg = dl * lg[e];
      const float s1 = warp_sum(gg), s2 = warp_sum(gg * lh);
      if (e == 0) {
        locs[2 * t] = s1 / (float)DT;
        locs[2 * t + 1] = s2 / (float)DT;
      }
    }
    p1[w * DT + e] = q1;
    p2[w * DT + e] = q2;
    __syncthreads();
    if (tid < DT) {
      float s1 = 0.f, s2 = 0.f;
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        s1 += p1[k * DT + tid];
        s2 += p2[k * DT + tid];
      }
      RR_ADD(M.sl.loc_g, tid, s1);
      RR_ADD(M.sl.loc_b, tid, s2);
    }
  } else {
  for (int e = tid; e < d.D; e += blockDim.x) {
    float s1 = 0.f, s2 = 0.f;
    for (int t = 0; t < d.T; ++t) {
      s1 += dls[t * d.D + e] * lhs[t * d.D + e];
      s2 += dls[t * d.D + e];
    }
    RR_ADD(M.sl.loc_g, e, s1);
    RR_ADD(M.sl.loc_b, e, s2);
  }
  for (int t = tid; t < d.T; t += blockDim.x) {
    float s1 = 0.f, s2 = 0.f;
    for (int e = 0; e < d.D; ++e) {
      const float gg = dls[t * d.D + e] * lg[e];
      s1 += gg;
      s2 += gg * lhs[t * d.D + e];
    }
    // stash per-t means in the tail of locs (no longer needed after dloc)
    locs[2 * t] = s1 / (float)d.D;
    locs[2 * t + 1] = s2 / (float)d.D;
  }
  }
  }   // local stream
  __syncthreads();
  const float* lg = M.w[P_LOC_LN_G].p;
  for (int j = tid; j < d.H; j += blockDim.x) {
    const int t = j / d.D, e = j % d.D;
    float de = 0.f;
    if (vf.local) {
      de = (dls[j] * lg[e] - locs[2 * t] - lhs[j] * locs[2 * t + 1]) * lis[t];
    }
    // embedding gradient (ops.py:234-243 scatter-add): integer adds commute,
    // so the fixed-point sum is the same whatever order the rows arrive in
    if (!(M.dbg & 1))
      atomicAdd((unsigned long long*)&M.a.emb_acc[ctx[t] * d.D + e],
                (unsigned long long)emb_to_fixed(de + dxs[j]));
  }
  if (multi) __syncthreads();   // the next row reuses every smem row buffer
  }   // rows of this CTA
#undef RR_ADD
  if (multi) {
    float* part = M.a.trunk_part + (long long)blockIdx.x * (M.sl.trunk1 - t0);
    for (int c = tid; c < M.sl.trunk1 - t0; c += blockDim.x) part[c] = acc[c];
  }
}

void launch_trunk_bwd(const ModelPtrs& M, const uint8_t* src, long long ld_src, int use_col,
                      cudaStream_t s) {
  const Dims& d = M.d;
  if (row_warp_enabled(d.B, 7) && launch_trunk_bwd_w(M, src, ld_src, use_col, s)) return;
  const bool multi = d.B > M.trunk_grid;
  const size_t smem =
      sizeof(float) * (6 * d.H + d.K * d.D * (d.D + 1) + 3 * d.D + 32 + ((d.T + 3) & ~3)) +
      sizeof(int) * ((d.T + 3) & ~3) + (multi ? sizeof(float) * (M.sl.trunk1 - M.sl.trunk0) : 0);
  static const cudaError_t a1 = cudaFuncSetAttribute(
      k_trunk_bwd<32, 16, 3>, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
  static const cudaError_t a2 = cudaFuncSetAttribute(
      k_trunk_bwd<0, 0, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  (void)a1;
  (void)a2;
  const dim3 grid(M.trunk_grid);
  if (d.D == 32 && d.T == 16 && d.K == 3)
    launch_pdl(k_trunk_bwd<32, 16, 3>, grid, dim3(kTrunkThreads), smem, s, M, src, ld_src, use_col);
  else
    launch_pdl(k_trunk_bwd<0, 0, 0>, grid, dim3(kTrunkThreads), smem, s, M, src, ld_src, use_col);
}

// Column sums of the per-row reduction buffer + dlogits (b_head), in a fixed
// order, then Adam on the small-parameter arena.  Also the step loss.
constexpr int kColWarps = 16;
constexpr int kColAcc = 8;
// one CTA per 32 columns of the rowred/dlogits matrices; 16 warps x 8
// independent accumulators keep 8 row loads in flight per thread (the column
// sum is latency bound: 19.6 MB that just landed in L2).  Partials combine in
// a fixed order, so the result is deterministic.
// Extra CTAs past the column blocks apply the embedding update from the
// fixed-point accumulator (and clear it for the next step).  Last kernel of a
// step: with `advance` it moves the step state to the next column.
// (40 registers: 512 x 40 fits on an SM beside the two W_route/W_mem update
// CTAs still running at the end of the step; at 64 it waited for them, +1 us)
__global__ void __maxnreg__(40) k_small_adam(ModelPtrs M, int grad_only,
                                                               double* losses, double* alpha_tape,
                                                               int col_blocks, int advance) {
  pdl_enter();
  if ((int)blockIdx.x >= col_blocks) {
    const int q = ((int)blockIdx.x - col_blocks) * blockDim.x + threadIdx.x;
    if (q >= kAlphabet * M.d.D) return;
    long long* acc = M.a.emb_acc + q;
    const float g = emb_from_fixed(*acc);
    *acc = 0;
    Tensor4 t = M.w[P_EMB];
    if (grad_only) t.g[q] = g;
    else adam_update(M.st->adam, g, t.p + q, t.m + q, t.v + q);
    return;
  }
  __shared__ float part[kColWarps][33];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int c = blockIdx.x * 32 + lane;
  const int R = M.sl.rowred;
  const int total = R + kAlphabet;
  float acc[kColAcc];
#pragma unroll
  for (int k = 0; k < kColAcc; ++k) acc[k] = 0.f;
  if (c < total) {
    // trunk_bwd's columns come as one partial row per trunk_bwd CTA
    const bool trunk = c >= M.sl.trunk0 && c < M.sl.trunk1;
    const float* base = trunk ? M.a.trunk_part + (c - M.sl.trunk0)
                              : ((c < R) ? M.a.rowred + c : M.a.dlogits + (c - R));
    const long long ld = trunk ? M.sl.trunk1 - M.sl.trunk0 : ((c < R) ? R : kAlphabet);
    const int rows = trunk ? M.trunk_grid : ((c < R) ? M.rr_rows : M.d.B);
    int b = w;
    for (; b + (kColAcc - 1) * kColWarps < rows; b += kColAcc * kColWarps) {
#pragma unroll
      for (int k = 0; k < kColAcc; ++k) acc[k] += base[(long long)(b + k * kColWarps) * ld];
    }
    for (; b < rows; b += kColWarps) acc[0] += base[(long long)b * ld];
  }
  const float s = ((acc[0] + acc[1]) + (acc[2] + acc[3])) + ((acc[4] + acc[5]) + (acc[6] + acc[7]));
  part[w][lane] = s;
  __syncthreads();
  if (w == 0 && c < total) {
    float g = 0.f;
#pragma unroll
    for (int k = 0; k < kColWarps; ++k) g += part[k][lane];
    if (grad_only) M.small_g[c] = g;
    else adam_update(M.st->adam, g, M.small_p + c, M.small_m + c, M.small_v + c);
  }
  if (blockIdx.x == 0 && w == 1) {
    // mean cross-entropy: lane-strided partials, then a fixed xor tree
    double l = 0.0;
    for (int b = lane; b < M.d.B; b += 32) l += M.a.nll[b];
    l = warp_sum_d(l) / (double)M.d.B;
    // router statistics of this step's predict for the metrics tape
    // (model.py:197-199: mean, min, max of alpha over [B, H])
    double as = 0.0;
    float amn = 3.4e38f, amx = -3.4e38f;
    if (alpha_tape) {
      for (int b = lane; b < M.d.B; b += 32) {
        as += M.a.alpha_row[3 * b];
        amn = fminf(amn, M.a.alpha_row[3 * b + 1]);
        amx = fmaxf(amx, M.a.alpha_row[3 * b + 2]);
      }
      as = warp_sum_d(as);
      amn = -warp_max(-amn);
      amx = warp_max(amx);
    }
    if (lane == 0) {
      StepState* st = M.st;
      if (!isfinite(l)) record_error(st, st->col, 0, 5);
      if (losses) losses[st->col - st->loss_base] = l;
      if (M.tape) *tape_at(M, 4) = gtimer_ns();
      if (alpha_tape) {
        double* rec = alpha_tape + 3 * (st->col - st->loss_base);
        rec[0] = as / ((double)M.d.B * M.d.H);
        rec[1] = amn;
        rec[2] = amx;
      }
      // nothing else in this grid reads the column; the next step waits for us
      if (advance) {
        st->col += 1;
        st->step_count += 1;
      }
    }
  }
}

void launch_small_adam(const ModelPtrs& M, int grad_only, double* losses, double* alpha_tape,
                       int advance, cudaStream_t s) {
  const int col_blocks = cdiv(M.sl.rowred + kAlphabet, 32);
  const int emb_blocks = cdiv(kAlphabet * M.d.D, 32 * kColWarps);
  launch_pdl(k_small_adam, dim3(col_blocks + emb_blocks), dim3(32 * kColWarps), 0, s, M, grad_only,
             losses, alpha_tape, col_blocks, advance);
}

}  // namespace fade
