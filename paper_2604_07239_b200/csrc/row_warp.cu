// Warp-per-row variants of the hidden-width row kernels (H a multiple of 128,
// H <= 1024 -- the default H = 512 and the mid test geometry H = 128).
//
// One warp owns one stream row: lane l holds columns 4l + 128k (k < NV = H/128)
// as float4s, so every global access of the row is one coalesced 512-byte
// transaction per k, all of a row's loads are in flight together, and the
// LayerNorm / residual reductions are warp butterflies -- no __syncthreads and
// no shared memory.  A CTA carries kRowWarps rows.  Against one 512-thread CTA
// per row this removes the barrier-separated phases that made every row a
// chain of dependent round trips (B = 4096: mix_fwd 87 us, coarse_bwd 129 us
// in the step graph).
//
// Semantics are those of the CTA-per-row kernels in model_kernels.cu
// (model.py:128-172 and their backward); only the summation order of the
// fixed-order reductions differs (lane partials, then the butterfly), and it
// is the same for the encoder and the decoder.
#include "model.cuh"

namespace fade {

constexpr int kRowWarps = 4;

template <int NV>
struct RowV {
  float4 v[NV];
};

template <int NV>
__device__ __forceinline__ RowV<NV> ld_row(const float* __restrict__ row) {
  const int lane = threadIdx.x & 31;
  RowV<NV> r;
#pragma unroll
  for (int k = 0; k < NV; ++k) r.v[k] = *(const float4*)(row + 4 * lane + 128 * k);
  return r;
}
template <int NV>
__device__ __forceinline__ void st_row(float* __restrict__ row, const RowV<NV>& r) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int k = 0; k < NV; ++k) *(float4*)(row + 4 * lane + 128 * k) = r.v[k];
}
// element e (0..3) of float4 k
__device__ __forceinline__ float& el(float4& f, int e) {
  return e == 0 ? f.x : (e == 1 ? f.y : (e == 2 ? f.z : f.w));
}
__device__ __forceinline__ float el(const float4& f, int e) {
  return e == 0 ? f.x : (e == 1 ? f.y : (e == 2 ? f.z : f.w));
}
// GEMM-only operands stored rounded to nearest TF32 (common.cuh tf32_rne)
template <int NV>
__device__ __forceinline__ RowV<NV> rne_row(RowV<NV> r) {
#pragma unroll
  for (int k = 0; k < NV; ++k) r.v[k] = tf32_rne4(r.v[k]);
  return r;
}
template <int NV>
__device__ __forceinline__ float row_sum(const RowV<NV>& r) {
  float s = 0.f;
#pragma unroll
  for (int k = 0; k < NV; ++k) s += (r.v[k].x + r.v[k].y) + (r.v[k].z + r.v[k].w);
  return warp_sum(s);
}
// Split-K planes of a [B][H] GEMM output reduced in plane order into four
// interleaved accumulators (the split_sum order), row `row`.
template <int NV>
__device__ __forceinline__ RowV<NV> ld_split(const float* __restrict__ ws, long long plane,
                                             long long rowoff, int S) {
  const int lane = threadIdx.x & 31;
  RowV<NV> out;
#pragma unroll
  for (int k = 0; k < NV; ++k) {
    float4 a[4];
#pragma unroll
    for (int g = 0; g < 4; ++g) a[g] = make_float4(0.f, 0.f, 0.f, 0.f);
    const float* p = ws + rowoff + 4 * lane + 128 * k;
#pragma unroll 4
    for (int s = 0; s < S; ++s) {
      const float4 v = *(const float4*)(p + s * plane);
      float4& t = a[s & 3];
      t.x += v.x;
      t.y += v.y;
      t.z += v.z;
      t.w += v.w;
    }
    out.v[k] = make_float4((a[0].x + a[1].x) + (a[2].x + a[3].x), (a[0].y + a[1].y) + (a[2].y + a[3].y),
                           (a[0].z + a[1].z) + (a[2].z + a[3].z), (a[0].w + a[1].w) + (a[2].w + a[3].w));
  }
  return out;
}
// LayerNorm statistics (ops.py:94-101): mean, then mean of squared deviations
template <int NV>
__device__ __forceinline__ void row_ln_stats(const RowV<NV>& x, float n, float* mu, float* inv) {
  const float m = row_sum(x) / n;
  float q = 0.f;
#pragma unroll
  for (int k = 0; k < NV; ++k)
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const float c = el(x.v[k], e) - m;
      q += c * c;
    }
  const float var = warp_sum(q) / n;
  *mu = m;
  *inv = __fdiv_rn(1.0f, __fsqrt_rn(var + kLnEps));
}

#define ROW_PROLOGUE                                                   \
  pdl_enter();                                                         \
  const int lane = threadIdx.x & 31;                                   \
  const int b = blockIdx.x * kRowWarps + (threadIdx.x >> 5);           \
  if (b >= M.d.B) return;                                              \
  const int H = NV * 128;                                              \
  const long long rH = (long long)b * H;                               \
  const long long plane = (long long)M.d.B * H;                        \
  (void)plane;                                                         \
  (void)lane;

// ---------------------------------------------------------------------------
// forward

// global stream finish + router + mixer LayerNorm (model.py:128-153)
template <int NV>
__global__ void __launch_bounds__(32 * kRowWarps) k_mix_fwd_w(ModelPtrs M) {
  ROW_PROLOGUE
  // count this step's roll of the ring-buffer cache (see k_mix_fwd)
  if (ring_cache(M) && b == 0 && lane == 0) M.st->ring += 1;
  const VFlags vf = vflags(M.variant);
  const float lam = M.w[P_LAM_MEM].p[0];
  RowV<NV> hg, hm, up, x, hl, rp;
  if (vf.global) {
    up = ld_split<NV>(M.a.ws_mem, plane, rH, M.splits_mem);
    x = ld_row<NV>(M.a.x + rH);
  }
  if (vf.local) hl = ld_row<NV>(M.a.h_l + rH);
  if (vf.router) rp = ld_split<NV>(M.sk[S_RPRE].ws, plane, rH, M.sk[S_RPRE].S);
  float asum = 0.f, amin = 3.4e38f, amax = -3.4e38f;
  RowV<NV> al;
#pragma unroll
  for (int k = 0; k < NV; ++k)
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      float g = 0.f, h;
      if (vf.global) g = gelu_f(el(up.v[k], e)) + el(x.v[k], e) * lam;
      if (vf.router) {
        const float a = sigmoid_f(el(rp.v[k], e));
        h = a * g + (1.0f - a) * el(hl.v[k], e);
        el(al.v[k], e) = a;
        asum += a;
        amin = fminf(amin, a);
        amax = fmaxf(amax, a);
      } else {
        h = vf.global ? g : el(hl.v[k], e);
      }
      el(hg.v[k], e) = g;
      el(hm.v[k], e) = h;
    }
  if (vf.global) {
    st_row<NV>(M.a.upre + rH, up);
    st_row<NV>(M.a.h_g + rH, hg);
  }
  st_row<NV>(M.a.h_mix + rH, hm);
  st_row<NV>(M.a.hm_tc + rH, rne_row<NV>(hm));
  if (vf.router) {
    st_row<NV>(M.a.alpha + rH, al);
    const float s = warp_sum(asum);
    const float mn = -warp_max(-amin), mx = warp_max(amax);
    if (lane == 0) {
      M.a.alpha_row[3 * b + 0] = s;
      M.a.alpha_row[3 * b + 1] = mn;
      M.a.alpha_row[3 * b + 2] = mx;
    }
  }
  if (!vf.mixer) return;
  float mu, inv;
  row_ln_stats<NV>(hm, (float)H, &mu, &inv);
  const RowV<NV> g = ld_row<NV>(M.w[P_MIX_LN_G].p), bb = ld_row<NV>(M.w[P_MIX_LN_B].p);
  RowV<NV> zh, z;
#pragma unroll
  for (int k = 0; k < NV; ++k)
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const float t = (el(hm.v[k], e) - mu) * inv;
      el(zh.v[k], e) = t;
      el(z.v[k], e) = t * el(g.v[k], e) + el(bb.v[k], e);
    }
  st_row<NV>(M.a.z_hat + rH, zh);
  st_row<NV>(M.a.z + rH, rne_row<NV>(z));
  if (lane == 0) M.a.z_inv[b] = inv;
}

// self-gated coarse refiner + FNR LayerNorm (model.py:156-167)
template <int NV>
__global__ void __launch_bounds__(32 * kRowWarps) k_coarse_fwd_w(ModelPtrs M) {
  ROW_PROLOGUE
  const VFlags vf = vflags(M.variant);
  const float lam = M.w[P_LAM_MIX].p[0];
  const RowV<NV> in = ld_split<NV>(M.sk[S_INNER].ws, plane, rH, M.sk[S_INNER].S);
  const RowV<NV> hm = ld_row<NV>(M.a.h_mix + rH);
  RowV<NV> cp, gt, hc;
  if (vf.gate) cp = ld_split<NV>(M.sk[S_CPRE].ws, plane, rH, M.sk[S_CPRE].S);
#pragma unroll
  for (int k = 0; k < NV; ++k)
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const float t = vf.gate ? sigmoid_f(el(cp.v[k], e)) : 1.0f;   // mixer_nogate: inner * 1
      el(gt.v[k], e) = t;
      el(hc.v[k], e) = el(in.v[k], e) * t + el(hm.v[k], e) * lam;
    }
  st_row<NV>(M.a.inner + rH, in);
  st_row<NV>(M.a.gate + rH, gt);
  st_row<NV>(M.a.h_c + rH, hc);
  if (!vf.fnr) return;
  float mu, inv;
  row_ln_stats<NV>(hc, (float)H, &mu, &inv);
  const RowV<NV> g = ld_row<NV>(M.w[P_REF_LN_G].p), bb = ld_row<NV>(M.w[P_REF_LN_B].p);
  RowV<NV> zh, z;
#pragma unroll
  for (int k = 0; k < NV; ++k)
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const float t = (el(hc.v[k], e) - mu) * inv;
      el(zh.v[k], e) = t;
      el(z.v[k], e) = t * el(g.v[k], e) + el(bb.v[k], e);
    }
  st_row<NV>(M.a.z2_hat + rH, zh);
  st_row<NV>(M.a.z2 + rH, rne_row<NV>(z));
  if (lane == 0) M.a.z2_inv[b] = inv;
}

// FNR output: split-K reduce, LayerNorm, gelu, residual (model.py:170-172)
template <int NV>
__global__ void __launch_bounds__(32 * kRowWarps) k_out_fwd_w(ModelPtrs M) {
  ROW_PROLOGUE
  const RowV<NV> np = ld_split<NV>(M.a.ws_f, plane, rH, M.splits_f);
  const RowV<NV> hc = ld_row<NV>(M.a.h_c + rH);
  const RowV<NV> g = ld_row<NV>(M.w[P_OUT_LN_G].p), bb = ld_row<NV>(M.w[P_OUT_LN_B].p);
  const float lam = M.w[P_LAM_OUT].p[0];
  float mu, inv;
  row_ln_stats<NV>(np, (float)H, &mu, &inv);
  RowV<NV> nh, nv, h;
#pragma unroll
  for (int k = 0; k < NV; ++k)
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const float t = (el(np.v[k], e) - mu) * inv;
      const float v = t * el(g.v[k], e) + el(bb.v[k], e);
      el(nh.v[k], e) = t;
      el(nv.v[k], e) = v;
      el(h.v[k], e) = gelu_f(v) + el(hc.v[k], e) * lam;
    }
  st_row<NV>(M.a.n_hat + rH, nh);
  st_row<NV>(M.a.nrm + rH, nv);
  st_row<NV>(M.a.h + rH, rne_row<NV>(h));
  if (lane == 0) M.a.n_inv[b] = inv;
}

// ---------------------------------------------------------------------------
// backward

// LayerNorm backward means (ops.py:103-113): m1 = mean(dy*g), m2 = mean(dy*g*xhat)
template <int NV>
__device__ __forceinline__ void row_ln_bwd_means(const RowV<NV>& dy, const RowV<NV>& g,
                                                 const RowV<NV>& xh, float n, float* m1, float* m2) {
  float s1 = 0.f, s2 = 0.f;
#pragma unroll
  for (int k = 0; k < NV; ++k)
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const float gg = el(dy.v[k], e) * el(g.v[k], e);
      s1 += gg;
      s2 += gg * el(xh.v[k], e);
    }
  *m1 = warp_sum(s1) / n;
  *m2 = warp_sum(s2) / n;
}

// Per-row gradient columns of the small parameters (LayerNorm gains / biases
// and the lam scalars) for k_small_adam.  M.rr_rows == B: one rowred row per
// stream row.  M.rr_rows == B / kRowWarps (B >= 2048, all three backward row
// kernels warp-per-row): the CTA's rows are summed in warp order (w = 0, 1, 2,
// 3) through shared memory and written as ONE rowred row per CTA -- a quarter
// of the bytes written here and read back by small_adam.
template <int NV>
__device__ __forceinline__ void rr_store(const ModelPtrs& M, int b, bool two, int off0,
                                         const RowV<NV>& r0, int off1, const RowV<NV>& r1,
                                         bool has_l, int offl, float l) {
  constexpr int H = NV * 128, ld = 2 * H + 4;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if (M.rr_rows == M.d.B) {
    float* rr = M.a.rowred + (long long)b * M.sl.rowred;
    if (two) {
      st_row<NV>(rr + off0, r0);
      st_row<NV>(rr + off1, r1);
    }
    if (has_l && lane == 0) rr[offl] = l;
    return;
  }
  extern __shared__ float4 rr_sm4[];
  float* sm = (float*)rr_sm4;
  float* slot = sm + w * ld;
  if (two) {
    st_row<NV>(slot, r0);
    st_row<NV>(slot + H, r1);
  }
  if (lane == 0) slot[2 * H] = l;
  __syncthreads();
  float* rr = M.a.rowred + (long long)blockIdx.x * M.sl.rowred;
  for (int c = threadIdx.x; c <= 2 * H; c += blockDim.x) {
    if (c < 2 * H ? !two : !has_l) continue;
    float v = sm[c];
#pragma unroll
    for (int k = 1; k < kRowWarps; ++k) v += sm[k * ld + c];
    rr[c < H ? off0 + c : (c < 2 * H ? off1 + c - H : offl)] = v;
  }
  __syncthreads();   // the slots are rewritten by a following rr_store
}

int rowred_rows(int B, int H) {
  // (the CTA-per-row fallbacks -- H not a multiple of 128 -- write every row)
  return (B % kRowWarps == 0 && H % 128 == 0 && H <= 1024 && row_warp_enabled(B, 3) &&
          row_warp_enabled(B, 4) && row_warp_enabled(B, 5))
             ? B / kRowWarps
             : B;
}

// h = gelu(LN(npre)) + lam_out * h_c   (model.py:170-172 backward)
template <int NV>
__global__ void __launch_bounds__(32 * kRowWarps) k_out_bwd_w(ModelPtrs M) {
  ROW_PROLOGUE
  const float lam = M.w[P_LAM_OUT].p[0];
  const RowV<NV> dh = ld_split<NV>(M.sk[S_DH].ws, plane, rH, M.sk[S_DH].S);
  const RowV<NV> nrm = ld_row<NV>(M.a.nrm + rH), nh = ld_row<NV>(M.a.n_hat + rH);
  const RowV<NV> hc = ld_row<NV>(M.a.h_c + rH), g = ld_row<NV>(M.w[P_OUT_LN_G].p);
  const float inv = M.a.n_inv[b];
  RowV<NV> dn, rg, dhc;
  float lsum = 0.f;
#pragma unroll
  for (int k = 0; k < NV; ++k)
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const float d = el(dh.v[k], e);
      const float v = d * gelu_grad_f(el(nrm.v[k], e));
      el(dn.v[k], e) = v;
      el(rg.v[k], e) = v * el(nh.v[k], e);
      lsum += d * el(hc.v[k], e);
      el(dhc.v[k], e) = d * lam;
    }
  st_row<NV>(M.a.dhc + rH, dhc);
  rr_store<NV>(M, b, true, M.sl.out_g, rg, M.sl.out_b, dn, true, M.sl.lam_out, warp_sum(lsum));
  float m1, m2;
  row_ln_bwd_means<NV>(dn, g, nh, (float)H, &m1, &m2);
  RowV<NV> dx;
#pragma unroll
  for (int k = 0; k < NV; ++k)
#pragma unroll
    for (int e = 0; e < 4; ++e)
      el(dx.v[k], e) = (el(dn.v[k], e) * el(g.v[k], e) - m1 - el(nh.v[k], e) * m2) * inv;
  st_row<NV>(M.a.dnpre + rH, dx);
}

// z2 = LN(h_c); h_c = inner * sigmoid(cpre) + lam_mix * h_mix   (backward)
template <int NV>
__global__ void __launch_bounds__(32 * kRowWarps) k_coarse_bwd_w(ModelPtrs M) {
  ROW_PROLOGUE
  const VFlags vf = vflags(M.variant);
  RowV<NV> dhc, rg, rb;
  if (vf.fnr) {
    const RowV<NV> dz = ld_split<NV>(M.a.ws_dz2, plane, rH, M.splits_dz2);
    const RowV<NV> zh = ld_row<NV>(M.a.z2_hat + rH), g = ld_row<NV>(M.w[P_REF_LN_G].p);
    const RowV<NV> din = ld_row<NV>(M.a.dhc + rH);
    const float inv = M.a.z2_inv[b];
#pragma unroll
    for (int k = 0; k < NV; ++k)
#pragma unroll
      for (int e = 0; e < 4; ++e) el(rg.v[k], e) = el(dz.v[k], e) * el(zh.v[k], e);
    rb = dz;
    float m1, m2;
    row_ln_bwd_means<NV>(dz, g, zh, (float)H, &m1, &m2);
#pragma unroll
    for (int k = 0; k < NV; ++k)
#pragma unroll
      for (int e = 0; e < 4; ++e)
        el(dhc.v[k], e) = el(din.v[k], e) +
                          (el(dz.v[k], e) * el(g.v[k], e) - m1 - el(zh.v[k], e) * m2) * inv;
  } else {
    // without the FNR, h = h_coarse and dh arrives straight from the head GEMM
    dhc = ld_split<NV>(M.sk[S_DH].ws, plane, rH, M.sk[S_DH].S);
  }
  const RowV<NV> gt = ld_row<NV>(M.a.gate + rH), hm = ld_row<NV>(M.a.h_mix + rH);
  RowV<NV> inner, di, dc;
  if (vf.gate) inner = ld_row<NV>(M.a.inner + rH);
  float lsum = 0.f;
#pragma unroll
  for (int k = 0; k < NV; ++k)
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const float d = el(dhc.v[k], e), t = el(gt.v[k], e);
      el(di.v[k], e) = d * t;
      if (vf.gate) el(dc.v[k], e) = d * el(inner.v[k], e) * t * (1.0f - t);
      lsum += d * el(hm.v[k], e);
    }
  st_row<NV>(M.a.dhc + rH, dhc);
  st_row<NV>(M.a.dinner + rH, di);
  if (vf.gate) st_row<NV>(M.a.dcpre + rH, dc);
  rr_store<NV>(M, b, vf.fnr, M.sl.ref_g, rg, M.sl.ref_b, rb, true, M.sl.lam_mix, warp_sum(lsum));
}

// mixer LayerNorm + router mix + global-stream gelu (model.py:128-153 backward)
template <int NV>
__global__ void __launch_bounds__(32 * kRowWarps) k_mix_bwd_w(ModelPtrs M) {
  ROW_PROLOGUE
  const VFlags vf = vflags(M.variant);
  RowV<NV> dhm, rg, rb;
  if (vf.mixer) {
    const RowV<NV> dz = ld_split<NV>(M.sk[S_DZ].ws, plane, rH, M.sk[S_DZ].S);
    const RowV<NV> zh = ld_row<NV>(M.a.z_hat + rH), g = ld_row<NV>(M.w[P_MIX_LN_G].p);
    const RowV<NV> dc = ld_row<NV>(M.a.dhc + rH);
    RowV<NV> dm;
    if (vf.gate) dm = ld_split<NV>(M.sk[S_DHMC].ws, plane, rH, M.sk[S_DHMC].S);
    const float inv = M.a.z_inv[b];
    const float lam_mix = M.w[P_LAM_MIX].p[0];
#pragma unroll
    for (int k = 0; k < NV; ++k)
#pragma unroll
      for (int e = 0; e < 4; ++e) el(rg.v[k], e) = el(dz.v[k], e) * el(zh.v[k], e);
    rb = dz;
    float m1, m2;
    row_ln_bwd_means<NV>(dz, g, zh, (float)H, &m1, &m2);
#pragma unroll
    for (int k = 0; k < NV; ++k)
#pragma unroll
      for (int e = 0; e < 4; ++e)
        el(dhm.v[k], e) = el(dc.v[k], e) * lam_mix + (vf.gate ? el(dm.v[k], e) : 0.f) +
                          (el(dz.v[k], e) * el(g.v[k], e) - m1 - el(zh.v[k], e) * m2) * inv;
  } else {
    dhm = ld_split<NV>(M.sk[S_DH].ws, plane, rH, M.sk[S_DH].S);   // h = h_mix
  }
  const float lam_mem = M.w[P_LAM_MEM].p[0];
  RowV<NV> al, hg, hl, up, x;
  if (vf.router) {
    al = ld_row<NV>(M.a.alpha + rH);
    hg = ld_row<NV>(M.a.h_g + rH);
    hl = ld_row<NV>(M.a.h_l + rH);
  }
  if (vf.global) {
    up = ld_row<NV>(M.a.upre + rH);
    x = ld_row<NV>(M.a.x + rH);
  }
  RowV<NV> drp, dl, dup, dxp;
  float lsum = 0.f;
#pragma unroll
  for (int k = 0; k < NV; ++k)
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const float d = el(dhm.v[k], e);
      float dg = d, dlc = d;
      if (vf.router) {
        const float a = el(al.v[k], e);
        const float da = d * (el(hg.v[k], e) - el(hl.v[k], e));
        dg = d * a;
        dlc = d * (1.0f - a);
        el(drp.v[k], e) = da * a * (1.0f - a);
      }
      el(dl.v[k], e) = dlc;
      if (vf.global) {
        el(dup.v[k], e) = dg * gelu_grad_f(el(up.v[k], e));
        el(dxp.v[k], e) = dg * lam_mem;
        lsum += dg * el(x.v[k], e);
      }
    }
  if (vf.router) st_row<NV>(M.a.drpre + rH, drp);
  if (vf.local) st_row<NV>(M.a.dh_l + rH, dl);
  if (vf.global) {
    st_row<NV>(M.a.dupre + rH, dup);
    st_row<NV>(M.a.dx_part + rH, dxp);
  }
  rr_store<NV>(M, b, vf.mixer, M.sl.mix_g, rg, M.sl.mix_b, rb, vf.global, M.sl.lam_mem,
               vf.global ? warp_sum(lsum) : 0.f);
}

// ---------------------------------------------------------------------------
// ---------------------------------------------------------------------------
// trunk + local stream forward, warp per row (model.py:118-137; the
// compiled geometry D = 32, T = 16, K = 3 only, rolling cache not a ring).
// Lane e holds column e of every context symbol t (es[t] = emb[ctx[t]][e]),
// so the input LayerNorm, the per-symbol LayerNorm and the GeGLU block are
// warp butterflies / shuffles, and the conv runs lane = output channel over
// the warp's normalised window staged in shared memory (float4 broadcasts).
// The weights are staged once per CTA; warps walk rows b = warp id,
// + grid warps, ...  Same semantics as k_trunk_fwd<32, 16, 3>; only the
// summation order of its reductions differs.
constexpr int kTfWarps = 8;
constexpr int kTfD = 32, kTfT = 16, kTfK = 3, kTfH = kTfD * kTfT;
constexpr int kTfSmemFloats = 2 * kTfD * kTfD + kTfK * kTfD * kTfD + kTfWarps * kTfH;

__global__ void __launch_bounds__(32 * kTfWarps, 2) k_trunk_fwd_w(ModelPtrs M, const uint8_t* src,
                                                                 long long ld_src, int use_col) {
  pdl_enter();
  extern __shared__ float4 tf_sm4[];
  float* wg = (float*)tf_sm4;                 // [D][D]   W_gate
  float* wv = wg + kTfD * kTfD;               // [D][D]   W_val
  float* ck = wv + kTfD * kTfD;               // [K][D][D] conv taps [tap][ci][co]
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  float* locw = ck + kTfK * kTfD * kTfD + w * kTfH;   // this warp's normalised window
  const VFlags vf = vflags(M.variant);
  const Dims& d = M.d;
  const long long c0 = use_col ? M.st->col - kTfT : 0;
  if (M.tape && blockIdx.x == 0 && tid == 0) *tape_at(M, 0) = gtimer_ns();
  {
    const float4* g4 = (const float4*)M.w[P_W_GATE].p;
    const float4* v4 = (const float4*)M.w[P_W_VAL].p;
    const float4* k4 = (const float4*)M.w[P_CONV_K].p;
    float4* s4 = tf_sm4;
    for (int j = tid; j < kTfD * kTfD / 4; j += blockDim.x) {
      s4[j] = g4[j];
      s4[kTfD * kTfD / 4 + j] = v4[j];
    }
    for (int j = tid; j < kTfK * kTfD * kTfD / 4; j += blockDim.x) s4[kTfD * kTfD / 2 + j] = k4[j];
  }
  __syncthreads();
  const float* E = M.w[P_EMB].p;
  const float* g_in = M.w[P_IN_LN_G].p;
  const float* b_in = M.w[P_IN_LN_B].p;
  const int n4 = (d.C - kTfD) / 4;        // float4 count the roll moves
  for (int b = blockIdx.x * kTfWarps + w; b < d.B; b += gridDim.x * kTfWarps) {
    const long long rH = (long long)b * kTfH;
    const int sym = lane < kTfT ? src[(long long)b * ld_src + c0 + lane] : 0;
    float es[kTfT];
#pragma unroll
    for (int t = 0; t < kTfT; ++t) es[t] = E[__shfl_sync(0xffffffffu, sym, t) * kTfD + lane];
    float* crow = M.a.cache + (long long)b * d.C;
    // input LayerNorm over the flattened window (ops.py:94-101)
    float s = 0.f;
#pragma unroll
    for (int t = 0; t < kTfT; ++t) s += es[t];
    const float mu = warp_sum(s) / (float)kTfH;
    float q = 0.f;
#pragma unroll
    for (int t = 0; t < kTfT; ++t) {
      const float c = es[t] - mu;
      q += c * c;
    }
    const float inv = __fdiv_rn(1.0f, __fsqrt_rn(warp_sum(q) / (float)kTfH + kLnEps));
    float x15 = 0.f;
#pragma unroll
    for (int t = 0; t < kTfT; ++t) {
      const int j = t * kTfD + lane;
      const float xh = (es[t] - mu) * inv;
      const float xv = xh * g_in[j] + b_in[j];
      M.a.x_hat[rH + j] = xh;
      M.a.x[rH + j] = xv;
      M.a.x_tc[rH + j] = tf32_rne(xv);
      if (t == kTfT - 1) x15 = xv;
    }
    if (lane == 0) M.a.x_inv[b] = inv;
    if (vf.global) {
      // roll the cache in place (new[j] = old[j + D]) eight float4 per lane
      // at a time: every group's loads precede its stores, and a store only
      // overwrites data a load of the same or an earlier group has read
      for (int base = 0; base < n4; base += 8 * 32) {
        float4 r[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const int qq = base + u * 32 + lane;
          if (qq < n4) r[u] = *(const float4*)(crow + kTfD + 4 * qq);
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const int qq = base + u * 32 + lane;
          if (qq < n4) *(float4*)(crow + 4 * qq) = r[u];
        }
      }
      // GeGLU block of the newest symbol: output o = lane, x_t[i] from lane i
      float g = 0.f, v = 0.f;
#pragma unroll
      for (int i = 0; i < kTfD; ++i) {
        const float xi = __shfl_sync(0xffffffffu, x15, i);
        g += xi * wg[i * kTfD + lane];
        v += xi * wv[i * kTfD + lane];
      }
      M.a.gpre[(long long)b * kTfD + lane] = g;
      M.a.vpre[(long long)b * kTfD + lane] = v;
      crow[d.C - kTfD + lane] = tf32_rne(gelu_f(g) * v);
    }
    if (vf.local) {
      // per-symbol LayerNorm over D (ops.py:94-101 on (B,T,D))
      const float* lg = M.w[P_LOC_LN_G].p;
      const float* lb = M.w[P_LOC_LN_B].p;
      const float gl = lg[lane], bl = lb[lane];
#pragma unroll
      for (int t = 0; t < kTfT; ++t) {
        const float m = warp_sum(es[t]) / (float)kTfD;
        const float c = es[t] - m;
        const float tinv = __fdiv_rn(1.0f, __fsqrt_rn(warp_sum(c * c) / (float)kTfD + kLnEps));
        if (lane == 0) M.a.loc_inv[(long long)b * kTfT + t] = tinv;
        const float lh = c * tinv;
        const float lv = lh * gl + bl;
        M.a.loc_hat[rH + t * kTfD + lane] = lh;
        M.a.loc[rH + t * kTfD + lane] = lv;
        locw[t * kTfD + lane] = lv;
      }
      __syncwarp();
      // same-padded conv (ops.py:57-72), output channel co = lane: input
      // symbol s feeds outputs s + 1 (tap 0), s (tap 1) and s - 1 (tap 2)
      float acc[kTfT];
      const float cb = M.w[P_CONV_B].p[lane];
#pragma unroll
      for (int t = 0; t < kTfT; ++t) acc[t] = 0.f;
      const float4* l4 = (const float4*)locw;
#pragma unroll 1
      for (int c4 = 0; c4 < kTfD / 4; ++c4) {
        float k[kTfK][4];
#pragma unroll
        for (int tap = 0; tap < kTfK; ++tap)
#pragma unroll
          for (int c = 0; c < 4; ++c) k[tap][c] = ck[(tap * kTfD + 4 * c4 + c) * kTfD + lane];
#pragma unroll
        for (int sidx = 0; sidx < kTfT; ++sidx) {
          const float4 l = l4[sidx * (kTfD / 4) + c4];
          const float lv[4] = {l.x, l.y, l.z, l.w};
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            if (sidx + 1 < kTfT) acc[sidx + 1] += lv[c] * k[0][c];
            acc[sidx] += lv[c] * k[1][c];
            if (sidx >= 1) acc[sidx - 1] += lv[c] * k[2][c];
          }
        }
      }
#pragma unroll
      for (int t = 0; t < kTfT; ++t) {
        const float a = cb + acc[t];
        M.a.conv_pre[rH + t * kTfD + lane] = a;
        M.a.h_l[rH + t * kTfD + lane] = gelu_f(a);
      }
      __syncwarp();   // locw is rewritten by the warp's next row
    }
  }
}

bool launch_trunk_fwd_w(const ModelPtrs& M, const uint8_t* src, long long ld_src, int use_col,
                        cudaStream_t s) {
  const Dims& d = M.d;
  if (d.D != kTfD || d.T != kTfT || d.K != kTfK || M.ring_on || d.C % 4) return false;
  const size_t smem = sizeof(float) * kTfSmemFloats;
  static const cudaError_t attr =
      cudaFuncSetAttribute(k_trunk_fwd_w, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  (void)attr;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int grid = std::min(cdiv(d.B, kTfWarps), 2 * sms);
  launch_pdl(k_trunk_fwd_w, dim3(grid), dim3(32 * kTfWarps), smem, s, M, src, ld_src, use_col);
  return true;
}

// ---------------------------------------------------------------------------
// trunk + local stream backward at large B, in two launches (model.py:118-137
// backward; the compiled geometry D = 32, T = 16, K = 3 only):
//  * k_trunk_bwd_w, warp per row: the input-gradient chain (dx_t through
//    W_gate / W_val, the input LayerNorm backward, the conv input gradient,
//    the per-symbol LayerNorm backward, the embedding-gradient atomics).  It
//    leaves the row's pre-LayerNorm gradient dx and the conv input gradient
//    dloc in two [B][H] scratch rows for
//  * k_trunk_grads: the small-parameter gradients (in_g, in_b, loc_g, loc_b,
//    conv_b, conv_k, w_gate, w_val) as per-CTA sums over rows b = cta, cta +
//    grid, ... into trunk_part -- the layout k_small_adam reduces -- with
//    per-row sums in the order of k_trunk_bwd's multi-row path.
// Against the one-CTA-per-row k_trunk_bwd (eight warps through a chain of
// barrier-separated phases per row) the rows of a warp need no barrier.
__device__ __forceinline__ float split_at(const SplitBuf& k, long long plane, long long idx) {
  float a[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll 4
  for (int s = 0; s < k.S; ++s) a[s & 3] += k.ws[s * plane + idx];
  return (a[0] + a[1]) + (a[2] + a[3]);
}

constexpr int kTbWarps = 8;
// smem: W_gate^T, W_val^T [o][i], taps transposed [tap][co][ci], per-warp dconv
// window, then the CTA's embedding-gradient table [256][D] (int64 fixed point)
// and its touched-symbol flags
constexpr int kTbSmemFloats = 2 * kTfD * kTfD + kTfK * kTfD * kTfD + kTbWarps * kTfH;
constexpr size_t kTbSmemBytes = sizeof(float) * kTbSmemFloats + sizeof(long long) * 256 * kTfD +
                                sizeof(int) * 256;

__global__ void __launch_bounds__(32 * kTbWarps, 2) k_trunk_bwd_w(ModelPtrs M, const uint8_t* src,
                                                                 long long ld_src, int use_col) {
  pdl_enter();
  extern __shared__ float4 tb_sm4[];
  float* wgt = (float*)tb_sm4;               // [o][i] = W_gate[i][o]
  float* wvt = wgt + kTfD * kTfD;            // [o][i] = W_val[i][o]
  float* ckt = wvt + kTfD * kTfD;            // [tap][co][ci] = conv_k[tap][ci][co]
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  float* dcw = ckt + kTfK * kTfD * kTfD + w * kTfH;   // this warp's dconv window [t][co]
  // embedding-gradient rows of this CTA's rows, summed in shared memory first:
  // the global atomics then see one add per (CTA, symbol, channel) instead of
  // one per (row, position) -- frequent symbols no longer serialise on L2
  unsigned long long* eacc =
      (unsigned long long*)(ckt + kTfK * kTfD * kTfD + kTbWarps * kTfH);
  int* touched = (int*)(eacc + 256 * kTfD);
  for (int j = tid; j < 256 * kTfD; j += blockDim.x) eacc[j] = 0ull;
  for (int j = tid; j < 256; j += blockDim.x) touched[j] = 0;
  const VFlags vf = vflags(M.variant);
  const Dims& d = M.d;
  const long long c0 = use_col ? M.st->col - kTfT : 0;
  for (int j = tid; j < kTfD * kTfD; j += blockDim.x) {
    const int i = j / kTfD, o = j % kTfD;
    wgt[o * kTfD + i] = M.w[P_W_GATE].p[j];
    wvt[o * kTfD + i] = M.w[P_W_VAL].p[j];
  }
  for (int j = tid; j < kTfK * kTfD * kTfD; j += blockDim.x) {
    const int tap = j / (kTfD * kTfD), ci = (j / kTfD) % kTfD, co = j % kTfD;
    ckt[(tap * kTfD + co) * kTfD + ci] = M.w[P_CONV_K].p[j];
  }
  __syncthreads();
  const float* gin = M.w[P_IN_LN_G].p;
  const float gl = M.w[P_LOC_LN_G].p[lane];
  const long long planeH = (long long)d.B * kTfH, planeD = (long long)d.B * kTfD;
  for (int b = blockIdx.x * kTbWarps + w; b < d.B; b += gridDim.x * kTbWarps) {
    const long long rH = (long long)b * kTfH;
    const int sym = lane < kTfT ? src[(long long)b * ld_src + c0 + lane] : 0;
    // every load of the row first (independent, all in flight), then the sums
    float dx[kTfT], xh[kTfT], dp[kTfT];
#pragma unroll
    for (int t = 0; t < kTfT; ++t) {
      const long long j = rH + t * kTfD + lane;
      xh[t] = M.a.x_hat[j];
      dp[t] = vf.global ? M.a.dx_part[j] : 0.f;
      dx[t] = (vf.router && M.sk[S_DXR].S == 1) ? M.sk[S_DXR].ws[j] : 0.f;
    }
    // dx_t through the GeGLU block (lane = input i; dg / dv of output o from lane o)
    float dxt = 0.f;
    if (vf.global) {
      const float gp = M.a.gpre[(long long)b * kTfD + lane];
      const float vp = M.a.vpre[(long long)b * kTfD + lane];
      const float db = M.sk[S_DBLOCK].S == 1 ? M.sk[S_DBLOCK].ws[(long long)b * kTfD + lane]
                                              : split_at(M.sk[S_DBLOCK], planeD, (long long)b * kTfD + lane);
      const float dg = db * vp * gelu_grad_f(gp), dv = db * gelu_f(gp);
      float a1 = 0.f, a2 = 0.f;
#pragma unroll
      for (int o = 0; o < kTfD; ++o) {
        a1 += __shfl_sync(0xffffffffu, dg, o) * wgt[o * kTfD + lane];
        a2 += __shfl_sync(0xffffffffu, dv, o) * wvt[o * kTfD + lane];
      }
      dxt = a1 + a2;
    }
    // dx (router + global skip + dx_t) and the input LayerNorm backward
    if (vf.router && M.sk[S_DXR].S != 1)
#pragma unroll
      for (int t = 0; t < kTfT; ++t) dx[t] = split_at(M.sk[S_DXR], planeH, rH + t * kTfD + lane);
    float s1 = 0.f, s2 = 0.f;
#pragma unroll
    for (int t = 0; t < kTfT; ++t) {
      const long long j = rH + t * kTfD + lane;
      float v = dx[t];
      if (vf.global) v = vf.router ? v + dp[t] : dp[t];
      if (t == kTfT - 1) v += dxt;
      dx[t] = v;
      xh[t] = M.a.x_hat[j];
      M.a.tb_dx[j] = v;
      const float gg = v * gin[t * kTfD + lane];
      s1 += gg;
      s2 += gg * xh[t];
    }
    const float m1 = warp_sum(s1) / (float)kTfH, m2 = warp_sum(s2) / (float)kTfH;
    const float xinv = M.a.x_inv[b];
#pragma unroll
    for (int t = 0; t < kTfT; ++t) dx[t] = (dx[t] * gin[t * kTfD + lane] - m1 - xh[t] * m2) * xinv;
    if (vf.local) {
      // dconv (lane = co) staged for the broadcast reads of the input gradient
      float lh[kTfT], li[kTfT];
#pragma unroll
      for (int t = 0; t < kTfT; ++t) {
        const long long j = rH + t * kTfD + lane;
        lh[t] = M.a.loc_hat[j];
        li[t] = M.a.loc_inv[(long long)b * kTfT + t];
        dcw[t * kTfD + lane] = M.a.dh_l[j] * gelu_grad_f(M.a.conv_pre[j]);
      }
      __syncwarp();
      // conv input gradient, lane = ci: output t of tap `tap` read input
      // symbol s = t + tap - 1 (ops.py:74-88)
      float dl[kTfT];
#pragma unroll
      for (int t = 0; t < kTfT; ++t) dl[t] = 0.f;
      const float4* g4 = (const float4*)dcw;
#pragma unroll 1
      for (int c4 = 0; c4 < kTfD / 4; ++c4) {
        float k[kTfK][4];
#pragma unroll
        for (int tap = 0; tap < kTfK; ++tap)
#pragma unroll
          for (int c = 0; c < 4; ++c) k[tap][c] = ckt[(tap * kTfD + 4 * c4 + c) * kTfD + lane];
#pragma unroll
        for (int t = 0; t < kTfT; ++t) {
          const float4 g = g4[t * (kTfD / 4) + c4];
          const float gv[4] = {g.x, g.y, g.z, g.w};
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            if (t >= 1) dl[t - 1] += gv[c] * k[0][c];
            dl[t] += gv[c] * k[1][c];
            if (t + 1 < kTfT) dl[t + 1] += gv[c] * k[2][c];
          }
        }
      }
      // per-symbol LayerNorm backward over D, lane = channel e
#pragma unroll
      for (int t = 0; t < kTfT; ++t) {
        const long long j = rH + t * kTfD + lane;
        M.a.tb_dls[j] = dl[t];
        const float gg = dl[t] * gl;
        const float q1 = warp_sum(gg) / (float)kTfD, q2 = warp_sum(gg * lh[t]) / (float)kTfD;
        dx[t] += (gg - q1 - lh[t] * q2) * li[t];
      }
      __syncwarp();   // dcw is rewritten by the warp's next row
    }
    // embedding gradient (ops.py:234-243 scatter-add), fixed point: the
    // integer sums do not depend on the order the rows arrive in
#pragma unroll
    for (int t = 0; t < kTfT; ++t) {
      const int sy = __shfl_sync(0xffffffffu, sym, t);
      atomicAdd(&eacc[sy * kTfD + lane], (unsigned long long)emb_to_fixed(dx[t]));
      if (lane == 0) touched[sy] = 1;
    }
  }
  __syncthreads();
  for (int j = tid; j < 256 * kTfD; j += blockDim.x)
    if (touched[j / kTfD] && !(M.dbg & 1))
      atomicAdd((unsigned long long*)&M.a.emb_acc[j], eacc[j]);
}

// Small-parameter gradients of the trunk from the rows' saved activations and
// k_trunk_bwd_w's dx / dloc rows: per-CTA sums (rows b = cta, cta + grid, ...)
// into trunk_part[cta] -- one owner thread per column.
// PART 1: conv_k, conv_b, w_gate, w_val (inputs ready after the dx_r / dblock
// GEMM: runs on a second stream beside k_trunk_bwd_w); PART 2: in_g, in_b,
// loc_g, loc_b (needs k_trunk_bwd_w's dx / dloc rows)
constexpr int kTgThreads = 256;
template <int PART>
__global__ void __launch_bounds__(kTgThreads, 4) k_trunk_grads(ModelPtrs M) {
  pdl_enter();
  __shared__ __align__(16) float loc[kTfH], dcv[kTfH], dxr[kTfH], xhr[kTfH], dls[kTfH], lhr[kTfH];
  __shared__ float xt[kTfD], dg[kTfD], dv[kTfD];
  const int tid = threadIdx.x;
  const VFlags vf0 = vflags(M.variant);
  // the flags of what this part computes
  const bool loc_on = vf0.local, glob_on = PART == 1 && vf0.global;
  const bool conv_on = PART == 1 && loc_on, lnl_on = PART == 2 && loc_on;
  const Dims& d = M.d;
  const long long planeD = (long long)d.B * kTfD;
  // conv_k: co = tid % 32, ci = 4 * (tid / 32) + c, all three taps
  const int co = tid & 31, ci0 = 4 * (tid >> 5);
  float ak[kTfK][4] = {}, agv[8] = {}, ain[4] = {};
  float acb = 0.f, alg = 0.f, alb = 0.f;
  // the next row's loads are issued (into registers) before this row's sums:
  // one row's L2 round trip hides behind the previous row's arithmetic
  float r_dx[2], r_xh[2], r_loc[2], r_dh[2], r_cp[2], r_dls[2], r_lh[2];
  float r_gp = 0.f, r_vp = 0.f, r_db = 0.f, r_xt = 0.f;
  auto load = [&](int b) {
    const long long rH = (long long)b * kTfH;
#pragma unroll
    for (int k = 0; k < 2; ++k) {
      const long long j = rH + tid + kTgThreads * k;
      if (PART == 2) {
        r_dx[k] = M.a.tb_dx[j];
        r_xh[k] = M.a.x_hat[j];
      }
      if (conv_on) {
        r_loc[k] = M.a.loc[j];
        r_dh[k] = M.a.dh_l[j];
        r_cp[k] = M.a.conv_pre[j];
      }
      if (lnl_on) {
        r_dls[k] = M.a.tb_dls[j];
        r_lh[k] = M.a.loc_hat[j];
      }
    }
    if (glob_on && tid < kTfD) {
      r_gp = M.a.gpre[(long long)b * kTfD + tid];
      r_vp = M.a.vpre[(long long)b * kTfD + tid];
      r_db = split_at(M.sk[S_DBLOCK], planeD, (long long)b * kTfD + tid);
      r_xt = M.a.x[rH + kTfH - kTfD + tid];
    }
  };
  if ((int)blockIdx.x < d.B) load(blockIdx.x);
  for (int b = blockIdx.x; b < d.B; b += gridDim.x) {
#pragma unroll
    for (int k = 0; k < 2; ++k) {
      const int j = tid + kTgThreads * k;
      if (PART == 2) {
        dxr[j] = r_dx[k];
        xhr[j] = r_xh[k];
      }
      if (conv_on) {
        loc[j] = r_loc[k];
        dcv[j] = r_dh[k] * gelu_grad_f(r_cp[k]);
      }
      if (lnl_on) {
        dls[j] = r_dls[k];
        lhr[j] = r_lh[k];
      }
    }
    if (glob_on && tid < kTfD) {
      dg[tid] = r_db * r_vp * gelu_grad_f(r_gp);
      dv[tid] = r_db * gelu_f(r_gp);
      xt[tid] = r_xt;
    }
    __syncthreads();
    if (b + (int)gridDim.x < d.B) load(b + gridDim.x);
    if (glob_on) {
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const int q = tid + kTgThreads * k, i = q / kTfD, o = q % kTfD;
        agv[k] += xt[i] * dg[o];
        agv[4 + k] += xt[i] * dv[o];
      }
    }
    if (PART == 2)
#pragma unroll
      for (int k = 0; k < 2; ++k) {
        const int j = tid + kTgThreads * k;
        ain[k] += dxr[j] * xhr[j];
        ain[2 + k] += dxr[j];
      }
    if (conv_on) {
      // per row: sum over t ascending of loc[t + tap - 1][ci] * dcv[t][co]
      float r[kTfK][4] = {};
#pragma unroll
      for (int t = 0; t < kTfT; ++t) {
        const float g = dcv[t * kTfD + co];
#pragma unroll
        for (int tap = 0; tap < kTfK; ++tap) {
          const int sidx = t + tap - kTfK / 2;
          if (sidx < 0 || sidx >= kTfT) continue;
          const float4 l = *(const float4*)(loc + sidx * kTfD + ci0);
          r[tap][0] += l.x * g;
          r[tap][1] += l.y * g;
          r[tap][2] += l.z * g;
          r[tap][3] += l.w * g;
        }
      }
#pragma unroll
      for (int tap = 0; tap < kTfK; ++tap)
#pragma unroll
        for (int c = 0; c < 4; ++c) ak[tap][c] += r[tap][c];
      if (tid < kTfD) {
        float cbs = 0.f;
#pragma unroll
        for (int t = 0; t < kTfT; ++t) cbs += dcv[t * kTfD + tid];
        acb += cbs;
      }
    }
    if (lnl_on && tid < kTfD) {
      float s1 = 0.f, s2 = 0.f;
#pragma unroll
      for (int t = 0; t < kTfT; ++t) {
        s1 += dls[t * kTfD + tid] * lhr[t * kTfD + tid];
        s2 += dls[t * kTfD + tid];
      }
      alg += s1;
      alb += s2;
    }
    __syncthreads();   // the next row overwrites the staged rows
  }
  const SmallLayout& L = M.sl;
  float* part = M.a.trunk_part + (long long)blockIdx.x * (L.trunk1 - L.trunk0) - L.trunk0;
  if (PART == 1) {
#pragma unroll
    for (int tap = 0; tap < kTfK; ++tap)
#pragma unroll
      for (int c = 0; c < 4; ++c) part[L.conv_k + tap * kTfD * kTfD + (ci0 + c) * kTfD + co] = ak[tap][c];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      part[L.w_gate + tid + kTgThreads * k] = agv[k];
      part[L.w_val + tid + kTgThreads * k] = agv[4 + k];
    }
    if (tid < kTfD) part[L.conv_b + tid] = acb;
  } else {
#pragma unroll
    for (int k = 0; k < 2; ++k) {
      part[L.in_g + tid + kTgThreads * k] = ain[k];
      part[L.in_b + tid + kTgThreads * k] = ain[2 + k];
    }
    if (tid < kTfD) {
      part[L.loc_g + tid] = alg;
      part[L.loc_b + tid] = alb;
    }
  }
}

bool launch_trunk_bwd_w(const ModelPtrs& M, const uint8_t* src, long long ld_src, int use_col,
                        cudaStream_t s) {
  const Dims& d = M.d;
  if (!trunk_bwd_split(M)) return false;
  const size_t smem = kTbSmemBytes;
  static const cudaError_t attr =
      cudaFuncSetAttribute(k_trunk_bwd_w, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  (void)attr;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int grid = std::min(cdiv(d.B, kTbWarps), 2 * sms);
  launch_pdl(k_trunk_bwd_w, dim3(grid), dim3(32 * kTbWarps), smem, s, M, src, ld_src, use_col);
  launch_pdl(k_trunk_grads<2>, dim3(M.trunk_grid), dim3(kTgThreads), 0, s, M);
  return true;
}

bool trunk_bwd_split(const ModelPtrs& M) {
  const Dims& d = M.d;
  return row_warp_enabled(d.B, 7) && d.D == kTfD && d.T == kTfT && d.K == kTfK && M.a.tb_dx;
}

void launch_trunk_grads_conv(const ModelPtrs& M, cudaStream_t s) {
  launch_pdl(k_trunk_grads<1>, dim3(M.trunk_grid), dim3(kTgThreads), 0, s, M);
}

// dispatch: returns false when the geometry needs the CTA-per-row kernels

#define ROW_LAUNCH(kern)                                                              \
  bool launch_##kern##_w(const ModelPtrs& M, cudaStream_t s) {                         \
    if (M.d.H % 128 || M.d.H > 1024) return false;                                     \
    const dim3 grid(cdiv(M.d.B, kRowWarps)), block(32 * kRowWarps);                    \
    switch (M.d.H / 128) {                                                             \
      case 1: launch_pdl(k_##kern##_w<1>, grid, block, 0, s, M); return true;          \
      case 2: launch_pdl(k_##kern##_w<2>, grid, block, 0, s, M); return true;          \
      case 4: launch_pdl(k_##kern##_w<4>, grid, block, 0, s, M); return true;          \
      case 8: launch_pdl(k_##kern##_w<8>, grid, block, 0, s, M); return true;          \
    }                                                                                  \
    return false;                                                                      \
  }

ROW_LAUNCH(mix_fwd)
ROW_LAUNCH(coarse_fwd)
ROW_LAUNCH(out_fwd)
// the backward kernels carry the combined rowred rows' shared memory (rr_store)
#define ROW_LAUNCH_RR(kern)                                                           \
  bool launch_##kern##_w(const ModelPtrs& M, cudaStream_t s) {                         \
    if (M.d.H % 128 || M.d.H > 1024) return false;                                     \
    const dim3 grid(cdiv(M.d.B, kRowWarps)), block(32 * kRowWarps);                    \
    const size_t sm = M.rr_rows == M.d.B ? 0 : sizeof(float) * kRowWarps * (2 * M.d.H + 4); \
    switch (M.d.H / 128) {                                                             \
      case 1: launch_pdl(k_##kern##_w<1>, grid, block, sm, s, M); return true;         \
      case 2: launch_pdl(k_##kern##_w<2>, grid, block, sm, s, M); return true;         \
      case 4: launch_pdl(k_##kern##_w<4>, grid, block, sm, s, M); return true;         \
      case 8: launch_pdl(k_##kern##_w<8>, grid, block, sm, s, M); return true;         \
    }                                                                                  \
    return false;                                                                      \
  }

ROW_LAUNCH_RR(out_bwd)
ROW_LAUNCH_RR(coarse_bwd)
ROW_LAUNCH_RR(mix_bwd)

}  // namespace fade
