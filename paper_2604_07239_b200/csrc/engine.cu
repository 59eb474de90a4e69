// The FADE step engine: device state, the per-timestep kernel schedule
// (model stream + weight-gradient side stream + CSPP coder stream), CUDA-graph
// replay, and the C ABI of include/fade_b200.h sections 2-3.
//
// One timestep (pipeline.py:211-223 serial order, 251-287 pipelined):
//   forward  : trunk -> {route, mem} GEMMs -> mix -> down GEMM -> bmm ->
//              {up, cgate} GEMMs -> coarse -> e12 GEMM (GeGLU epilogue) ->
//              f GEMM (split-K) -> out -> head GEMM -> head (softmax, quantise,
//              cum slot, [decode], xent)
//   coder    : encode(cum slot) on its own stream, overlapping the backward
//   backward : dX GEMMs + row kernels on the model stream; every dW GEMM (with
//              Adam fused in its epilogue) on a side stream as soon as its
//              input gradient exists and the dX GEMM that reads the old weight
//              is done; small parameters and the embedding last.
#include <chrono>
#include <cstring>
#include <memory>
#include <array>
#include <mutex>
#include <string>
#include <vector>

#include <nvtx3/nvToolsExt.h>   // header-only NVTX v3: ranges for nsys / ncu --nvtx

#include "../../include/fade_b200.h"
#include "model.cuh"
#include "stream_coder.cuh"

namespace fade {

#define TRY(expr)                    \
  do {                               \
    int _s = (expr);                 \
    if (_s != FADE_OK) return _s;    \
  } while (0)

static int cuda_fail(cudaError_t e, const char* what) {
  if (e == cudaSuccess) return FADE_OK;
  set_last_error(std::string(what) + ": " + cudaGetErrorString(e));
  return FADE_ERR_CUDA;
}
#define CK(expr) TRY(cuda_fail((expr), #expr))
// the ABI call runs on this device; the caller's current device is restored
#define ON_DEVICE(dev)          \
  DeviceScope _dscope(dev);     \
  CK(_dscope.status)

static size_t align_up(size_t n, size_t a) { return (n + a - 1) / a * a; }

struct DevArena {            // one cudaMalloc carved into 256-byte aligned pieces
  char* base = nullptr;
  size_t used = 0, cap = 0;
  std::vector<std::pair<size_t, size_t>> pending;
  size_t reserve(size_t bytes) {
    const size_t off = align_up(used, 256);
    used = off + bytes;
    return off;
  }
};

enum GemmId {
  G_ROUTE_MEM, G_DOWN, G_UP_CGATE, G_E12, G_F, G_HEAD,          // forward
  G_DH, G_DWIDE, G_DZ2, G_DU_DHMC, G_DZ, G_DXR_DBLOCK,          // input gradients
  G_WHEAD, G_WF, G_W12, G_WUP_WCGATE, G_WDOWN, G_WROUTE_WMEM,   // weight gradients + Adam
  G_COUNT
};

}  // namespace fade

using namespace fade;

// Device allocations come from the stream-ordered pool, which keeps freed
// memory for reuse: a plain cudaFree can stall for 100+ ms (it synchronises and
// unmaps), which showed up as a variable per-call cost in compress_bytes.
static cudaError_t dev_alloc(void** p, size_t bytes, cudaStream_t s) {
  static std::mutex mu;
  static std::vector<bool> done;   // per device: release threshold raised
  int dev = 0;
  if (cudaGetDevice(&dev) == cudaSuccess) {
    std::lock_guard<std::mutex> lk(mu);
    if ((int)done.size() <= dev) done.resize(dev + 1, false);
    cudaMemPool_t pool;
    if (!done[dev] && cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
      uint64_t keep = ~0ull;
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
      done[dev] = true;
    }
  }
  return cudaMallocAsync(p, bytes, s);
}
static void dev_free(void* p, cudaStream_t s) {
  if (p) cudaFreeAsync(p, s);
}

struct fade_model {
  fade_config_t cfg;
  long long step_offset = 0;    // column - Predictor.step_count of the running call
  Dims d;
  SmallLayout sl;
  int device = 0;
  cudaStream_t s_main = nullptr, s_side = nullptr, s_coder = nullptr;
  cudaStream_t s_side2 = nullptr;   // second weight-update stream (side2_mask)
  cudaEvent_t ev_side2_done = nullptr;
  cudaEvent_t ev_tg[2] = {};        // large-B trunk weight gradients on s_side2: fork / join
  cudaEvent_t ev[8] = {};
  cudaEvent_t ev_cum[2] = {}, ev_enc[2] = {}, ev_side_done = nullptr, ev_coder_join = nullptr;
  cudaEvent_t ev_wu[2] = {};    // W_U update forked off the model stream (experiments)
  void* mem = nullptr;
  ModelPtrs M;
  StepState* st = nullptr;      // device
  GemmParams G[G_COUNT];        // step schedule (Adam fused into dW epilogues)
  GemmParams Gg[G_COUNT];       // loss_grads variant (dW epilogues store gradients)
  int bn[G_COUNT];
  const uint8_t* bench_src = nullptr;   // last fade_bench_compress_steps input (probe)
  long long bench_L = 0;
  uint8_t* ctx_buf = nullptr;   // [B][T]  (predict API)
  uint8_t* tgt_buf = nullptr;   // [B]
  double* loss_buf = nullptr;   // [1]
  // cache snapshots (cache [B][C] + ring position): [0] the state before the
  // last predict (restored when it fails, replayed when a test hook ran in
  // between), [1] the state around forward_debug / loss_grads
  float* cache_snap[2] = {};
  long long* ring_snap[2] = {};
  uint8_t* live_ctx = nullptr;  // [B][T] context of the pending predict
  float* w12_g = nullptr;
  bool live = false;            // a predict is pending train_step
  int launches_per_step = 0;
  // fade_bench_compress_steps: the captured timestep, owned by this model (a
  // cache keyed by the model's address replayed a destroyed model's graph when
  // a new model reused the address) and tied to the coder it was captured with
  cudaGraphExec_t bench_exec = nullptr;    // steps_per_graph() timesteps
  cudaGraphExec_t bench_exec1 = nullptr;   // one timestep
  const void* bench_coder = nullptr;
  size_t l2_window_max = 0, l2_persist = 0;   // access-policy window cap, persisting carve-out
};

struct fade_coder {
  int B = 0;
  int device = 0;
  long long L = 0, cap = 0;
  void* mem = nullptr;
  EncState e{};
  std::vector<long long> lengths;
  cudaStream_t s = nullptr;
  ~fade_coder() {   // every exit path, the error paths of fade_compress included
    if (!mem) return;
    DeviceScope ds(device);
    cudaFreeAsync(mem, s);
    cudaStreamSynchronize(s);
  }
};

namespace fade {

// ---------------------------------------------------------------------------
// allocation

static SmallLayout make_small_layout(const Dims& d) {
  SmallLayout s;
  int o = 0;
  s.out_g = o; o += d.H;  s.out_b = o; o += d.H;
  s.ref_g = o; o += d.H;  s.ref_b = o; o += d.H;
  s.mix_g = o; o += d.H;  s.mix_b = o; o += d.H;
  s.in_g = o;  o += d.H;  s.in_b = o;  o += d.H;
  s.loc_g = o; o += d.D;  s.loc_b = o; o += d.D;  s.conv_b = o; o += d.D;
  s.conv_k = o; o += d.K * d.D * d.D;
  s.w_gate = o; o += d.D * d.D;  s.w_val = o; o += d.D * d.D;
  s.trunk0 = s.in_g;
  s.trunk1 = o;   // in_g, in_b, loc_g, loc_b, conv_b, conv_k, w_gate, w_val
  s.lam_out = o++; s.lam_mix = o++; s.lam_mem = o++;
  // rowred rows start 16-byte aligned (the warp-per-row kernels store float4s);
  // the 0-3 padding slots stay zero: zero gradient, Adam leaves them at 0
  o = (o + 3) / 4 * 4;
  s.rowred = o;
  s.b_head = o; o += 256;
  s.total = o;
  return s;
}

// element count of parameter i in the reference layout
static long long ref_numel(const Dims& d, int i) {
  switch (i) {
    case P_EMB: return 256LL * d.D;
    case P_IN_LN_G: case P_IN_LN_B: case P_MIX_LN_G: case P_MIX_LN_B: case P_REF_LN_G:
    case P_REF_LN_B: case P_OUT_LN_G: case P_OUT_LN_B: return d.H;
    case P_W_GATE: case P_W_VAL: return (long long)d.D * d.D;
    case P_W_MEM: return (long long)d.C * d.H;
    case P_LAM_MEM: case P_LAM_MIX: case P_LAM_OUT: return 1;
    case P_LOC_LN_G: case P_LOC_LN_B: case P_CONV_B: return d.D;
    case P_CONV_K: return (long long)d.K * d.D * d.D;
    case P_W_ROUTE: case P_W_CGATE: return (long long)d.H * d.H;
    case P_W_DOWN: case P_W_UP: return (long long)d.H * d.X;
    case P_W_MIX: return (long long)d.B * d.X * d.X;
    case P_W_E1: case P_W_E2: return (long long)d.H * d.E;
    case P_W_F: return (long long)d.E * d.H;
    case P_W_HEAD: return (long long)d.H * 256;
    case P_B_HEAD: return 256;
  }
  return 0;
}

static int small_offset(const SmallLayout& s, int i) {
  switch (i) {
    case P_OUT_LN_G: return s.out_g;  case P_OUT_LN_B: return s.out_b;
    case P_REF_LN_G: return s.ref_g;  case P_REF_LN_B: return s.ref_b;
    case P_MIX_LN_G: return s.mix_g;  case P_MIX_LN_B: return s.mix_b;
    case P_IN_LN_G: return s.in_g;    case P_IN_LN_B: return s.in_b;
    case P_LOC_LN_G: return s.loc_g;  case P_LOC_LN_B: return s.loc_b;
    case P_CONV_B: return s.conv_b;   case P_CONV_K: return s.conv_k;
    case P_W_GATE: return s.w_gate;   case P_W_VAL: return s.w_val;
    case P_LAM_OUT: return s.lam_out; case P_LAM_MIX: return s.lam_mix;
    case P_LAM_MEM: return s.lam_mem; case P_B_HEAD: return s.b_head;
  }
  return -1;
}

constexpr int kWideBN = 256;

// split-K count: as many slices as fit in ONE wave of 148 SMs (a second,
// partial wave doubles the kernel time), each slice at least 4 k-tiles
static int choose_splits(int tiles, int k_tiles) {
  int s = 148 / std::max(1, tiles);
  s = std::max(1, std::min(s, k_tiles / 4));
  return s;
}

// Split-K factors of one launch group of narrow (64-wide tile) GEMMs:
// repeatedly double the split of the problem with the most k-tiles per CTA
// while the group stays within one wave of 148 CTAs and every slice keeps at
// least 2 k-tiles.
struct SplitPlan {
  int id;
  long long M, N, K;
};
static void plan_splits(ModelPtrs& M, std::initializer_list<SplitPlan> group) {
  std::vector<SplitPlan> g(group);
  std::vector<int> S(g.size(), 1);
  auto tiles = [](const SplitPlan& p) { return (int)(cdiv(p.M, kBM) * cdiv(p.N, 64)); };
  // slices the GEMM actually makes of kt k-tiles for a requested s (gemm_setup)
  auto made = [](int kt, int s) { return (int)cdiv(kt, cdiv(kt, s)); };
  int total = 0;
  for (auto& p : g) total += tiles(p);
  for (;;) {
    // give one more slice to the problem with the longest per-CTA K, while the
    // launch stays within one wave and every slice keeps >= 2 k-tiles
    int best = -1, best_per = 0, best_s = 0;
    for (size_t i = 0; i < g.size(); ++i) {
      const int kt = (int)cdiv(g[i].K, kBK);
      int s = S[i] + 1;
      while (s <= kt && made(kt, s) != s) ++s;      // next slice count the GEMM realises
      if (s > kt || cdiv(kt, s) < 2 || total + tiles(g[i]) * (s - S[i]) > 148) continue;
      const int per = (int)cdiv(kt, S[i]);
      if (per > best_per) {
        best_per = per;
        best = (int)i;
        best_s = s;
      }
    }
    if (best < 0) break;
    total += tiles(g[best]) * (best_s - S[best]);
    S[best] = best_s;
  }
  for (size_t i = 0; i < g.size(); ++i) M.sk[g[i].id].S = S[i];
}

struct Builder {
  GemmParams* G;
  int BN;
  int weight_b;   // forward / input-gradient group: B is a parameter (GemmProblem::b_pre)
  int add(GemmDesc d) {
    if (G->nprob >= kMaxProblems) {
      set_last_error("too many GEMM problems in one group");
      return FADE_ERR_USAGE;
    }
    d.pair = G->pair;
    d.b_pre = weight_b;
    return gemm_setup(&G->prob[G->nprob++], d, BN);
  }
};

static GemmDesc gd(const float* A, long long lda, int at, const float* B, long long ldb, int bt,
                   int M, int N, int K, int epi, float* C, long long ldc) {
  GemmDesc g{};
  g.A = A; g.lda = lda; g.a_trans = at;
  g.B = B; g.ldb = ldb; g.b_trans = bt;
  g.M = M; g.N = N; g.K = K;
  g.splits = 1;
  g.epi = epi;
  g.C = C; g.ldc = ldc;
  return g;
}

// grad_only = true builds the loss_grads variant: weight-gradient GEMMs store
// the raw gradient into the g buffers instead of applying Adam.
static int build_gemms(fade_model* m, GemmParams* Gs, bool grad_only) {
  const Dims& d = m->d;
  ModelPtrs& M = m->M;
  Acts& a = M.a;
  const int B = d.B, H = d.H, X = d.X, E = d.E, Ep = d.Ep, C = d.C;
  for (int i = 0; i < G_COUNT; ++i) {
    memset(&Gs[i], 0, sizeof(GemmParams));
    m->bn[i] = 64;
    Gs[i].adam = &m->st->adam;
  }
  // wide tiles where N is large or K is long: half the L2 operand re-reads
  m->bn[G_E12] = m->bn[G_ROUTE_MEM] = m->bn[G_F] = m->bn[G_DZ2] = kWideBN;
  // weight-gradient GEMMs and the GeGLU backward: wide tiles too, with their
  // Adam p/m/v (a1/a2) inputs streamed through the idle stages
  m->bn[G_DWIDE] = kWideBN;
  // the big Adam GEMMs: 128-wide tiles at two CTAs per SM, so one CTA's
  // streamed Adam epilogue overlaps the other's mainloop
  static const long occ1_ids = knob("FADE_OCC1") ? atol(knob("FADE_OCC1")) : 0;   // experiments
  for (int id : {G_W12, G_WF, G_WROUTE_WMEM}) {
    m->bn[id] = 128;
    Gs[id].occ = ((occ1_ids >> id) & 1) ? 1 : 2;
  }
  // the backward's narrow GEMMs at half the shared memory (4-stage ring,
  // ~97 KB instead of 8 stages / ~193 KB, or 5 stages + 3 dedicated Adam
  // tiles for W_up): each fits on an SM beside one weight-update CTA instead
  // of waiting for a whole SM.  Input gradients dh, du, dz, dx_r: -5.5 us per
  // step together (du alone +7 us; the forward's narrow GEMMs +3 us); the
  // W_up/W_cgate/W_down update (streamed Adam epilogue then): -4.5 us
  static const long occ2_ids = knob("FADE_OCC2") ? atol(knob("FADE_OCC2"))
                                                   : (1L << G_DH) | (1L << G_DU_DHMC) |
                                                     (1L << G_DZ) | (1L << G_DXR_DBLOCK) |
                                                     (1L << G_WUP_WCGATE);
  for (int id = 0; id < G_COUNT; ++id)
    if (((occ2_ids >> id) & 1) && m->bn[id] == 64) Gs[id].occ = 2;
  // W_route/W_mem update at 64-wide tiles: 288 CTAs fill both per-SM slots
  // (23 -> 16 us alone, -3 us per step); W_f measured slower that way
  static const long bn64_ids = knob("FADE_BN64") ? atol(knob("FADE_BN64"))
                                                   : (1L << G_WROUTE_WMEM);
  for (int id = 0; id < G_COUNT; ++id)
    if ((bn64_ids >> id) & 1) m->bn[id] = 64;
  // B <= 128: the expand GEMM at 128-wide single-CTA tiles (150 tiles over
  // 148 persistent CTAs instead of 75 pair tiles over 74 pairs: the one
  // doubled unit is half as long): -3 us per timestep at B = 64 / 128,
  // +4 / +8 us at B = 256 / 512
  if (M.d.B <= 128) m->bn[G_E12] = 128;
  static const long bn128_ids = knob("FADE_BN128") ? atol(knob("FADE_BN128")) : 0;   // experiments
  for (int id = 0; id < G_COUNT; ++id)
    if ((bn128_ids >> id) & 1) m->bn[id] = 128;
  static const long bn256_ids = knob("FADE_BN256") ? atol(knob("FADE_BN256")) : 0;   // experiments
  for (int id = 0; id < G_COUNT; ++id)
    if ((bn256_ids >> id) & 1) {
      m->bn[id] = 256;
      Gs[id].occ = 1;
    }
  // CTA pairs (cta_group::2, 256-row tiles): half the operand bytes per SM
  // (W12 update, the GeGLU backward and dz2: -15 us per step together; the
  // FNR project GEMM F (split-K 18, 144 CTAs): -1.7 us;
  // neutral or slower for the narrower W_f / W_route / W_mem updates and the
  // other forward GEMMs)
  static const long pair_ids = knob("FADE_PAIR") ? atol(knob("FADE_PAIR"))
                                                   : (1L << G_W12) | (1L << G_DWIDE) |
                                                     (1L << G_DZ2) | (1L << G_F);
  // (experiments: FADE_OCC2P = bit per GemmId, pair GEMMs at two CTAs per SM)
  static const long occ2p_ids = knob("FADE_OCC2P") ? atol(knob("FADE_OCC2P")) : 0;
  for (int id = 0; id < G_COUNT; ++id) {
    if (!((pair_ids >> id) & 1) || m->bn[id] < 128) continue;
    Gs[id].pair = 2;
    if ((occ2p_ids >> id) & 1) Gs[id].occ = 2;
    if (Gs[id].occ == 2) m->bn[id] = 256;   // pair tiles 256 x 256 at two CTAs per SM
  }
  // persistent warp-specialised kernel (gemm_ws.cuh) for the store/GeGLU GEMMs
  // (the FNR expand GEMM: -2.6 us per step; neutral or slower elsewhere)
  static const long ws_ids = knob("FADE_WS") ? atol(knob("FADE_WS")) : (1L << G_E12);
  for (int id = 0; id < G_COUNT; ++id) {
    if (!((ws_ids >> id) & 1)) continue;
    Gs[id].ws = 1;
    if (Gs[id].pair != 2 && m->bn[id] == 256) Gs[id].pair = 2;   // 256-wide needs pairs here
    Gs[id].occ = 1;
  }
  // B of every forward and input-gradient GEMM is a parameter that only a
  // weight-update GEMM forked AFTER it (or the previous step) writes
  static const bool early_b = !knob("FADE_EARLYB") || atoi(knob("FADE_EARLYB")) != 0;
  auto b = [&](int id) { return Builder{&Gs[id], m->bn[id], early_b && id < G_WHEAD ? 1 : 0}; };
  Tensor4* w = M.w;
  // ablation variants (model.py:121-175) drop whole GEMMs; an empty launch
  // group is a no-op
  const VFlags vf = vflags(M.variant);
  float* h_final = vf.fnr ? a.h : (vf.mixer ? a.h_c : a.hm_tc);
  // the cache operand of the W_mem GEMMs is a ring buffer (allocate: ring_on)
  // (the forward GEMM runs before mix_fwd counts this step's roll: bias 1)
  auto ring_operand = [&](GemmDesc& g, int kind) {
    if (!M.ring_on) return;
    g.a_ring = kind;
    g.ring_bias = kind == 1 ? 1 : 0;
    g.ring_len = C;
    g.ring_rows = B;
    g.ring_step = d.D / kBK;
    g.ring = &m->st->ring;
  };
  // narrow GEMMs write split-K slices their consumer reduces (plan_splits)
  auto sk = [&](GemmDesc g, int id) {
    g.C = M.sk[id].ws;
    g.ldc = g.N;
    g.splits = M.sk[id].S;
    return g;
  };
  // forward
  {
    auto bl = b(G_ROUTE_MEM);
    if (vf.router)
      TRY(bl.add(sk(gd(a.x_tc, H, 0, w[P_W_ROUTE].p, H, 0, B, H, H, EPI_STORE, nullptr, 0), S_RPRE)));
    GemmDesc g = gd(a.cache, C, 0, w[P_W_MEM].p, H, 0, B, H, C, EPI_STORE, a.ws_mem, H);
    g.splits = M.splits_mem;
    ring_operand(g, 1);
    if (vf.global) TRY(bl.add(g));
  }
  if (vf.mixer) {
    TRY(b(G_DOWN).add(sk(gd(a.z, H, 0, w[P_W_DOWN].p, X, 0, B, X, H, EPI_STORE, nullptr, 0), S_ZD)));
    auto bl = b(G_UP_CGATE);
    TRY(bl.add(sk(gd(a.u, X, 0, w[P_W_UP].p, H, 0, B, H, X, EPI_STORE, nullptr, 0), S_INNER)));
    if (vf.gate)
      TRY(bl.add(sk(gd(a.hm_tc, H, 0, w[P_W_CGATE].p, H, 0, B, H, H, EPI_STORE, nullptr, 0), S_CPRE)));
  }
  if (vf.fnr) {
    GemmDesc g = gd(a.z2, H, 0, w[P_W_E1].p, 2LL * Ep, 0, B, 2 * Ep, H, EPI_GEGLU, a.a12, 2LL * Ep);
    g.aux0 = a.wide;
    g.ld_aux = Ep;
    g.aux_cols = Ep;
    TRY(b(G_E12).add(g));
  }
  if (vf.fnr) {
    GemmDesc g = gd(a.wide, Ep, 0, w[P_W_F].p, H, 0, B, H, E, EPI_STORE, a.ws_f, H);
    g.splits = M.splits_f;
    TRY(b(G_F).add(g));
  }
  {
    GemmDesc g = sk(gd(h_final, H, 0, w[P_W_HEAD].p, 256, 0, B, 256, H, EPI_STORE, nullptr, 0), S_LOGITS);
    g.bias = w[P_B_HEAD].p;
    TRY(b(G_HEAD).add(g));
  }
  // input gradients
  TRY(b(G_DH).add(sk(gd(a.dlogits, 256, 0, w[P_W_HEAD].p, 256, 1, B, H, 256, EPI_STORE, nullptr, 0), S_DH)));
  if (vf.fnr) {
    GemmDesc g = gd(a.dnpre, H, 0, w[P_W_F].p, H, 1, B, E, H, EPI_GEGLU_BWD, a.da12, 2LL * Ep);
    g.aux1 = a.a12;
    g.ld_aux = 2LL * Ep;
    g.c_cols = 2LL * Ep;
    g.aux_cols = 2LL * Ep;
    // W_f has E rows; rows [E, Ep) read as zeros through the TMA bounds, and the
    // tiles cover whole 64-column interleave blocks of dA12
    TRY(b(G_DWIDE).add(g));
    Gs[G_DWIDE].prob[0].N = Ep;
    Gs[G_DWIDE].prob[0].tiles_n = cdiv(Ep, m->bn[G_DWIDE]);
  }
  if (vf.fnr) {
    GemmDesc g = gd(a.da12, 2LL * Ep, 0, w[P_W_E1].p, 2LL * Ep, 1, B, H, 2 * Ep, EPI_STORE, a.ws_dz2, H);
    g.splits = M.splits_dz2;
    TRY(b(G_DZ2).add(g));
  }
  if (vf.mixer) {
    auto bl = b(G_DU_DHMC);
    TRY(bl.add(sk(gd(a.dinner, H, 0, w[P_W_UP].p, H, 1, B, X, H, EPI_STORE, nullptr, 0), S_DU)));
    if (vf.gate)
      TRY(bl.add(sk(gd(a.dcpre, H, 0, w[P_W_CGATE].p, H, 1, B, H, H, EPI_STORE, nullptr, 0), S_DHMC)));
    TRY(b(G_DZ).add(sk(gd(a.dzd, X, 0, w[P_W_DOWN].p, X, 1, B, H, X, EPI_STORE, nullptr, 0), S_DZ)));
  }
  {
    auto bl = b(G_DXR_DBLOCK);
    if (vf.router)
      TRY(bl.add(sk(gd(a.drpre, H, 0, w[P_W_ROUTE].p, H, 1, B, H, H, EPI_STORE, nullptr, 0), S_DXR)));
    if (vf.global)
      TRY(bl.add(sk(gd(a.dupre, H, 0, w[P_W_MEM].p + (long long)(C - d.D) * H, H, 1, B, d.D, H,
                       EPI_STORE, nullptr, 0), S_DBLOCK)));
  }
  // weight gradients with the Adam step fused into the epilogue
  auto adam = [&](GemmDesc g, const Tensor4& t) {
    if (grad_only) {
      g.epi = EPI_GRAD;
      g.C = t.g;
    } else {
      g.C = t.p;
      g.aux0 = t.m;
      g.aux2 = t.v;
    }
    return g;
  };
  // Adam GEMMs whose p/m/v are pulled into L2 before their mainloop: the
  // W_route/W_mem update, which ends the step beside the latency-bound
  // trunk_bwd / small_adam while HBM has room (B = 512 -1.2 us per timestep,
  // early and steady state); the W12 / W_f / W_up-group updates run beside
  // the HBM-heavy chain and measured slower with it (profiles/r2_experiments.md).
  // (experiments: FADE_ADAM_PF = bit per GemmId)
  static const long pf_ids = knob("FADE_ADAM_PF") ? atol(knob("FADE_ADAM_PF"))
                                                   : (1L << G_WROUTE_WMEM);
  auto pf = [&](GemmDesc g, int id) {
    if ((pf_ids >> id) & 1) g.l2_pf = 1 << 20;   // every chunk of the tile
    return g;
  };
  // W_head rides in the W_f launch and W_down in the W_up/W_cgate launch:
  // fewer side-stream kernels (each costs a fixed ~10 us of latency)
  // (experiments: FADE_MERGE_WF=1 puts W_head + W_f into the W12 launch, so
  // their tiles follow W12's on the SMs it frees instead of queueing behind
  // the model stream's kernels)
  static const bool merge_wf = knob("FADE_MERGE_WF") && atoi(knob("FADE_MERGE_WF")) != 0;
  if (vf.fnr)
    TRY(b(G_W12).add(pf(adam(gd(a.z2, H, 1, a.da12, 2LL * Ep, 0, H, 2 * Ep, B, EPI_ADAM, nullptr, 2LL * Ep), w[P_W_E1]), G_W12)));
  {
    auto bl = b(merge_wf && vf.fnr ? G_W12 : G_WF);
    TRY(bl.add(pf(adam(gd(h_final, H, 1, a.dlogits, 256, 0, H, 256, B, EPI_ADAM, nullptr, 256), w[P_W_HEAD]), G_WF)));
    if (vf.fnr)
      TRY(bl.add(pf(adam(gd(a.wide, Ep, 1, a.dnpre, H, 0, E, H, B, EPI_ADAM, nullptr, H), w[P_W_F]), G_WF)));
  }
  if (vf.mixer) {
    auto bl = b(G_WUP_WCGATE);
    TRY(bl.add(pf(adam(gd(a.u, X, 1, a.dinner, H, 0, X, H, B, EPI_ADAM, nullptr, H), w[P_W_UP]), G_WUP_WCGATE)));
    if (vf.gate)
      TRY(bl.add(pf(adam(gd(a.hm_tc, H, 1, a.dcpre, H, 0, H, H, B, EPI_ADAM, nullptr, H), w[P_W_CGATE]), G_WUP_WCGATE)));
    TRY(bl.add(pf(adam(gd(a.z, H, 1, a.dzd, X, 0, H, X, B, EPI_ADAM, nullptr, X), w[P_W_DOWN]), G_WUP_WCGATE)));
  }
  {
    auto bl = b(G_WROUTE_WMEM);
    if (vf.router)
      TRY(bl.add(pf(adam(gd(a.x_tc, H, 1, a.drpre, H, 0, H, H, B, EPI_ADAM, nullptr, H), w[P_W_ROUTE]), G_WROUTE_WMEM)));
    if (vf.global) {
      GemmDesc g = gd(a.cache, C, 1, a.dupre, H, 0, C, H, B, EPI_ADAM, nullptr, H);
      ring_operand(g, 2);
      TRY(bl.add(pf(adam(g, w[P_W_MEM]), G_WROUTE_WMEM)));
    }
  }
  return FADE_OK;
}

// FADE_DBG_SKIP (1 side-stream, 2 model-stream GEMMs) and FADE_DBG_SKIPID (a
// bit per GemmId) drop GEMM launches to measure what each costs on the
// critical path.  Timing experiments only: the results are wrong.
// (experiments build only: the shipped library never skips work)
static int run_gemm(fade_model* m, int id, cudaStream_t s, bool grad_only = false) {
#ifdef FADE_EXPERIMENTS
  static const int dbg_skip = knob("FADE_DBG_SKIP") ? atoi(knob("FADE_DBG_SKIP")) : 0;
  static const long dbg_ids = knob("FADE_DBG_SKIPID") ? atol(knob("FADE_DBG_SKIPID")) : 0;
  static std::once_flag warned;
  if (dbg_skip || dbg_ids)
    std::call_once(warned, [] {
      fprintf(stderr, "[fade] FADE_DBG_SKIP/FADE_DBG_SKIPID set: GEMMs are skipped, results are invalid\n");
    });
  if ((dbg_skip & 1) && (s == m->s_side || s == m->s_side2)) return FADE_OK;
  if ((dbg_skip & 2) && s != m->s_side && s != m->s_side2) return FADE_OK;
  if (dbg_ids & (1L << id)) return FADE_OK;
#endif
  return gemm_launch(grad_only ? m->Gg[id] : m->G[id], m->bn[id], s);
}

static int allocate(fade_model* m) {
  const Dims& d = m->d;
  const long long B = d.B, H = d.H, X = d.X, Ep = d.Ep, C = d.C;
  ModelPtrs& M = m->M;
  memset(&M, 0, sizeof(M));
  M.d = d;
  M.sl = m->sl;
  // split-K factors sized to ~one wave of 148 SMs (kWideBN tiles)
  const int tiles = cdiv(B, kBM) * cdiv(H, kWideBN);
  M.splits_mem = choose_splits(tiles, cdiv(C, kBK));
  // F and dz2 capped: below B = 512 one wave of slices writes as many
  // partial-plane bytes as the GEMM reads weight bytes, and the row kernel
  // after it reads them all back (B = 64 / 128 / 256, F: 74 / 74 / 37 slices
  // -> 18 and dz2 74 / 74 / 37 -> 36 / 36 / 18: -6 / -18 / -4 us per
  // timestep; B = 512 keeps 18 / 18)
  M.splits_f = std::min(choose_splits(tiles, cdiv(d.E, kBK)), 18);
  if (const char* e = knob("FADE_SPLITS_F")) M.splits_f = std::max(1, atoi(e));   // experiments
  M.splits_dz2 = std::min(choose_splits(tiles, cdiv(2 * Ep, kBK)), B <= 128 ? 36 : 18);
  if (const char* e = knob("FADE_DBG_TRUNK")) M.dbg = atoi(e);   // experiments (invalid results)
  if (const char* e = knob("FADE_SPLITS_MEM")) M.splits_mem = std::max(1, atoi(e));   // experiments
  if (const char* e = knob("FADE_SPLITS_DZ2")) M.splits_dz2 = std::max(1, atoi(e));   // experiments
  // Only the forward's narrow GEMMs split: in the backward the side stream's
  // weight updates hold most SMs, and a 128-CTA input-gradient GEMM waits for
  // slots an 8-40-CTA one slips into (measured: each backward split +2-7 us
  // per step, the forward W_down / W_up+W_cgate splits -4 us)
  for (int k = 0; k < S_COUNT; ++k) M.sk[k].S = 1;
  // the router GEMM (K = H) shares a launch with the split-K W_mem GEMM
  // (K = C / 16 per slice): two slices balance the two
  static const int rsplit = knob("FADE_RPRE_SPLIT") ? atoi(knob("FADE_RPRE_SPLIT")) : 2;
  M.sk[S_RPRE].S = std::max(1, rsplit);
  plan_splits(M, {{S_ZD, B, X, H}});
  plan_splits(M, {{S_INNER, B, H, X}, {S_CPRE, B, H, H}});
  plan_splits(M, {{S_LOGITS, B, 256, H}});     // head GEMM: -2..5 us (dh split: +1 us)
  // (experiments: FADE_BWD_SPLIT = bit mask of backward narrow GEMMs to split:
  // 1 dh, 2 du + dhm_c, 4 dz, 8 dx_r + dblock)
  static const int bwd_split = knob("FADE_BWD_SPLIT") ? atoi(knob("FADE_BWD_SPLIT")) : 0;
  if (bwd_split & 1) plan_splits(M, {{S_DH, B, H, 256}});
  if (bwd_split & 2) plan_splits(M, {{S_DU, B, X, H}, {S_DHMC, B, H, H}});
  if (bwd_split & 4) plan_splits(M, {{S_DZ, B, H, X}});
  if (bwd_split & 8) plan_splits(M, {{S_DXR, B, H, H}, {S_DBLOCK, B, d.D, H}});
  M.variant = m->cfg.variant;
  // the rolling cache as a ring buffer: block writes instead of a (C - D)
  // float roll per row; needs D and B to be whole numbers of 32-float
  // k-tiles so the W_mem GEMMs can rotate their TMA coordinates block by
  // block.  Bit-identical to the roll, but measured slower (B = 512: 341 vs
  // 335.5 us per timestep, same box; B = 1024 / 4096: neutral): the roll's
  // rewrite is cheap (2-3 us of trunk_fwd) and the W_mem GEMMs read the ring
  // operand more slowly (ncu, cold: +1.0 us forward, +3.1 us update), even
  // block-major and with the old blocks prefetched before the dependency
  // wait.  Experiments build: FADE_RING=1 turns it on.
  const bool ring_req = knob("FADE_RING") && atoi(knob("FADE_RING")) != 0;
  M.ring_on = ring_req && (d.D % kBK == 0) && (d.B % kBK == 0) && vflags(m->cfg.variant).global
                  ? 1 : 0;
  M.lr = m->cfg.lr;
  M.beta1 = m->cfg.beta1;
  M.beta2 = m->cfg.beta2;
  M.adam_eps = m->cfg.adam_eps;

  struct Item { void** ptr; size_t bytes; };
  std::vector<Item> items;
  auto F = [&](float** p, long long n) { items.push_back({(void**)p, sizeof(float) * (size_t)n}); };
  // parameters: big tensors get p/m/v/g; small ones live in the small arena
  float* big[P_COUNT][4] = {};
  for (int i = 0; i < P_COUNT; ++i) {
    if (small_offset(m->sl, i) >= 0 || i == P_W_E2) continue;
    long long n = ref_numel(d, i);
    if (i == P_W_E1) n = H * 2 * Ep;   // interleaved W12
    for (int k = 0; k < 4; ++k) F(&big[i][k], n);
  }
  float *sp, *smm, *sv, *sg;
  F(&sp, m->sl.total); F(&smm, m->sl.total); F(&sv, m->sl.total); F(&sg, m->sl.total);
  Acts& a = M.a;
  F(&a.x, B * H); F(&a.x_tc, B * H); F(&a.hm_tc, B * H); F(&a.x_hat, B * H); F(&a.x_inv, B); F(&a.gpre, B * d.D); F(&a.vpre, B * d.D);
  F(&a.loc, B * H); F(&a.loc_hat, B * H); F(&a.loc_inv, B * d.T); F(&a.conv_pre, B * H);
  F(&a.h_l, B * H); F(&a.cache, B * C);
  F(&a.ws_mem, (long long)M.splits_mem * B * H); F(&a.upre, B * H); F(&a.h_g, B * H);
  F(&a.alpha, B * H); F(&a.h_mix, B * H); F(&a.z_hat, B * H); F(&a.z_inv, B); F(&a.z, B * H);
  F(&a.zd, B * X); F(&a.u, B * X); F(&a.inner, B * H); F(&a.gate, B * H);
  F(&a.h_c, B * H); F(&a.z2_hat, B * H); F(&a.z2_inv, B); F(&a.z2, B * H);
  F(&a.a12, B * 2 * Ep); F(&a.wide, B * Ep); F(&a.ws_f, (long long)M.splits_f * B * H);
  F(&a.n_hat, B * H); F(&a.n_inv, B); F(&a.nrm, B * H); F(&a.h, B * H); F(&a.logits, B * 256);
  items.push_back({(void**)&a.probs, sizeof(double) * (size_t)B * 256});
  items.push_back({(void**)&a.cum, sizeof(unsigned) * 2 * (size_t)B * kCumLd});
  items.push_back({(void**)&a.nll, sizeof(double) * (size_t)B});
  F(&a.alpha_row, B * 3);
  F(&a.dlogits, B * 256); F(&a.dhc, B * H); F(&a.dnpre, B * H);
  F(&a.da12, B * 2 * Ep); F(&a.ws_dz2, (long long)M.splits_dz2 * B * H); F(&a.dinner, B * H);
  F(&a.dcpre, B * H); F(&a.dzd, B * X);
  F(&a.drpre, B * H); F(&a.dupre, B * H); F(&a.dh_l, B * H); F(&a.dx_part, B * H);
  F(&a.tb_dx, B * H); F(&a.tb_dls, B * H);
  M.rr_rows = rowred_rows((int)B, (int)H);
  F(&a.rowred, (long long)M.rr_rows * m->sl.rowred);
  {
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    M.trunk_grid = (int)std::min<long long>(B, 4LL * sms);
  }
  F(&a.trunk_part, (long long)M.trunk_grid * (m->sl.trunk1 - m->sl.trunk0));
  const long long sk_width[S_COUNT] = {X, H, H, 256, H, X, H, H, H, d.D, H};
  for (int k = 0; k < S_COUNT; ++k) F(&M.sk[k].ws, (long long)M.sk[k].S * B * sk_width[k]);
  items.push_back({(void**)&a.emb_acc, sizeof(long long) * 256 * (size_t)d.D});
  items.push_back({(void**)&m->st, sizeof(StepState)});
  items.push_back({(void**)&m->ctx_buf, (size_t)B * d.T});
  items.push_back({(void**)&m->tgt_buf, (size_t)B});
  items.push_back({(void**)&m->loss_buf, sizeof(double) * 4});
  for (int k = 0; k < 2; ++k) {
    F(&m->cache_snap[k], B * C);
    items.push_back({(void**)&m->ring_snap[k], sizeof(long long)});
  }
  items.push_back({(void**)&m->live_ctx, (size_t)B * d.T});

  size_t total = 0;
  std::vector<size_t> offs;
  for (auto& it : items) {
    total = align_up(total, 256);
    offs.push_back(total);
    total += it.bytes;
  }
  CK(dev_alloc(&m->mem, total, m->s_main));
  CK(cudaMemsetAsync(m->mem, 0, total, m->s_main));
  CK(cudaStreamSynchronize(m->s_main));
  for (size_t k = 0; k < items.size(); ++k) *items[k].ptr = (char*)m->mem + offs[k];

  M.small_p = sp; M.small_m = smm; M.small_v = sv; M.small_g = sg;
  for (int i = 0; i < P_COUNT; ++i) {
    const int so = small_offset(m->sl, i);
    if (so >= 0) {
      M.w[i] = Tensor4{sp + so, smm + so, sv + so, sg + so};
    } else {
      const int src = (i == P_W_E2) ? P_W_E1 : i;   // e1 and e2 share the interleaved W12
      M.w[i] = Tensor4{big[src][0], big[src][1], big[src][2], big[src][3]};
    }
  }
  M.st = m->st;
  StepState init{};
  init.err_key = ~0ull;
  CK(cudaMemcpy(m->st, &init, sizeof(init), cudaMemcpyHostToDevice));
  return FADE_OK;
}

// ---------------------------------------------------------------------------
// the timestep schedule

struct StepIO {
  double* alpha_tape;        // per-step router stats [steps][3] or null
  const uint8_t* src;        // context source (stream matrix or ctx buffer)
  long long ld_src;
  int use_col;               // ctx = src[b, col-T:col] (else src[b, 0:T])
  HeadArgs head;
};

// L2 persistence for the per-stream W_U values (33.5 MB at B = 512, read by
// bmm_fwd and read-modify-written by bmm_bwd every step) in the persisting L2
// carve-out: -3 us per step at B = 256 / 512.  It only pays while W_U is a
// small part of the 126 MB L2: at B = 1024 (67 MB) the step takes 600 instead
// of 532 us and at B = 4096 (268 MB) 2.30 instead of 1.61 ms (the carve-out
// starves every other kernel's L2; bmm_bwd alone runs at 2.7 instead of
// 6.2 TB/s).  Pinning p and m (67 MB) measured +32 us at B = 512.
// Experiments build: FADE_L2PIN=0/1/2 overrides.
constexpr size_t kL2PinMaxBytes = 48ull << 20;
static int l2_pin_mode(const Dims& d) {
  static const int forced = knob("FADE_L2PIN") ? atoi(knob("FADE_L2PIN")) : -1;
  if (forced >= 0) return forced;
  return sizeof(float) * (size_t)d.B * d.X * d.X <= kL2PinMaxBytes ? 1 : 0;
}
struct L2Pin {
  explicit L2Pin(const fade_model* m) {
    const int mode = l2_pin_mode(m->d);
    if (!mode) return;
    const Tensor4& t = m->M.w[P_W_MIX];
    const size_t n = sizeof(float) * (size_t)m->d.B * m->d.X * m->d.X;
    cudaAccessPolicyWindow& w = l2_window();
    w.base_ptr = t.p;
    w.num_bytes = mode == 2 ? (size_t)((char*)t.m - (char*)t.p) + n : n;
    // the window is capped by the device (128 MB on B200); past the persisting
    // carve-out only that fraction of the lines is marked persisting
    w.num_bytes = std::min(w.num_bytes, m->l2_window_max);
    w.hitRatio = w.num_bytes ? std::min(1.0f, (float)m->l2_persist / (float)w.num_bytes) : 0.f;
    w.hitProp = cudaAccessPropertyPersisting;
    w.missProp = cudaAccessPropertyStreaming;
  }
  ~L2Pin() { l2_window().num_bytes = 0; }
};

static int forward(fade_model* m, const StepIO& io, bool with_head) {
  cudaStream_t s = m->s_main;
  const ModelPtrs& M = m->M;
  launch_trunk_fwd(M, io.src, io.ld_src, io.use_col, s);
  TRY(run_gemm(m, G_ROUTE_MEM, s));
  launch_mix_fwd(M, s);
  TRY(run_gemm(m, G_DOWN, s));
  const VFlags vf = vflags(M.variant);
  if (vf.mixer) {
    L2Pin pin(m);
    launch_bmm_fwd(M, s);
  }
  TRY(run_gemm(m, G_UP_CGATE, s));
  if (vf.mixer) launch_coarse_fwd(M, s);
  TRY(run_gemm(m, G_E12, s));
  TRY(run_gemm(m, G_F, s));
  if (vf.fnr) launch_out_fwd(M, s);
  TRY(run_gemm(m, G_HEAD, s));
  if (with_head) launch_head(M, io.head, s);
  CK(cudaGetLastError());
  return FADE_OK;
}

// fork the side stream off the model stream at this point
static int fork_side(fade_model* m, int k, cudaStream_t side) {
  CK(cudaEventRecord(m->ev[k], m->s_main));
  CK(cudaStreamWaitEvent(side, m->ev[k], 0));
  return FADE_OK;
}

// advance = 1: the step counts as trained (the last kernel moves the column
// and the step count; Predictor.train_step semantics, model.py:214)
static int backward(fade_model* m, const StepIO& io, bool grad_only, double* losses, int advance) {
  cudaStream_t s = m->s_main, side = m->s_side;
  const ModelPtrs& M = m->M;
  // side-stream weight updates and the model-stream position after which each
  // is forked (0 dh, 1 out_bwd, 2 dwide, 3 dz2, 4 coarse_bwd, 5 du, 6 bmm_bwd,
  // 7 dz, 8 mix_bwd, 9 dxr, 10 trunk_bwd); earliest legal: WF 1, W12 2, WUP 6,
  // WROUTE 8.  Measured (us/step): W12 after dz2 and W_f/W_head after
  // coarse_bwd (W12 runs first) 373.6; the earliest forks (2,3,7,9) 384.5;
  // W_f first (2,2 / 3,2) 382-386; W12 or W_f after bmm_bwd or later 382-429.
  // (a function-local static initialised once, thread-safely: models may run
  // their steps on several host threads)
  // B >= 2048 (throughput-bound): W_f after dz2 and W12 after du, so the
  // tensor-bound W12 update runs beside the HBM-bound W_U update (bmm_bwd)
  // instead of beside coarse_bwd / du: B = 2048 / 4096 -6 / -16..21 us per
  // timestep (B = 1024: +9 us)
  static const std::array<int, 5> forced = [] {
    std::array<int, 5> a{0, 0, 0, 0, 0};
    if (const char* e = knob("FADE_SCHED"))
      a[4] = sscanf(e, "%d,%d,%d,%d", &a[0], &a[1], &a[2], &a[3]) == 4;
    return a;
  }();
  std::array<int, 4> at{4, 3, 7, 9};
  if (M.d.B >= 2048) at = {3, 5, 7, 9};
  if (forced[4]) at = {forced[0], forced[1], forced[2], forced[3]};
  const int ids[4] = {G_WF, G_W12, G_WUP_WCGATE, G_WROUTE_WMEM};
  // bit k of side2_mask puts update ids[k] on a second side stream, where it
  // overlaps the other updates instead of queueing behind them.  B <= 256:
  // the W_route/W_mem update (the step's last kernel: the side stream, not
  // the model stream, ends a small-B step) -9 / -11 / -4 us per timestep at
  // B = 64 / 128 / 256; B = 512: +10 us (it then competes with trunk_bwd).
  // Experiments: FADE_SIDE2 = mask.
  static const int side2_env = knob("FADE_SIDE2") ? atoi(knob("FADE_SIDE2")) : -1;
  const int side2_mask = side2_env >= 0 ? side2_env : (M.d.B <= 256 ? 8 : 0);
  bool used2 = false;
  int pos = 0;
  auto sides = [&]() -> int {
    bool forked[2] = {false, false};
    for (int k = 0; k < 4; ++k) {
      if (at[k] != pos) continue;
      const int j = (side2_mask >> k) & 1;
      cudaStream_t ss = j ? m->s_side2 : side;
      if (!forked[j]) TRY(fork_side(m, pos % 8, ss));
      forked[j] = true;
      used2 |= j != 0;
      TRY(run_gemm(m, ids[k], ss, grad_only));
    }
    ++pos;
    return FADE_OK;
  };
  // the Adam step counter and bias-correction scalars were prepared by the
  // head kernel (HeadArgs.adam_prep); the last kernel advances the column
  const VFlags vf = vflags(M.variant);
  TRY(run_gemm(m, G_DH, s));
  TRY(sides());
  if (vf.fnr) launch_out_bwd(M, s);
  TRY(sides());
  TRY(run_gemm(m, G_DWIDE, s));
  TRY(sides());
  TRY(run_gemm(m, G_DZ2, s));
  TRY(sides());
  if (vf.mixer) launch_coarse_bwd(M, s);
  TRY(sides());
  TRY(run_gemm(m, G_DU_DHMC, s));
  TRY(sides());
  // fused dzd + W_U Adam (mode 3): measured faster than moving the 201 MB W_U
  // RMW to the side stream (it then contends with the critical path for HBM)
  // (experiments: FADE_WU_STREAM=1 / 2 keeps only the input gradient dzd on
  // the model stream and runs the W_U read-modify-write on the coder / side
  // stream, joined at the end of the step)
  static const int wu_stream = knob("FADE_WU_STREAM") ? atoi(knob("FADE_WU_STREAM")) : 0;
  bool wu_forked = false;
  if (vf.mixer) {
    L2Pin pin(m);
    if (wu_stream) {
      launch_bmm_bwd(M, grad_only, 1, s);
      cudaStream_t ws = wu_stream == 1 ? m->s_coder : side;
      CK(cudaEventRecord(m->ev_wu[0], s));
      CK(cudaStreamWaitEvent(ws, m->ev_wu[0], 0));
      launch_bmm_bwd(M, grad_only, 2, ws);
      CK(cudaEventRecord(m->ev_wu[1], ws));
      wu_forked = true;
    } else {
      launch_bmm_bwd(M, grad_only, 3, s);
    }
  }
  TRY(sides());
  TRY(run_gemm(m, G_DZ, s));
  TRY(sides());
  launch_mix_bwd(M, s);
  TRY(sides());
  TRY(run_gemm(m, G_DXR_DBLOCK, s));
  TRY(sides());
  // large B: the conv / GeGLU weight gradients of the trunk need only the
  // dx_r / dblock GEMM's outputs -- on the second side stream beside the
  // trunk input-gradient chain, joined before small_adam
  const bool tsplit = trunk_bwd_split(M);
  if (tsplit) {
    CK(cudaEventRecord(m->ev_tg[0], s));
    CK(cudaStreamWaitEvent(m->s_side2, m->ev_tg[0], 0));
    launch_trunk_grads_conv(M, m->s_side2);
    CK(cudaEventRecord(m->ev_tg[1], m->s_side2));
  }
  launch_trunk_bwd(M, io.src, io.ld_src, io.use_col, s);
  TRY(sides());
  if (tsplit) CK(cudaStreamWaitEvent(s, m->ev_tg[1], 0));
  launch_small_adam(M, grad_only, losses, io.alpha_tape, advance, s);
  CK(cudaEventRecord(m->ev_side_done, side));
  CK(cudaStreamWaitEvent(s, m->ev_side_done, 0));
  if (used2) {
    CK(cudaEventRecord(m->ev_side2_done, m->s_side2));
    CK(cudaStreamWaitEvent(s, m->ev_side2_done, 0));
  }
  if (wu_forked) CK(cudaStreamWaitEvent(s, m->ev_wu[1], 0));
  CK(cudaGetLastError());
  return FADE_OK;
}

static int check_error(fade_model* m, fade_error_t* err) {
  unsigned long long key = 0;
  CK(cudaMemcpy(&key, &m->st->err_key, sizeof(key), cudaMemcpyDeviceToHost));
  if (key == ~0ull) return FADE_OK;
  const int code = (int)(key & 7);
  const long long stream = (long long)((key >> 3) & ((1ull << 21) - 1));
  const long long step = (long long)(key >> 24);
  int kind = FADE_ERR_CORRUPT, why = 0;
  const char* msg = "";
  switch (code) {
    case 1: kind = FADE_ERR_CORRUPT; why = 1; msg = "invalid code value"; break;
    case 2: kind = FADE_ERR_CORRUPT; why = 2; msg = "truncated stream"; break;
    case 3: kind = FADE_ERR_DIVERGED; msg = "non-finite value in forward output"; break;
    case 4: kind = FADE_ERR_QUANT; msg = "row does not sum to 1 within quantizer tolerance"; break;
    case 5: kind = FADE_ERR_DIVERGED; msg = "non-finite loss"; break;
    case 6: kind = FADE_ERR_CORRUPT; why = 2; msg = "stream shorter than coder tail"; break;
  }
  if (err) {
    err->kind = kind;
    err->why = why;
    err->stream = stream;
    // errors are keyed by column so the earliest one in time wins; a coder
    // error reports the column (coder.py:85-86,117-128), a divergence the
    // model's step_count at that column (model.py:190-193,208-209), which in
    // the executors is column - warm
    err->step = code == 6 ? -1 : (kind == FADE_ERR_DIVERGED ? step - m->step_offset : step);
  }
  set_last_error(msg);
  // reset so the model object stays usable after the caller handles the error
  unsigned long long none = ~0ull;
  CK(cudaMemcpy(&m->st->err_key, &none, sizeof(none), cudaMemcpyHostToDevice));
  return kind;
}

// position the device step state at column `col`; losses[0] is the loss of
// column loss_base.  step_count (Predictor.step_count) is unchanged, so the
// divergence report maps a column back to it through step_offset.
static int set_col(fade_model* m, long long col, long long loss_base) {
  long long v[2] = {col, loss_base}, sc = 0;
  CK(cudaMemcpyAsync(&m->st->col, &v[0], sizeof(long long), cudaMemcpyHostToDevice, m->s_main));
  CK(cudaMemcpyAsync(&m->st->loss_base, &v[1], sizeof(long long), cudaMemcpyHostToDevice, m->s_main));
  CK(cudaMemcpyAsync(&sc, &m->st->step_count, sizeof(long long), cudaMemcpyDeviceToHost, m->s_main));
  CK(cudaStreamSynchronize(m->s_main));
  m->step_offset = col - sc;
  return FADE_OK;
}

// the cache (and its ring position) before a call that must leave no trace:
// forward_debug, loss_grads, a predict that fails
static int snapshot_cache(fade_model* m, int k) {
  const size_t cbytes = sizeof(float) * m->d.B * m->d.C;
  CK(cudaMemcpyAsync(m->cache_snap[k], m->M.a.cache, cbytes, cudaMemcpyDeviceToDevice, m->s_main));
  CK(cudaMemcpyAsync(m->ring_snap[k], &m->st->ring, sizeof(long long), cudaMemcpyDeviceToDevice,
                     m->s_main));
  return FADE_OK;
}
static int restore_cache(fade_model* m, int k) {
  const size_t cbytes = sizeof(float) * m->d.B * m->d.C;
  CK(cudaMemcpyAsync(m->M.a.cache, m->cache_snap[k], cbytes, cudaMemcpyDeviceToDevice, m->s_main));
  CK(cudaMemcpyAsync(&m->st->ring, m->ring_snap[k], sizeof(long long), cudaMemcpyDeviceToDevice,
                     m->s_main));
  return FADE_OK;
}
// the Predictor API's step input: the context uploaded to ctx_buf
static StepIO api_io(fade_model* m) {
  StepIO io{};
  io.src = m->ctx_buf;
  io.ld_src = m->d.T;
  io.use_col = 0;
  return io;
}
// A test hook (forward_debug, loss_grads) ran between predict and
// train_step and overwrote the saved activations; the reference keeps its
// live graph (model.py:195-200, 217-237).  Re-run the pending predict from
// its saved state: same inputs, same kernels, so the activations are
// bit-identical to the original ones.
static int replay_live(fade_model* m) {
  if (!m->live) return FADE_OK;
  TRY(restore_cache(m, 0));
  CK(cudaMemcpyAsync(m->ctx_buf, m->live_ctx, (size_t)m->d.B * m->d.T, cudaMemcpyDeviceToDevice,
                     m->s_main));
  StepIO io = api_io(m);
  io.head.want_probs = 1;
  TRY(forward(m, io, true));
  return FADE_OK;
}

// NVTX range over a scope (profiler ranges per phase of
// the executors -- upload, warm-up coding, graph capture, the replayed
// timesteps, flush / decode fetch); free when no tool is attached
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};

// runs a callable when the scope exits (every error path included)
template <class F>
struct Defer {
  F f;
  ~Defer() { f(); }
};
template <class F>
static Defer<F> defer(F f) {
  return Defer<F>{f};
}

// Timesteps per captured graph.  One: several timesteps in one graph measured
// slower than the ~2.5 us launch gap they remove (B = 512: 339.0 us at 1,
// 341.2 / 342.6 / 342.9 at 2 / 4 / 8; B = 64: 230.4 vs 248.9 at 4) -- inside
// one graph the next step's first kernels wait on the join of every stream
// as full dependencies.  Experiments: FADE_STEPS_PER_GRAPH.
static int steps_per_graph() {
  static const int forced = knob("FADE_STEPS_PER_GRAPH") ? atoi(knob("FADE_STEPS_PER_GRAPH")) : 0;
  return forced > 0 ? forced : 1;
}

// Captures `per` consecutive calls of `body` (one timestep each, on the model
// stream; the device-side column counter moves them along) into one graph.
template <class Body>
static int capture_steps(fade_model* m, int per, Body body, cudaGraphExec_t* exec,
                         size_t* nodes = nullptr) {
  cudaGraph_t graph = nullptr;
  auto cleanup = defer([&] {
    if (graph) cudaGraphDestroy(graph);
  });
  CK(cudaStreamBeginCapture(m->s_main, cudaStreamCaptureModeThreadLocal));
  int status = FADE_OK;
  for (int k = 0; k < per && status == FADE_OK; ++k) status = body();
  const cudaError_t ce = cudaStreamEndCapture(m->s_main, &graph);
  if (status != FADE_OK) return status;
  CK(ce);
  CK(cudaGraphInstantiate(exec, graph, 0));
  if (nodes) CK(cudaGraphGetNodes(graph, nullptr, nodes));
  return FADE_OK;
}

// Replays `body` (one timestep) n times through graphs of steps_per_graph()
// timesteps plus one graph for the remainder.  The event tape pointer rides
// in the captured kernel parameters only.
template <class Body>
static int replay_steps(fade_model* m, long long n, unsigned long long* tape, Body body) {
  cudaGraphExec_t exec = nullptr, rest = nullptr;
  auto cleanup = defer([&] {
    if (exec) cudaGraphExecDestroy(exec);
    if (rest) cudaGraphExecDestroy(rest);
  });
  const int per = (int)std::max<long long>(1, std::min<long long>(steps_per_graph(), n));
  const long long full = n / per, rem = n % per;
  m->M.tape = tape;
  {
    NvtxRange r("fade: capture timestep graph");
    auto untape = defer([&] { m->M.tape = nullptr; });
    TRY(capture_steps(m, per, body, &exec));
    if (rem) TRY(capture_steps(m, (int)rem, body, &rest));
  }
  NvtxRange r("fade: timesteps (graph replays)");
  for (long long i = 0; i < full; ++i) CK(cudaGraphLaunch(exec, m->s_main));
  if (rem) CK(cudaGraphLaunch(rest, m->s_main));
  CK(cudaStreamSynchronize(m->s_main));
  return FADE_OK;
}

}  // namespace fade

// ===========================================================================
// C ABI
extern "C" {

int fade_model_create(const fade_config_t* cfg, int device, fade_model_t** out) {
  *out = nullptr;
  if (cfg->alphabet != 256 || cfg->embed_dim % 4 || cfg->mix_dim % 4 || cfg->expand_dim % 4 ||
      cfg->cache_dim % cfg->embed_dim || cfg->conv_kernel % 2 == 0 || cfg->batch < 1 ||
      cfg->ctx_len < 1) {
    set_last_error("unsupported model geometry for the B200 kernels");
    return FADE_ERR_USAGE;
  }
  if (cfg->variant < 0 || cfg->variant >= V_COUNT) {
    set_last_error("unknown model variant");
    return FADE_ERR_USAGE;
  }
  std::unique_ptr<fade_model> m(new fade_model());
  m->cfg = *cfg;
  m->device = device;
  Dims& d = m->d;
  d.B = cfg->batch;
  d.T = cfg->ctx_len;
  d.D = cfg->embed_dim;
  d.H = cfg->ctx_len * cfg->embed_dim;
  d.C = cfg->cache_dim;
  d.X = cfg->mix_dim;
  d.E = cfg->expand_dim;
  d.Ep = (cfg->expand_dim + 63) / 64 * 64;
  d.K = cfg->conv_kernel;
  m->sl = make_small_layout(d);
  ON_DEVICE(device);
  // the model stream is the critical path: its CTAs take SM slots ahead of
  // the side stream's (HBM-bound) weight-update GEMMs when both are pending
  int prio_lo = 0, prio_hi = 0;
  CK(cudaDeviceGetStreamPriorityRange(&prio_lo, &prio_hi));
  static const int dbg_prio = knob("FADE_DBG_PRIO") ? atoi(knob("FADE_DBG_PRIO")) : 1;
  if (!dbg_prio) prio_hi = prio_lo;
  CK(cudaStreamCreateWithPriority(&m->s_main, cudaStreamNonBlocking, prio_hi));
  CK(cudaStreamCreateWithPriority(&m->s_side, cudaStreamNonBlocking, prio_lo));
  CK(cudaStreamCreateWithPriority(&m->s_side2, cudaStreamNonBlocking, prio_lo));
  CK(cudaEventCreateWithFlags(&m->ev_side2_done, cudaEventDisableTiming));
  for (auto& e : m->ev_tg) CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  CK(cudaStreamCreateWithPriority(&m->s_coder, cudaStreamNonBlocking, prio_hi));
  for (auto& e : m->ev) CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  for (int i = 0; i < 2; ++i) {
    CK(cudaEventCreateWithFlags(&m->ev_cum[i], cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&m->ev_enc[i], cudaEventDisableTiming));
  }
  CK(cudaEventCreateWithFlags(&m->ev_side_done, cudaEventDisableTiming));
  CK(cudaEventCreateWithFlags(&m->ev_coder_join, cudaEventDisableTiming));
  for (auto& e : m->ev_wu) CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  TRY(allocate(m.get()));
  if (l2_pin_mode(d)) {
    const size_t want = sizeof(float) * (size_t)d.B * d.X * d.X * (l2_pin_mode(d) == 2 ? 2 : 1);
    int maxp = 0, maxw = 0;
    CK(cudaDeviceGetAttribute(&maxp, cudaDevAttrMaxPersistingL2CacheSize, device));
    CK(cudaDeviceGetAttribute(&maxw, cudaDevAttrMaxAccessPolicyWindowSize, device));
    m->l2_persist = std::min(want, (size_t)maxp);
    m->l2_window_max = (size_t)maxw;
    CK(cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, m->l2_persist));
  }
  TRY(build_gemms(m.get(), m->G, false));
  TRY(build_gemms(m.get(), m->Gg, true));
  *out = m.release();
  return FADE_OK;
}

int fade_model_destroy(fade_model_t* m) {
  if (!m) return FADE_OK;
  DeviceScope dscope(m->device);
  cudaDeviceSynchronize();
  if (m->bench_exec) cudaGraphExecDestroy(m->bench_exec);
  if (m->bench_exec1) cudaGraphExecDestroy(m->bench_exec1);
  if (m->l2_persist) {
    // give the persisting carve-out back: a later, larger model (whose W_U
    // does not fit) must not run with part of L2 set aside
    cudaCtxResetPersistingL2Cache();
    cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, 0);
  }
  dev_free(m->mem, m->s_main);
  cudaStreamSynchronize(m->s_main);
  for (auto& e : m->ev) cudaEventDestroy(e);
  for (int i = 0; i < 2; ++i) {
    cudaEventDestroy(m->ev_cum[i]);
    cudaEventDestroy(m->ev_enc[i]);
  }
  cudaEventDestroy(m->ev_side_done);
  cudaEventDestroy(m->ev_side2_done);
  for (auto& e : m->ev_tg) cudaEventDestroy(e);
  cudaEventDestroy(m->ev_coder_join);
  for (auto& e : m->ev_wu) cudaEventDestroy(e);
  cudaStreamDestroy(m->s_main);
  cudaStreamDestroy(m->s_side);
  cudaStreamDestroy(m->s_side2);
  cudaStreamDestroy(m->s_coder);
  delete m;
  return FADE_OK;
}

static float* tensor_base(fade_model_t* m, int kind, int index) {
  const Tensor4& t = m->M.w[index];
  switch (kind) {
    case 0: return t.p;
    case 1: return t.m;
    case 2: return t.v;
    case 3: return t.g;
  }
  return nullptr;
}

// w_e1 / w_e2 live interleaved in W12 (model.cuh): 64-column blocks
static int copy_w12(fade_model_t* m, float* dev, int which, float* host, bool to_dev) {
  const Dims& d = m->d;
  const size_t dpitch = sizeof(float) * 2 * d.Ep, spitch = sizeof(float) * d.E;
  for (int j = 0; j * 64 < d.E; ++j) {
    const int w = std::min(64, d.E - 64 * j);
    float* dptr = dev + 128 * j + 64 * which;
    float* hptr = host + 64 * j;
    cudaError_t e = to_dev ? cudaMemcpy2D(dptr, dpitch, hptr, spitch, sizeof(float) * w, d.H,
                                          cudaMemcpyHostToDevice)
                           : cudaMemcpy2D(hptr, spitch, dptr, dpitch, sizeof(float) * w, d.H,
                                          cudaMemcpyDeviceToHost);
    CK(e);
  }
  return FADE_OK;
}

int fade_model_set_tensor(fade_model_t* m, int kind, int index, const float* host, int64_t n) {
  if (index < 0 || index >= P_COUNT || kind < 0 || kind > 3 || n != ref_numel(m->d, index)) {
    set_last_error("set_tensor: bad kind/index/size");
    return FADE_ERR_USAGE;
  }
  ON_DEVICE(m->device);
  float* dev = tensor_base(m, kind, index);
  if (index == P_W_E1 || index == P_W_E2)
    return copy_w12(m, dev, index == P_W_E2, const_cast<float*>(host), true);
  CK(cudaMemcpy(dev, host, sizeof(float) * n, cudaMemcpyHostToDevice));
  return FADE_OK;
}

int fade_model_get_tensor(fade_model_t* m, int kind, int index, float* host, int64_t n) {
  if (index < 0 || index >= P_COUNT || kind < 0 || kind > 3 || n != ref_numel(m->d, index)) {
    set_last_error("get_tensor: bad kind/index/size");
    return FADE_ERR_USAGE;
  }
  ON_DEVICE(m->device);
  CK(cudaDeviceSynchronize());
  float* dev = tensor_base(m, kind, index);
  if (index == P_W_E1 || index == P_W_E2) return copy_w12(m, dev, index == P_W_E2, host, false);
  CK(cudaMemcpy(host, dev, sizeof(float) * n, cudaMemcpyDeviceToHost));
  return FADE_OK;
}

// The cache crosses the ABI in the reference's logical order ([B][C], oldest
// block first, model.py:125-127); on the device it may be the block-major ring
// (ModelPtrs.ring_on): logical column c of stream b at
// [((c/32 + shift) mod C/32) * B + b] * 32 + c mod 32.
static float* ring_block(const Dims& d, float* ring, int shift, int b, int j) {
  return ring + (((size_t)((j + shift) % (d.C / 32)) * d.B + b) << 5);
}
static void logical_to_ring(const Dims& d, const float* logical, float* ring) {
  for (int b = 0; b < d.B; ++b)
    for (int j = 0; j < d.C / 32; ++j)
      memcpy(ring_block(d, ring, 0, b, j), logical + (size_t)b * d.C + 32 * j, 32 * sizeof(float));
}
static void ring_to_logical(const Dims& d, float* ring, int shift, float* logical) {
  for (int b = 0; b < d.B; ++b)
    for (int j = 0; j < d.C / 32; ++j)
      memcpy(logical + (size_t)b * d.C + 32 * j, ring_block(d, ring, shift, b, j), 32 * sizeof(float));
}

int fade_model_set_cache(fade_model_t* m, const float* host) {
  ON_DEVICE(m->device);
  CK(cudaDeviceSynchronize());
  const Dims& d = m->d;
  const size_t n = (size_t)d.B * d.C;
  if (m->M.ring_on) {
    std::vector<float> tmp(n);
    logical_to_ring(d, host, tmp.data());
    CK(cudaMemcpy(m->M.a.cache, tmp.data(), sizeof(float) * n, cudaMemcpyHostToDevice));
  } else {
    CK(cudaMemcpy(m->M.a.cache, host, sizeof(float) * n, cudaMemcpyHostToDevice));
  }
  const long long zero = 0;
  CK(cudaMemcpy(&m->st->ring, &zero, sizeof(long long), cudaMemcpyHostToDevice));
  return FADE_OK;
}

int fade_model_get_cache(fade_model_t* m, float* host) {
  ON_DEVICE(m->device);
  CK(cudaDeviceSynchronize());
  const Dims& d = m->d;
  const size_t n = (size_t)d.B * d.C;
  if (!m->M.ring_on) {
    CK(cudaMemcpy(host, m->M.a.cache, sizeof(float) * n, cudaMemcpyDeviceToHost));
    return FADE_OK;
  }
  long long r = 0;
  CK(cudaMemcpy(&r, &m->st->ring, sizeof(long long), cudaMemcpyDeviceToHost));
  const int nb = d.C / 32;
  std::vector<float> tmp(n);
  CK(cudaMemcpy(tmp.data(), m->M.a.cache, sizeof(float) * n, cudaMemcpyDeviceToHost));
  ring_to_logical(d, tmp.data(), (int)((r * (d.D / 32)) % nb), host);
  return FADE_OK;
}

int fade_model_set_counters(fade_model_t* m, int64_t adam_t, int64_t step_count) {
  ON_DEVICE(m->device);
  long long v[2] = {adam_t, step_count};
  CK(cudaMemcpy(&m->st->adam_t, &v[0], sizeof(long long), cudaMemcpyHostToDevice));
  CK(cudaMemcpy(&m->st->step_count, &v[1], sizeof(long long), cudaMemcpyHostToDevice));
  return FADE_OK;
}

int fade_model_get_counters(fade_model_t* m, int64_t* adam_t, int64_t* step_count) {
  ON_DEVICE(m->device);
  CK(cudaDeviceSynchronize());
  long long v[2];
  CK(cudaMemcpy(&v[0], &m->st->adam_t, sizeof(long long), cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(&v[1], &m->st->step_count, sizeof(long long), cudaMemcpyDeviceToHost));
  *adam_t = v[0];
  *step_count = v[1];
  return FADE_OK;
}


int fade_model_predict(fade_model_t* m, const uint8_t* ctx, double* probs, double* alpha,
                       fade_error_t* err) {
  ON_DEVICE(m->device);
  const Dims& d = m->d;
  int64_t sc = 0, t = 0;
  TRY(fade_model_get_counters(m, &t, &sc));
  TRY(set_col(m, sc, sc));
  // the trunk kernel rolls the cache in place before the head can find a
  // non-finite logit; the reference commits the cache only after its finite
  // check (model.py:190-196), so a failed predict restores the snapshot
  TRY(snapshot_cache(m, 0));
  CK(cudaMemcpyAsync(m->ctx_buf, ctx, (size_t)d.B * d.T, cudaMemcpyHostToDevice, m->s_main));
  CK(cudaMemcpyAsync(m->live_ctx, m->ctx_buf, (size_t)d.B * d.T, cudaMemcpyDeviceToDevice,
                     m->s_main));
  StepIO io = api_io(m);
  io.head.want_probs = 1;
  TRY(forward(m, io, true));
  CK(cudaStreamSynchronize(m->s_main));
  if (int st = check_error(m, err)) {
    m->live = false;
    TRY(restore_cache(m, 0));
    CK(cudaStreamSynchronize(m->s_main));
    return st;
  }
  if (probs)
    CK(cudaMemcpy(probs, m->M.a.probs, sizeof(double) * d.B * 256, cudaMemcpyDeviceToHost));
  if (alpha) {
    std::vector<float> rows(3 * (size_t)d.B);
    CK(cudaMemcpy(rows.data(), m->M.a.alpha_row, sizeof(float) * rows.size(), cudaMemcpyDeviceToHost));
    double s = 0.0, mn = rows[1], mx = rows[2];
    for (int b = 0; b < d.B; ++b) {
      s += rows[3 * b];
      mn = std::min(mn, (double)rows[3 * b + 1]);
      mx = std::max(mx, (double)rows[3 * b + 2]);
    }
    alpha[0] = s / ((double)d.B * d.H);
    alpha[1] = mn;
    alpha[2] = mx;
  }
  m->live = true;
  return FADE_OK;
}

int fade_model_train_step(fade_model_t* m, const uint8_t* targets, double* loss, fade_error_t* err) {
  if (!m->live) {
    set_last_error("train_step requires a preceding predict");
    return FADE_ERR_STATE;
  }
  ON_DEVICE(m->device);
  const Dims& d = m->d;
  CK(cudaMemcpyAsync(m->tgt_buf, targets, (size_t)d.B, cudaMemcpyHostToDevice, m->s_main));
  StepIO io = api_io(m);
  io.head.xent = 1;
  io.head.tgt = m->tgt_buf;
  io.head.ld_tgt = 1;
  io.head.adam_prep = 1;
  launch_head(m->M, io.head, m->s_main);     // dlogits + nll for these targets
  TRY(backward(m, io, false, m->loss_buf, 1));
  CK(cudaStreamSynchronize(m->s_main));
  TRY(check_error(m, err));
  CK(cudaMemcpy(loss, m->loss_buf, sizeof(double), cudaMemcpyDeviceToHost));
  m->live = false;
  return FADE_OK;
}

static const float* part_ptr(fade_model_t* m, const char* part, int* width) {
  const Acts& a = m->M.a;
  *width = m->d.H;
  std::string p(part);
  if (p == "global") return a.h_g;
  if (p == "local") return a.h_l;
  if (p == "alpha") return a.alpha;
  if (p == "mix") return a.h_mix;
  if (p == "mixer_inner") return a.inner;
  const VFlags vf = vflags(m->M.variant);
  if (p == "coarse") return vf.mixer ? a.h_c : a.h_mix;
  if (p == "hidden") return vf.fnr ? a.h : (vf.mixer ? a.h_c : a.h_mix);
  if (p == "logits") { *width = 256; return a.logits; }
  return nullptr;
}

int fade_model_forward_debug(fade_model_t* m, const uint8_t* ctx, const char* part, float* out) {
  ON_DEVICE(m->device);
  int width = 0;
  const float* src = part_ptr(m, part, &width);
  if (!src) {
    set_last_error(std::string("unknown forward part ") + part);
    return FADE_ERR_USAGE;
  }
  const Dims& d = m->d;
  TRY(snapshot_cache(m, 1));
  CK(cudaMemcpyAsync(m->ctx_buf, ctx, (size_t)d.B * d.T, cudaMemcpyHostToDevice, m->s_main));
  StepIO io = api_io(m);
  // (the head kernel reduces the logits' split-K slices into a.logits)
  TRY(forward(m, io, true));
  CK(cudaMemcpyAsync(out, src, sizeof(float) * d.B * width, cudaMemcpyDeviceToHost, m->s_main));
  TRY(restore_cache(m, 1));
  TRY(replay_live(m));
  CK(cudaStreamSynchronize(m->s_main));
  return FADE_OK;
}

int fade_model_loss_grads(fade_model_t* m, const uint8_t* ctx, const uint8_t* targets, double* loss) {
  ON_DEVICE(m->device);
  const Dims& d = m->d;
  TRY(snapshot_cache(m, 1));
  CK(cudaMemcpyAsync(m->ctx_buf, ctx, (size_t)d.B * d.T, cudaMemcpyHostToDevice, m->s_main));
  CK(cudaMemcpyAsync(m->tgt_buf, targets, (size_t)d.B, cudaMemcpyHostToDevice, m->s_main));
  int64_t sc = 0, t = 0;
  TRY(fade_model_get_counters(m, &t, &sc));
  TRY(set_col(m, sc, sc));
  StepIO io = api_io(m);
  io.head.xent = 1;
  io.head.tgt = m->tgt_buf;
  io.head.ld_tgt = 1;
  TRY(forward(m, io, true));
  TRY(backward(m, io, true, m->loss_buf, 0));
  TRY(restore_cache(m, 1));
  TRY(replay_live(m));
  CK(cudaStreamSynchronize(m->s_main));
  TRY(check_error(m, nullptr));
  CK(cudaMemcpy(loss, m->loss_buf, sizeof(double), cudaMemcpyDeviceToHost));
  return FADE_OK;
}

// ---------------------------------------------------------------------------
// executors

static int coder_create(int B, long long L, int device, cudaStream_t s, fade_coder_t** out) {
  std::unique_ptr<fade_coder> c(new fade_coder());
  c->B = B;
  c->L = L;
  c->device = device;
  c->cap = 2 * L + 16;       // <= 2 bytes per symbol + the 5-shift flush
  c->s = s;
  const size_t nB = (size_t)B;
  size_t off[8], total = 0;
  const size_t sizes[8] = {8 * nB, 8 * nB, 4 * nB, 8 * nB, 8 * nB, nB * (size_t)c->cap, 8, 4};
  for (int i = 0; i < 8; ++i) {
    total = align_up(total, 256);
    off[i] = total;
    total += sizes[i];
  }
  CK(dev_alloc(&c->mem, total, s));
  char* base = (char*)c->mem;
  c->e.low = (unsigned long long*)(base + off[0]);
  c->e.rng = (unsigned long long*)(base + off[1]);
  c->e.cache = (int*)(base + off[2]);
  c->e.ncache = (long long*)(base + off[3]);
  c->e.blen = (long long*)(base + off[4]);
  c->e.buf = (uint8_t*)(base + off[5]);
  c->e.col = (long long*)(base + off[6]);
  c->e.done_blocks = (unsigned*)(base + off[7]);
  c->e.cap = c->cap;
  launch_enc_init(c->e, B, s);
  CK(cudaGetLastError());
  *out = c.release();
  return FADE_OK;
}

int fade_coder_destroy(fade_coder_t* c) {
  delete c;   // frees its device buffers on its own device
  return FADE_OK;
}

int fade_coder_fetch(fade_coder_t* c, uint8_t* payload, int64_t nbytes) {
  ON_DEVICE(c->device);
  long long total = 0;
  std::vector<long long> off(c->B);
  for (int b = 0; b < c->B; ++b) {
    off[b] = total;
    total += c->lengths[b];
  }
  if (nbytes != total) {
    set_last_error("coder_fetch: payload size mismatch");
    return FADE_ERR_USAGE;
  }
  if (total == 0) return FADE_OK;
  long long* doff = nullptr;
  uint8_t* dout = nullptr;
  auto cleanup = defer([&] {
    dev_free(doff, c->s);
    dev_free(dout, c->s);
    cudaStreamSynchronize(c->s);
  });
  CK(dev_alloc((void**)&doff, sizeof(long long) * c->B, c->s));
  CK(dev_alloc((void**)&dout, (size_t)total, c->s));
  CK(cudaMemcpyAsync(doff, off.data(), sizeof(long long) * c->B, cudaMemcpyHostToDevice, c->s));
  launch_compact(c->e, c->B, doff, dout, c->s);
  CK(cudaMemcpyAsync(payload, dout, (size_t)total, cudaMemcpyDeviceToHost, c->s));
  CK(cudaStreamSynchronize(c->s));
  return FADE_OK;
}

// pipelined compression quantises on the coder stream (k_head_quant) instead
// of in the head kernel; FADE_QUANT_CODER=0 keeps it in the head
static bool quant_on_coder() {
  static const bool on = !knob("FADE_QUANT_CODER") || atoi(knob("FADE_QUANT_CODER")) != 0;
  return on;
}

// one compression timestep; captured once into a CUDA graph and replayed
static int compress_step(fade_model_t* m, fade_coder_t* c, const uint8_t* data, long long L,
                         int pipelined, double* losses, double* alpha_tape = nullptr) {
  StepIO io{};
  io.alpha_tape = alpha_tape;
  io.src = data;
  io.ld_src = L;
  io.use_col = 1;
  io.head.xent = 1;
  io.head.tgt = data;
  io.head.ld_tgt = L;
  io.head.tgt_use_col = 1;
  io.head.adam_prep = 1;
  io.head.skip_quant = pipelined && quant_on_coder();
  TRY(forward(m, io, true));
  if (pipelined) {
    // CSPP: the coder stream quantises and drains this step's table while
    // the model stream runs the backward (pipeline.py:251-287)
    CK(cudaEventRecord(m->ev_cum[0], m->s_main));
    CK(cudaStreamWaitEvent(m->s_coder, m->ev_cum[0], 0));
    if (io.head.skip_quant) launch_head_quant(m->M, c->e.col, m->s_coder);
    launch_encode_col(c->e, m->d.B, data, L, m->M.a.cum, m->s_coder);
    CK(cudaEventRecord(m->ev_enc[0], m->s_coder));
  } else {
    launch_encode_col(c->e, m->d.B, data, L, m->M.a.cum, m->s_main);
  }
  TRY(backward(m, io, false, losses, 1));
  if (pipelined) CK(cudaStreamWaitEvent(m->s_main, m->ev_enc[0], 0));
  CK(cudaGetLastError());
  return FADE_OK;
}

int fade_compress(fade_model_t* m, int device, int batch, const uint8_t* data, int64_t L,
                  int64_t warm, int on_device, int pipelined, int64_t* lengths, double* losses,
                  double* alpha, uint64_t* tape, fade_coder_t** coder_out, fade_error_t* err) {
  *coder_out = nullptr;
  if (m && m->d.B != batch) {
    set_last_error("compress: batch does not match the model");
    return FADE_ERR_USAGE;
  }
  if (!m && L > warm) {
    set_last_error("compress: a model is required when L > warm");
    return FADE_ERR_USAGE;
  }
  const int dev = m ? m->device : device;
  ON_DEVICE(dev);
  cudaStream_t s = m ? m->s_main : nullptr;
  static const bool timing = getenv("FADE_TIMING") != nullptr;   // host timestamps only
  auto now = [] { return std::chrono::steady_clock::now(); };
  const auto tA = now();
  auto stamp = [&](const char* what) {
    if (timing) {
      cudaDeviceSynchronize();
      fprintf(stderr, "[fade] compress %-10s %.3f s\n", what,
              std::chrono::duration<double>(now() - tA).count());
    }
  };
  const size_t nbytes = (size_t)batch * (size_t)L;
  const long long nsteps = L > warm ? L - warm : 0;
  uint8_t* dmat = nullptr;
  double* dloss = nullptr;
  double* dalpha = nullptr;
  unsigned long long* dtape = nullptr;
  auto cleanup = defer([&] {
    dev_free(dmat, s);
    dev_free(dloss, s);
    dev_free(dalpha, s);
    dev_free(dtape, s);
    cudaStreamSynchronize(s);
  });
  NvtxRange range("fade_compress");
  const uint8_t* mat = data;
  if (!on_device && nbytes) {
    NvtxRange r("fade: upload stream matrix");
    CK(dev_alloc((void**)&dmat, nbytes, s));
    CK(cudaMemcpyAsync(dmat, data, nbytes, cudaMemcpyHostToDevice, s));
    mat = dmat;
  }
  stamp("upload");
  fade_coder_t* c = nullptr;
  TRY(coder_create(batch, L, dev, s, &c));
  std::unique_ptr<fade_coder> guard(c);
  launch_encode_warm(c->e, batch, mat, L, warm, s);
  stamp("coder");
  if (m && nsteps > 0) {
    TRY(set_col(m, warm, warm));
    CK(dev_alloc((void**)&dloss, sizeof(double) * (size_t)nsteps, s));
    if (alpha) CK(dev_alloc((void**)&dalpha, sizeof(double) * 3 * (size_t)nsteps, s));
    if (tape) {
      const size_t tb = sizeof(unsigned long long) * kTapeSlots * (size_t)nsteps;
      CK(dev_alloc((void**)&dtape, tb, s));
      CK(cudaMemsetAsync(dtape, 0, tb, s));
      c->e.tape = dtape;
      c->e.tape_base = warm;
    }
    CK(cudaStreamSynchronize(s));
    // capture one timestep into a graph, replay it L - warm times (the coder's
    // column counter starts where the model's does)
    TRY(replay_steps(m, nsteps, dtape, [&] { return compress_step(m, c, mat, L, pipelined, dloss, dalpha); }));
    c->e.tape = nullptr;
    stamp("loop");
    TRY(check_error(m, err));
    if (losses) CK(cudaMemcpy(losses, dloss, sizeof(double) * (size_t)nsteps, cudaMemcpyDeviceToHost));
    if (alpha) CK(cudaMemcpy(alpha, dalpha, sizeof(double) * 3 * (size_t)nsteps, cudaMemcpyDeviceToHost));
    if (tape)
      CK(cudaMemcpy(tape, dtape, sizeof(unsigned long long) * kTapeSlots * (size_t)nsteps,
                    cudaMemcpyDeviceToHost));
  }
  NvtxRange rf("fade: flush + lengths");
  launch_encode_flush(c->e, batch, s);
  c->lengths.resize(batch);
  CK(cudaMemcpyAsync(c->lengths.data(), c->e.blen, sizeof(long long) * batch,
                     cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  stamp("flush");
  for (int b = 0; b < batch; ++b) lengths[b] = c->lengths[b];
  *coder_out = guard.release();
  return FADE_OK;
}

int fade_decompress(fade_model_t* m, int device, int batch, const uint8_t* payload, int64_t nbytes,
                    const int64_t* lengths, int64_t L, int64_t warm, uint8_t* out, double* losses,
                    double* alpha, uint64_t* tape, fade_error_t* err) {
  if (m && m->d.B != batch) {
    set_last_error("decompress: batch does not match the model");
    return FADE_ERR_USAGE;
  }
  if (!m && L > warm) {
    set_last_error("decompress: a model is required when L > warm");
    return FADE_ERR_USAGE;
  }
  ON_DEVICE(m ? m->device : device);
  cudaStream_t s = m ? m->s_main : nullptr;
  // device copies: payload, offsets, lengths, decoder state, output matrix
  std::vector<long long> off(batch);
  long long tot = 0;
  for (int b = 0; b < batch; ++b) {
    off[b] = tot;
    tot += lengths[b];
  }
  if (tot != nbytes) {
    set_last_error("decompress: payload length does not match the stream table");
    return FADE_ERR_USAGE;
  }
  const long long nsteps = L > warm ? L - warm : 0;
  const size_t nB = (size_t)batch;
  const size_t sizes[8] = {(size_t)std::max<long long>(nbytes, 1), 8 * nB, 8 * nB, 8 * nB,
                           8 * nB, 8 * nB, (size_t)batch * (size_t)L + 1, 8};
  size_t offs[8], total = 0;
  for (int i = 0; i < 8; ++i) {
    total = align_up(total, 256);
    offs[i] = total;
    total += sizes[i];
  }
  void* mem = nullptr;
  double* dloss = nullptr;
  double* dalpha = nullptr;
  unsigned long long* dtape = nullptr;
  auto cleanup = defer([&] {
    dev_free(dloss, s);
    dev_free(dalpha, s);
    dev_free(dtape, s);
    dev_free(mem, s);
    cudaStreamSynchronize(s);
  });
  CK(dev_alloc(&mem, total, s));
  char* base = (char*)mem;
  DecState ds;
  ds.payload = (const uint8_t*)(base + offs[0]);
  ds.off = (const long long*)(base + offs[1]);
  ds.dlen = (const long long*)(base + offs[2]);
  ds.pos = (long long*)(base + offs[3]);
  ds.code = (unsigned long long*)(base + offs[4]);
  ds.rng = (unsigned long long*)(base + offs[5]);
  uint8_t* dmat = (uint8_t*)(base + offs[6]);
  unsigned long long* err_key = m ? &m->st->err_key : (unsigned long long*)(base + offs[7]);
  if (nbytes) CK(cudaMemcpyAsync((void*)ds.payload, payload, nbytes, cudaMemcpyHostToDevice, s));
  CK(cudaMemcpyAsync((void*)ds.off, off.data(), 8 * nB, cudaMemcpyHostToDevice, s));
  CK(cudaMemcpyAsync((void*)ds.dlen, lengths, 8 * nB, cudaMemcpyHostToDevice, s));
  if (!m) {
    unsigned long long none = ~0ull;
    CK(cudaMemcpyAsync(err_key, &none, 8, cudaMemcpyHostToDevice, s));
  }
  NvtxRange range("fade_decompress");
  launch_dec_prime(ds, batch, err_key, s);
  launch_decode_warm(ds, batch, dmat, L, warm, err_key, s);
  if (m && nsteps > 0) {
    TRY(set_col(m, warm, warm));
    CK(dev_alloc((void**)&dloss, sizeof(double) * (size_t)nsteps, s));
    if (alpha) CK(dev_alloc((void**)&dalpha, sizeof(double) * 3 * (size_t)nsteps, s));
    if (tape) {
      const size_t tb = sizeof(unsigned long long) * kTapeSlots * (size_t)nsteps;
      CK(dev_alloc((void**)&dtape, tb, s));
      CK(cudaMemsetAsync(dtape, 0, tb, s));
    }
    StepIO io{};
    io.alpha_tape = dalpha;
    io.src = dmat;
    io.ld_src = L;
    io.use_col = 1;
    io.head.xent = 1;
    io.head.decode = 1;
    io.head.out = dmat;
    io.head.ld_out = L;
    io.head.payload = ds.payload;
    io.head.off = ds.off;
    io.head.dlen = ds.dlen;
    io.head.dpos = ds.pos;
    io.head.dcode = ds.code;
    io.head.drng = ds.rng;
    io.head.adam_prep = 1;
    CK(cudaStreamSynchronize(s));
    // decode(i) -> train(i) -> predict(i+1) is strictly serial (pipeline.py:364-376)
    TRY(replay_steps(m, nsteps, dtape, [&] {
      int st = forward(m, io, true);
      return st == FADE_OK ? backward(m, io, false, dloss, 1) : st;
    }));
  }
  CK(cudaStreamSynchronize(s));
  if (m) {
    TRY(check_error(m, err));
  } else {
    unsigned long long key = 0;
    CK(cudaMemcpy(&key, err_key, 8, cudaMemcpyDeviceToHost));
    if (key != ~0ull) {
      const int code = (int)(key & 7);
      err->kind = FADE_ERR_CORRUPT;
      err->why = code == 1 ? 1 : 2;
      err->stream = (long long)((key >> 3) & ((1ull << 21) - 1));
      err->step = code == 6 ? -1 : (long long)(key >> 24);
      set_last_error(code == 6 ? "stream shorter than coder tail"
                               : (code == 1 ? "invalid code value" : "truncated stream"));
      return FADE_ERR_CORRUPT;
    }
  }
  CK(cudaMemcpy(out, dmat, (size_t)batch * (size_t)L, cudaMemcpyDeviceToHost));
  if (losses && dloss)
    CK(cudaMemcpy(losses, dloss, sizeof(double) * (size_t)nsteps, cudaMemcpyDeviceToHost));
  if (alpha && dalpha)
    CK(cudaMemcpy(alpha, dalpha, sizeof(double) * 3 * (size_t)nsteps, cudaMemcpyDeviceToHost));
  if (tape && dtape)
    CK(cudaMemcpy(tape, dtape, sizeof(unsigned long long) * kTapeSlots * (size_t)nsteps,
                  cudaMemcpyDeviceToHost));
  return FADE_OK;
}

int fade_model_stream(fade_model_t* m, void** stream) {
  *stream = (void*)m->s_main;
  return FADE_OK;
}

int fade_bench_probe(fade_model_t* m, int which, int iters, double* ms, double* bytes,
                     double* flops) {
  ON_DEVICE(m->device);
  const Dims& d = m->d;
  const double B = d.B, H = d.H, Ep = d.Ep, C = d.C, X = d.X;
  // trunk kernels: the context window of the last fade_bench_compress_steps
  // call (real data: the embedding-gradient atomics contend as in a step)
  if (which >= 5 && !m->bench_src) {
    set_last_error("bench_probe: run fade_bench_compress_steps first");
    return FADE_ERR_USAGE;
  }
  const uint8_t* probe_src = m->bench_src;
  auto launch = [&]() -> int {
    switch (which) {
      case 0: return run_gemm(m, G_E12, m->s_main);
      case 1: return run_gemm(m, G_W12, m->s_main);
      case 2: return run_gemm(m, G_WROUTE_WMEM, m->s_main);
      case 3: launch_bmm_bwd(m->M, 0, 3, m->s_main); return FADE_OK;
      case 4: return run_gemm(m, G_F, m->s_main);
      case 5: launch_trunk_bwd(m->M, probe_src, m->bench_L, 1, m->s_main); return FADE_OK;
      case 6: launch_trunk_fwd(m->M, probe_src, m->bench_L, 1, m->s_main); return FADE_OK;
      case 7: launch_small_adam(m->M, 0, nullptr, nullptr, 0, m->s_main); return FADE_OK;
    }
    set_last_error("bench_probe: unknown component");
    return FADE_ERR_USAGE;
  };
  // algorithmic work of one launch (SURVEY.md section 8d accounting)
  switch (which) {
    case 0:   // z2[B,H] . W12[H,2Ep]: read W12 + z2, write a12 + wide
      *flops = 2.0 * B * H * 2 * Ep;
      *bytes = 4.0 * (H * 2 * Ep + B * H + B * 2 * Ep + B * Ep);
      break;
    case 1:   // dW12 = z2^T dA12 with Adam: p, m, v read + written (24 B/param)
      *flops = 2.0 * H * 2 * Ep * B;
      *bytes = 24.0 * H * 2 * Ep + 4.0 * (B * H + B * 2 * Ep);
      break;
    case 2:   // dW_route + dW_mem with Adam
      *flops = 2.0 * (H * H + C * H) * B;
      *bytes = 24.0 * (H * H + C * H) + 4.0 * (B * H * 2 + B * C + B * H);
      break;
    case 3:   // per-stream W_U: p, m, v read + written
      *flops = 4.0 * B * X * X;
      *bytes = 24.0 * B * X * X + 4.0 * 3 * B * X;
      break;
    case 4:   // wide[B,E] . W_f[E,H] split-K partials
      *flops = 2.0 * B * d.E * H;
      *bytes = 4.0 * (d.E * H + B * Ep + (double)m->M.splits_f * B * H);
      break;
    default:   // trunk_bwd / trunk_fwd / small_adam: latency, not bytes
      *flops = 0.0;
      *bytes = 0.0;
      break;
  }
  TRY(launch());   // warm
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  CK(cudaEventRecord(e0, m->s_main));
  for (int i = 0; i < iters; ++i) TRY(launch());
  CK(cudaEventRecord(e1, m->s_main));
  CK(cudaEventSynchronize(e1));
  float t = 0.f;
  CK(cudaEventElapsedTime(&t, e0, e1));
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  *ms = t / iters;
  return FADE_OK;
}

int fade_bench_compress_steps(fade_model_t* m, const uint8_t* data_dev, int64_t L, int64_t start,
                              int64_t steps, fade_coder_t** coder, int* launches, void* stream) {
  (void)stream;
  ON_DEVICE(m->device);
  m->bench_src = data_dev;
  m->bench_L = L;
  if (!*coder) {
    TRY(coder_create(m->d.B, L, m->device, m->s_main, coder));
    TRY(set_col(m, start, start));
    long long v = start;
    CK(cudaMemcpy((*coder)->e.col, &v, sizeof(v), cudaMemcpyHostToDevice));
  }
  // graphs of steps_per_graph() timesteps (as the executors run them) and
  // of one timestep for the remainder of `steps`
  const int per = steps_per_graph();
  if (!m->bench_exec || m->bench_coder != *coder) {
    for (cudaGraphExec_t* e : {&m->bench_exec, &m->bench_exec1})
      if (*e) {
        CK(cudaGraphExecDestroy(*e));
        *e = nullptr;
      }
    auto body = [&] { return compress_step(m, *coder, data_dev, L, 1, nullptr); };
    size_t n = 0;
    TRY(capture_steps(m, per, body, &m->bench_exec, &n));
    if (per > 1) TRY(capture_steps(m, 1, body, &m->bench_exec1));   // (per == 1: bench_exec is it)
    m->launches_per_step = (int)(n / per);
    m->bench_coder = *coder;
  }
  for (long long i = 0; i < steps / per; ++i) CK(cudaGraphLaunch(m->bench_exec, m->s_main));
  for (long long i = 0; i < steps % per; ++i) CK(cudaGraphLaunch(m->bench_exec1, m->s_main));   // (per > 1 only)
  if (launches) *launches = m->launches_per_step;
  return FADE_OK;
}

}  // extern "C"
