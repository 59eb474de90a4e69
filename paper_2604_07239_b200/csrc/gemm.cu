// Host side of the tcgen05 GEMM: TMA descriptors, tiling, split-K, launch.
#include <cudaTypedefs.h>

#include <cstdlib>
#include <mutex>

#include "../../include/fade_b200.h"
#include "gemm.cuh"
#include "gemm_ws.cuh"

namespace fade {

static PFN_cuTensorMapEncodeTiled_v12000 g_encode = nullptr;

static int get_encoder() {
  static std::once_flag once;
  static int status = FADE_OK;
  std::call_once(once, [] {
    cudaDriverEntryPointQueryResult q;
    void* fn = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess || fn == nullptr) {
      set_last_error("cuTensorMapEncodeTiled unavailable from the driver");
      status = FADE_ERR_CUDA;
      return;
    }
    g_encode = (PFN_cuTensorMapEncodeTiled_v12000)fn;
  });
  return status;
}

static int encode(CUtensorMap* map, const float* ptr, long long inner, long long outer,
                  long long ld, int box_inner, int box_outer, CUtensorMapSwizzle swz) {
  if (int s = get_encoder()) return s;
  if (((uintptr_t)ptr & 15) || (ld * 4) % 16) {
    set_last_error("TMA operand must be 16-byte aligned with a 16-byte multiple row pitch");
    return FADE_ERR_USAGE;
  }
  cuuint64_t dims[2] = {(cuuint64_t)inner, (cuuint64_t)outer};
  cuuint64_t strides[1] = {(cuuint64_t)(ld * 4)};
  cuuint32_t box[2] = {(cuuint32_t)box_inner, (cuuint32_t)box_outer};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = g_encode(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, (void*)ptr, dims, strides, box,
                        estr, CU_TENSOR_MAP_INTERLEAVE_NONE, swz,
                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    char b[160];
    snprintf(b, sizeof(b), "cuTensorMapEncodeTiled failed (%d) inner=%lld outer=%lld ld=%lld", (int)r,
             inner, outer, ld);
    set_last_error(b);
    return FADE_ERR_CUDA;
  }
  return FADE_OK;
}

// K-major operand: logical [mn][k] rows of K; box = 32 K x box_mn rows
int make_tmap_kmajor(CUtensorMap* map, const float* ptr, long long mn, long long k, long long ld,
                     int box_mn) {
  return encode(map, ptr, k, mn, ld, kBK, box_mn, CU_TENSOR_MAP_SWIZZLE_128B);
}
// MN-major operand: logical [k][mn] rows of MN; box = 32 MN x BK rows of K
int make_tmap_mnmajor(CUtensorMap* map, const float* ptr, long long mn, long long k, long long ld) {
  return encode(map, ptr, mn, k, ld, 32, kBK, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B);
}

// split-K workspace [slices][rows][cols] (slice stride rows*ld): 32 x 128 x 1 boxes
static int make_tmap_slices(CUtensorMap* map, const float* ptr, long long rows, long long cols,
                            long long ld, int slices) {
  if (int s = get_encoder()) return s;
  cuuint64_t dims[3] = {(cuuint64_t)cols, (cuuint64_t)rows, (cuuint64_t)slices};
  cuuint64_t strides[2] = {(cuuint64_t)(ld * 4), (cuuint64_t)(rows * ld * 4)};
  cuuint32_t box[3] = {32, (cuuint32_t)kBM, 1};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = g_encode(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, (void*)ptr, dims, strides, box,
                        estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    set_last_error("cuTensorMapEncodeTiled (split-K slices) failed");
    return FADE_ERR_CUDA;
  }
  return FADE_OK;
}

int gemm_setup(GemmProblem* P, const GemmDesc& d, int BN) {
  memset(P, 0, sizeof(*P));
  P->M = d.M;
  P->N = d.N;
  P->K = d.K;
  // A: a_trans == 0 -> A[m*lda + k] (K-major); 1 -> A[k*lda + m] (M-major)
  P->a_mn = d.a_trans;
  P->b_pre = d.b_pre;
  P->l2_pf = d.l2_pf;
  // B: b_trans == 0 -> B[k*ldb + n] (N-major); 1 -> B[n*ldb + k] (K-major)
  P->b_mn = d.b_trans ? 0 : 1;
  int s;
  // a CTA pair splits the B tile: each CTA stages BN/2 columns
  const int pair = d.pair == 2 ? 2 : 1;
  if (d.a_ring) {
    // block-major ring [ring_len/32][ring_rows][32]: a 2-D view of 32-wide rows
    const long long rows = (long long)(d.ring_len / kBK) * d.ring_rows;
    if (d.ring_len % kBK || !d.ring || d.ring_rows % kBK || d.ring_step < 1) {
      set_last_error("ring-buffer operand: extent and rows must be 32-multiples");
      return FADE_ERR_USAGE;
    }
    s = !P->a_mn ? make_tmap_kmajor(&P->ta, d.A, rows, kBK, kBK, kBM)
                 : make_tmap_mnmajor(&P->ta, d.A, kBK, rows, kBK);
  } else if (!P->a_mn) {
    s = make_tmap_kmajor(&P->ta, d.A, d.M, d.K, d.lda, kBM);
  } else {
    s = make_tmap_mnmajor(&P->ta, d.A, d.M, d.K, d.lda);
  }
  if (s) return s;
  if (!P->b_mn) s = make_tmap_kmajor(&P->tb, d.B, d.N, d.K, d.ldb, BN / pair);
  else s = make_tmap_mnmajor(&P->tb, d.B, d.N, d.K, d.ldb);
  if (s) return s;
  const int kt = cdiv(d.K, kBK);
  const int splits = std::max(1, std::min(d.splits, kt));
  P->k_tiles_per_split = cdiv(kt, splits);
  P->splits = cdiv(kt, P->k_tiles_per_split);   // no empty split
  P->tiles_m = cdiv(d.M, kBM * pair);
  P->tiles_n = cdiv(d.N, BN);
  P->epi = d.epi;
  P->bias = d.bias;
  P->a_ring = d.a_ring;
  P->ring_len = d.ring_len;
  P->ring_rows = d.ring_rows;
  P->ring_step = d.ring_step;
  P->ring_bias = d.ring_bias;
  P->ring = d.ring;
  if (P->splits > 1 && d.epi != EPI_STORE) {
    set_last_error("split-K is only valid with the partial-store epilogue");
    return FADE_ERR_USAGE;
  }
  // output / aux tile maps (row-major, 32 x 128 boxes, 128B swizzle)
  const long long crow = d.c_rows ? d.c_rows : d.M, ccol = d.c_cols ? d.c_cols : d.N;
  const long long arow = d.aux_rows ? d.aux_rows : crow, acol = d.aux_cols ? d.aux_cols : ccol;
  P->c_rows = (int)crow;
  auto tile_map = [](CUtensorMap* m, const float* p, long long rows, long long cols, long long ld) {
    return make_tmap_kmajor(m, p, rows, cols, ld, kBM);
  };
  switch (d.epi) {
    case EPI_STORE:
    case EPI_GRAD:
      s = P->splits > 1 ? make_tmap_slices(&P->tc, d.C, crow, ccol, d.ldc, P->splits)
                        : tile_map(&P->tc, d.C, crow, ccol, d.ldc);
      break;
    case EPI_ADAM:
      s = tile_map(&P->tc, d.C, crow, ccol, d.ldc);
      if (!s) s = tile_map(&P->tx0, d.aux0, crow, ccol, d.ldc);
      if (!s) s = tile_map(&P->tx2, d.aux2, crow, ccol, d.ldc);
      break;
    case EPI_GEGLU:
      s = tile_map(&P->tc, d.C, crow, ccol, d.ldc);
      if (!s) s = tile_map(&P->tx0, d.aux0, arow, acol, d.ld_aux);
      break;
    case EPI_GEGLU_BWD:
      s = tile_map(&P->tc, d.C, crow, ccol, d.ldc);
      if (!s) s = tile_map(&P->tx1, d.aux1, arow, acol, d.ld_aux);
      break;
  }
  return s;
}

template <int BN, int ET, int OCC, int PAIR, bool RING>
static int launch_inst(GemmParams& G, cudaStream_t st) {
  using Cfg = GemmCfg<BN, ET, OCC, PAIR>;
  static std::once_flag once;
  static cudaError_t attr_err = cudaSuccess;
  std::call_once(once, [] {
    attr_err = cudaFuncSetAttribute(k_gemm_tf32<BN, ET, OCC, PAIR, RING>,
                                    cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::kSmem);
  });
  FADE_CUDA_TRY(attr_err);
  FADE_CUDA_TRY(launch_pdl_cluster(k_gemm_tf32<BN, ET, OCC, PAIR, RING>, dim3(G.total_tiles * PAIR),
                                   dim3(kGemmThreads), (size_t)Cfg::kSmem, st, PAIR, G));
  FADE_CUDA_TRY(cudaGetLastError());
  return FADE_OK;
}

// ring-buffer operands exist only for the single-CTA, stage-aliased
// configurations the W_mem GEMMs use
template <int BN, int ET, int OCC = 1, int PAIR = 1>
static int launch_cfg(GemmParams& G, cudaStream_t st) {
  bool ring = false;
  for (int q = 0; q < G.nprob; ++q) ring = ring || G.prob[q].a_ring;
  if (!ring) return launch_inst<BN, ET, OCC, PAIR, false>(G, st);
  if constexpr (PAIR == 1 && ET == 0) {
    return launch_inst<BN, ET, OCC, PAIR, true>(G, st);
  } else {
    set_last_error("ring-buffer operand in an unsupported GEMM configuration");
    return FADE_ERR_USAGE;
  }
}

template <int BN, int PAIR>
static int launch_ws(GemmParams& G, cudaStream_t st) {
  using Cfg = WsCfg<BN, PAIR>;
  static std::once_flag once;
  static cudaError_t attr_err = cudaSuccess;
  std::call_once(once, [] {
    attr_err = cudaFuncSetAttribute(k_gemm_ws<BN, PAIR>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    Cfg::kSmem);
  });
  FADE_CUDA_TRY(attr_err);
  int dev = 0, sms = 148;
  FADE_CUDA_TRY(cudaGetDevice(&dev));
  FADE_CUDA_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  const int units = std::min(G.total_tiles, sms / PAIR);
  FADE_CUDA_TRY(launch_pdl_cluster(k_gemm_ws<BN, PAIR>, dim3(units * PAIR), dim3(kGemmThreads),
                                   (size_t)Cfg::kSmem, st, PAIR, G));
  FADE_CUDA_TRY(cudaGetLastError());
  return FADE_OK;
}

#ifdef FADE_PHASE_PROBE
__device__ unsigned long long g_phase[2048][4];
extern "C" __attribute__((visibility("default"))) int fade_debug_phase(unsigned long long* out) {
  return (int)cudaMemcpyFromSymbol(out, g_phase, sizeof(g_phase));
}
#endif

int gemm_launch(GemmParams& G, int BN, cudaStream_t st) {
  int t = 0, et = 0, out = 0;
  if (G.pair != 2) G.pair = 1;
  for (int q = 0; q < G.nprob; ++q) {
    G.prob[q].tile_begin = t;
    t += G.prob[q].tiles_m * G.prob[q].tiles_n * G.prob[q].splits;
    // two-per-SM launches stream their epilogue inputs through the stages
    et = std::max(et, G.occ == 2 ? 0 : epi_tiles(G.prob[q].epi, BN));
    out = std::max(out, epi_out_tiles(G.prob[q].epi, BN));
  }
  G.total_tiles = t;
  if (t == 0) return FADE_OK;
  if (G.ws) {   // persistent: STORE / GEGLU epilogues only, no ring operands
    for (int q = 0; q < G.nprob; ++q)
      if ((G.prob[q].epi != EPI_STORE && G.prob[q].epi != EPI_GEGLU && G.prob[q].epi != EPI_ADAM) ||
          G.prob[q].a_ring ||
          (G.prob[q].epi == EPI_ADAM && (!kWsAdam || G.prob[q].splits > 1))) {
        set_last_error("the persistent GEMM runs only the store, GeGLU and Adam epilogues");
        return FADE_ERR_USAGE;
      }
    if (BN == 256 && G.pair == 2) return launch_ws<256, 2>(G, st);
    if (BN == 128 && G.pair == 2) return launch_ws<128, 2>(G, st);
    if (BN == 128 && G.pair != 2) return launch_ws<128, 1>(G, st);
    set_last_error("unsupported persistent GEMM configuration");
    return FADE_ERR_USAGE;
  }
  auto fits = [&](int alias_tiles) {
    if (et == 0 && out > alias_tiles) {
      set_last_error("GEMM epilogue tiles exceed the pipeline smem they alias");
      return false;
    }
    return true;
  };
  if (G.pair == 2) {   // CTA pairs: 256-row tiles, B staged half per CTA
    if (et != 0) {
      set_last_error("CTA-pair GEMMs need a streamed (stage-aliased) epilogue");
      return FADE_ERR_USAGE;
    }
    // two pairs per SM pair when the epilogue's output tiles fit the smaller
    // stage ring (the streamed Adam epilogue does), else one
    if (BN == 256 && G.occ == 2 && out <= GemmCfg<256, 0, 2, 2>::kAliasTiles)
      return launch_cfg<256, 0, 2, 2>(G, st);
    if (BN == 256 && fits(GemmCfg<256, 0, 1, 2>::kAliasTiles)) return launch_cfg<256, 0, 1, 2>(G, st);
    if (BN == 128 && fits(GemmCfg<128, 0, 1, 2>::kAliasTiles)) return launch_cfg<128, 0, 1, 2>(G, st);
    set_last_error("unsupported CTA-pair GEMM configuration");
    return FADE_ERR_USAGE;
  }
  if (G.occ == 2) {   // two CTAs per SM: one's epilogue overlaps the other's mainloop
    if (BN == 128 && et == 0 && fits(GemmCfg<128, 0, 2>::kAliasTiles)) return launch_cfg<128, 0, 2>(G, st);
    if (BN == 64 && et == 0 && fits(GemmCfg<64, 0, 2>::kAliasTiles)) return launch_cfg<64, 0, 2>(G, st);
    set_last_error("unsupported 2-CTA/SM GEMM configuration");
    return FADE_ERR_USAGE;
  }
  if (BN == 64 && et == 0 && fits(GemmCfg<64, 0>::kAliasTiles)) return launch_cfg<64, 0>(G, st);
  if (BN == 64 && et == 2) return launch_cfg<64, 2>(G, st);
  if (BN == 64 && et == 3) return launch_cfg<64, 3>(G, st);
  if (BN == 128 && et == 0 && fits(GemmCfg<128, 0>::kAliasTiles)) return launch_cfg<128, 0>(G, st);
  if (BN == 256 && et == 0 && fits(GemmCfg<256, 0>::kAliasTiles)) return launch_cfg<256, 0>(G, st);
  set_last_error("unsupported GEMM tile configuration");
  return FADE_ERR_USAGE;
}

}  // namespace fade
