// Persistent warp-specialised tcgen05 GEMM: the epilogue of tile j overlaps
// the mainloop of tile j+1.
//
// The one-tile-per-CTA kernel (gemm.cuh) runs mainloop -> epilogue in series,
// and its epilogue aliases the stage ring, so neither the tensor pipe nor the
// operand stream is busy while a tile drains.  Here every CTA (or CTA pair)
// walks a static tile schedule with
//   * two TMEM accumulators (2 x BN columns): the MMA warp fills one while the
//     epilogue warps drain the other (accf / acce barrier pairs),
//   * a dedicated double-buffered epilogue staging area: the drain streams the
//     tile out in 32-column sub-chunks by TMA while the stage ring keeps
//     feeding the next tile's mainloop.
// Epilogues: STORE (+ bias on split 0, split-K slices through the 3-D map),
// GEGLU (a1, a2 tiles + gelu(a1)*a2) and ADAM (the weight-update GEMMs: per
// 32-column sub-chunk the p / m / v boxes load by TMA into the staging area
// -- the next sub-chunk's while this one is updated -- and store back, so a
// tile's HBM-bound Adam pass overlaps the next tile's L2-bound mainloop
// instead of following it).  The GeGLU-backward epilogue stays on gemm.cuh.
#pragma once
#include "gemm.cuh"

namespace fade {

constexpr int kWsSub = 32 * kBM * 4;        // one 128-row x 32-column fp32 box (16 KiB)
constexpr int kWsEpiBytes = 3 * kWsSub;      // a GEGLU sub-chunk: a1, a2 and wide halves
#ifndef FADE_WS_EPIBUFS
#define FADE_WS_EPIBUFS 2
#endif
constexpr int kWsEpiBufs = FADE_WS_EPIBUFS;  // staging buffers the drain alternates
// The Adam epilogue serves only the experiments build's FADE_WS weight-update
// runs (measured slower than the one-tile kernel); the
// shipped expand GEMM compiles without it (121 instead of 128 registers)
#ifdef FADE_EXPERIMENTS
constexpr bool kWsAdam = true;
#else
constexpr bool kWsAdam = false;
#endif

template <int BN, int PAIR>
struct WsCfg {
  static constexpr int kBNL = BN / PAIR;
  static constexpr int kABytes = kBM * kBK * 4;
  static constexpr int kBBytes = kBNL * kBK * 4;
  static constexpr int kStageBytes = kABytes + kBBytes;
  static constexpr int kEpiBytes = kWsEpiBufs * kWsEpiBytes;
  static constexpr int kBarBytes = 256;
  static constexpr int kFree = kSmemLimit - 1024 - kBarBytes - kEpiBytes;
  static constexpr int kStages = (kFree / kStageBytes) > 8 ? 8 : (kFree / kStageBytes);
  static constexpr int kSmem = kStages * kStageBytes + kEpiBytes + kBarBytes + 1024;
  static constexpr int kTmemCols = 2 * BN;
  static_assert(kStages >= 3 && kTmemCols <= 512 && kSmem <= kSmemLimit, "persistent GEMM plan");
};

struct WsTile {
  const GemmProblem* P;
  int m0, n0, split, kt_begin, nkt;
};

__device__ __forceinline__ WsTile ws_decode(const GemmParams& G, int tile, int rank, int pair,
                                            int BN) {
  int pi = 0;
#pragma unroll 1
  for (int q = 0; q < G.nprob; ++q)
    if (tile >= G.prob[q].tile_begin) pi = q;
  WsTile t;
  t.P = &G.prob[pi];
  int local = tile - t.P->tile_begin;
  const int tn = local % t.P->tiles_n;
  local /= t.P->tiles_n;
  const int tm = local % t.P->tiles_m;
  t.split = local / t.P->tiles_m;
  t.m0 = tm * (kBM * pair) + rank * kBM;
  t.n0 = tn * BN;
  const int kt_total = cdiv(t.P->K, kBK);
  t.kt_begin = t.split * t.P->k_tiles_per_split;
  t.nkt = max(0, min(kt_total, t.kt_begin + t.P->k_tiles_per_split) - t.kt_begin);
  return t;
}

__device__ __forceinline__ void mbar_arrive_local(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_arrive_remote(uint32_t bar_cluster) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(bar_cluster)
               : "memory");
}

template <int BN, int PAIR>
__global__ void __launch_bounds__(kGemmThreads, 1) k_gemm_ws(const __grid_constant__ GemmParams G) {
  using Cfg = WsCfg<BN, PAIR>;
  constexpr int S = Cfg::kStages;
  constexpr int BNL = Cfg::kBNL;
  extern __shared__ uint8_t smem_raw[];
  // aligned by offsetting the shared array itself (not via an integer cast), so
  // the compiler keeps the shared state space: LDS/STS instead of generic LD/ST
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* epi_smem = smem + S * Cfg::kStageBytes;
  uint64_t* full = (uint64_t*)(epi_smem + Cfg::kEpiBytes);
  uint64_t* empty = full + S;
  uint64_t* accf = empty + S;     // [2] accumulator b is complete
  uint64_t* acce = accf + 2;      // [2] accumulator b drained (PAIR arrivals, on the leader)
  uint64_t* ldb = acce + 2;       // [2] Adam p / m / v sub-chunk loads, per staging buffer
  uint32_t* tmem_slot = (uint32_t*)(ldb + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  pdl_launch_dependents();
  const uint32_t rank = PAIR == 2 ? cluster_rank() : 0u;
  const bool leader = rank == 0;

  if (warp == 0 && lane == 0) {
    for (int q = 0; q < G.nprob; ++q) {
      tma_prefetch(&G.prob[q].ta);
      tma_prefetch(&G.prob[q].tb);
    }
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&accf[b], 1);
      mbar_init(&acce[b], PAIR);
      mbar_init(&ldb[b], 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    if (PAIR == 2) {
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                       smem_u32(tmem_slot)),
                   "r"(Cfg::kTmemCols));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    } else {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                       smem_u32(tmem_slot)),
                   "r"(Cfg::kTmemCols));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
  }
  tc_fence_before();
  __syncthreads();
  if (PAIR == 2) cluster_sync_all();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const int first = blockIdx.x / PAIR, step = gridDim.x / PAIR;
  // weight operand (GemmProblem::b_pre): the B halves of the first tile's
  // first ring stages load before the dependency wait
  auto load_b = [&](const WsTile& t, int i, int s) {
    const GemmProblem& P = *t.P;
    const int nb0 = t.n0 + (int)rank * BNL;
    uint8_t* sb = smem + s * Cfg::kStageBytes + Cfg::kABytes;
    const int k0 = (t.kt_begin + i) * kBK;
    const uint32_t fb = PAIR == 2 ? mapa_shared(smem_u32(&full[s]), 0) : 0u;
    auto load = [&](const CUtensorMap* map, void* dst, int c0, int c1) {
      if (PAIR == 2) tma_load_2d_pair(map, fb, dst, c0, c1);
      else tma_load_2d(map, &full[s], dst, c0, c1);
    };
    if (!P.b_mn) {
      load(&P.tb, sb, k0, nb0);
    } else {
#pragma unroll
      for (int c = 0; c < BNL / 32; ++c) load(&P.tb, sb + c * kBK * 128, nb0 + 32 * c, k0);
    }
  };
  int npre = 0;
  if (warp == 0 && lane == 0 && first < G.total_tiles) {
    const WsTile t = ws_decode(G, first, (int)rank, PAIR, BN);
    npre = t.P->b_pre ? min(t.nkt, S) : 0;
    for (int i = 0; i < npre; ++i) {
      if (leader) mbar_expect_tx(&full[i], PAIR * Cfg::kStageBytes);
      load_b(t, i, i);
    }
  }
  pdl_wait();
#ifdef FADE_PHASE_PROBE
  if (threadIdx.x == 0 && BN == 256) g_phase[1024 + blockIdx.x][0] = gtimer();
#endif

  if (warp == 0) {
    // ---------------- TMA producer: the stage ring runs across tiles ----------------
    if (lane == 0) {
      uint32_t it = 0;
      for (int tile = first; tile < G.total_tiles; tile += step) {
        const WsTile t = ws_decode(G, tile, (int)rank, PAIR, BN);
        const GemmProblem& P = *t.P;
        for (int i = 0; i < t.nkt; ++i, ++it) {
          const int s = (int)(it % S);
          const bool pre = it < (uint32_t)npre;   // B half and byte count already issued
          if (!pre) mbar_wait(&empty[s], ((it / S) & 1u) ^ 1u);
          uint8_t* sa = smem + s * Cfg::kStageBytes;
          const int k0 = (t.kt_begin + i) * kBK;
          if (leader && !pre) mbar_expect_tx(&full[s], PAIR * Cfg::kStageBytes);
          const uint32_t fb = PAIR == 2 ? mapa_shared(smem_u32(&full[s]), 0) : 0u;
          auto load = [&](const CUtensorMap* map, void* dst, int c0, int c1) {
            if (PAIR == 2) tma_load_2d_pair(map, fb, dst, c0, c1);
            else tma_load_2d(map, &full[s], dst, c0, c1);
          };
          if (!P.a_mn) {
            load(&P.ta, sa, k0, t.m0);
          } else {
#pragma unroll
            for (int c = 0; c < kBM / 32; ++c) load(&P.ta, sa + c * kBK * 128, t.m0 + 32 * c, k0);
          }
          if (!pre) load_b(t, i, s);
        }
      }
      if (PAIR == 2) {
        // the leader has released every stage this CTA filled before we exit
        const uint32_t tail = min(it, (uint32_t)S);
        for (uint32_t gi = it; gi < it + tail; ++gi)
          mbar_wait(&empty[gi % S], ((gi / S) & 1u) ^ 1u);
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer (pair leader) ----------------
    if (leader) {
      uint32_t it = 0, jj = 0;   // jj: tiles with a non-empty mainloop (accumulator uses)
      for (int tile = first; tile < G.total_tiles; tile += step) {
        const WsTile t = ws_decode(G, tile, 0, PAIR, BN);
        if (t.nkt == 0) continue;
        const GemmProblem& P = *t.P;
        const uint32_t buf = jj & 1u, use = jj >> 1;
        mbar_wait(&acce[buf], (use & 1u) ^ 1u);   // both CTAs drained this accumulator
        tc_fence_after();
        const uint32_t idesc = make_idesc(kBM * PAIR, BN, P.a_mn, P.b_mn);
        const uint32_t d = tmem + buf * BN;
        for (int i = 0; i < t.nkt; ++i, ++it) {
          const int s = (int)(it % S);
          mbar_wait(&full[s], (it / S) & 1u);
          tc_fence_after();
          if (lane == 0) {
            const uint32_t sa = smem_u32(smem + s * Cfg::kStageBytes);
            const uint32_t sb = sa + Cfg::kABytes;
#pragma unroll
            for (int kk = 0; kk < kBK / kUmmaK; ++kk) {
              const uint64_t ad = P.a_mn ? make_sdesc(sa + kk * 1024, kBK * 128, 512, 1)
                                         : make_sdesc(sa + kk * 32, 16, 1024);
              const uint64_t bd = P.b_mn ? make_sdesc(sb + kk * 1024, kBK * 128, 512, 1)
                                         : make_sdesc(sb + kk * 32, 16, 1024);
              const uint32_t acc = (i > 0 || kk > 0) ? 1u : 0u;
              if (PAIR == 2) tc_mma_tf32_pair(d, ad, bd, idesc, acc);
              else tc_mma_tf32(d, ad, bd, idesc, acc);
            }
            if (PAIR == 2) tc_commit_pair(&empty[s]);
            else tc_commit(&empty[s]);
          }
          __syncwarp();
        }
        if (lane == 0) {
          if (PAIR == 2) tc_commit_pair(&accf[buf]);
          else tc_commit(&accf[buf]);
        }
        __syncwarp();
        ++jj;
      }
    }
  } else {
    // ---------------- epilogue warps ----------------
    const int sub = warp & 3;
    const int r = sub * 32 + lane;
    const int c_lo = 16 * ((warp - 2) >> 2);   // the two warps of a lane quarter: 16 + 16 columns
    const bool lead = (warp == 2 && lane == 0);
    const uint32_t acce_leader = PAIR == 2 ? mapa_shared(smem_u32(&acce[0]), 0) : 0u;
    uint32_t jj = 0, chunk = 0;
    AdamScalars ad{};
    if (kWsAdam && G.adam) ad = *G.adam;   // (after the dependency wait: this step's scalars)
    for (int tile = first; tile < G.total_tiles; tile += step) {
      const WsTile t = ws_decode(G, tile, (int)rank, PAIR, BN);
      const GemmProblem& P = *t.P;
      const bool has = t.nkt > 0;
      const uint32_t buf = jj & 1u, use = jj >> 1;
      if (has) {
        mbar_wait(&accf[buf], use & 1u);
        tc_fence_after();
      }
#ifdef FADE_PHASE_PROBE
      if (lead && BN == 256 && jj < 2) g_phase[1024 + blockIdx.x][1 + jj] = gtimer();
#endif
      const uint32_t taddr = tmem + ((uint32_t)(sub * 32) << 16) + buf * BN;
      auto acc16 = [&](int col, float* v) {
        if (has) {
          tmem_ld16(taddr + col, v);
        } else {
#pragma unroll
          for (int q = 0; q < 16; ++q) v[q] = 0.f;
        }
      };
      const bool geglu = P.epi == EPI_GEGLU;
      const int nsub = geglu ? BN / 64 : BN / 32;
      if (kWsAdam && P.epi == EPI_ADAM) {
        // p / m / v of sub-chunk q land in staging buffer (chunk % 2); the
        // lead issues q + 1's loads once the store that last read that buffer
        // (sub-chunk q - 1) is done reading, then everyone waits for q's
        auto issue = [&](int q, uint32_t ch) {
          uint8_t* eb = epi_smem + (ch % kWsEpiBufs) * kWsEpiBytes;
          uint64_t* lb = &ldb[ch % kWsEpiBufs];
          mbar_expect_tx(lb, 3 * kWsSub);
          tma_load_2d(&P.tc, lb, eb, t.n0 + 32 * q, t.m0);
          tma_load_2d(&P.tx0, lb, eb + kWsSub, t.n0 + 32 * q, t.m0);
          tma_load_2d(&P.tx2, lb, eb + 2 * kWsSub, t.n0 + 32 * q, t.m0);
        };
        if (lead) {
          asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
          issue(0, chunk);
        }
        for (int q = 0; q < nsub; ++q, ++chunk) {
          uint8_t* eb = epi_smem + (chunk % kWsEpiBufs) * kWsEpiBytes;
          if (lead && q + 1 < nsub) {
            asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
            issue(q + 1, chunk + 1);
          }
          mbar_wait(&ldb[chunk % kWsEpiBufs], (chunk / kWsEpiBufs) & 1u);
          for (int c = c_lo; c < 32; c += 32) {
            float g[16];
            acc16(32 * q + c, g);
#pragma unroll
            for (int k = 0; k < 16; k += 4) {
              float4* pp = etile_at(eb, r, c + k);
              float4* pm = etile_at(eb + kWsSub, r, c + k);
              float4* pv = etile_at(eb + 2 * kWsSub, r, c + k);
              float4 p = *pp, m = *pm, v = *pv;
              adam_rn(ad, g[k], p.x, m.x, v.x);
              adam_rn(ad, g[k + 1], p.y, m.y, v.y);
              adam_rn(ad, g[k + 2], p.z, m.z, v.z);
              adam_rn(ad, g[k + 3], p.w, m.w, v.w);
              *pp = p;
              *pm = m;
              *pv = v;
            }
          }
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          epi_bar();
          if (lead) {
            tma_store_2d(&P.tc, eb, t.n0 + 32 * q, t.m0);
            tma_store_2d(&P.tx0, eb + kWsSub, t.n0 + 32 * q, t.m0);
            tma_store_2d(&P.tx2, eb + 2 * kWsSub, t.n0 + 32 * q, t.m0);
            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
          }
        }
      } else
      for (int q = 0; q < nsub; ++q, ++chunk) {
        uint8_t* eb = epi_smem + (chunk % kWsEpiBufs) * kWsEpiBytes;
        // the TMA store that last read this buffer (two chunks ago) is done
        if (lead) {
          if (kWsEpiBufs == 1) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
          else asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
        }
        epi_bar();
        if (geglu) {
          // 128-column interleave block jb = [a1 | a2]; this sub-chunk is its
          // 32-column half h of a1, of a2 and of wide
          const int jb = q >> 1, h = q & 1;
          for (int c = c_lo; c < 32; c += 32) {
            float a1[16], a2[16];
            acc16(128 * jb + 32 * h + c, a1);
            acc16(128 * jb + 64 + 32 * h + c, a2);
#pragma unroll
            for (int k = 0; k < 16; k += 4) {
              *etile_at(eb, r, c + k) = make_float4(a1[k], a1[k + 1], a1[k + 2], a1[k + 3]);
              *etile_at(eb + kWsSub, r, c + k) = make_float4(a2[k], a2[k + 1], a2[k + 2], a2[k + 3]);
              // wide is only a GEMM operand (F, W_f update): stored TF32-rounded
              *etile_at(eb + 2 * kWsSub, r, c + k) =
                  tf32_rne4(make_float4(gelu_f(a1[k]) * a2[k], gelu_f(a1[k + 1]) * a2[k + 1],
                                        gelu_f(a1[k + 2]) * a2[k + 2], gelu_f(a1[k + 3]) * a2[k + 3]));
            }
          }
        } else {
          for (int c = c_lo; c < 32; c += 32) {
            float v[16];
            acc16(32 * q + c, v);
            if (P.bias && t.split == 0) {
#pragma unroll
              for (int k = 0; k < 16; ++k) {
                const int n = t.n0 + 32 * q + c + k;
                v[k] += (n < P.N) ? P.bias[n] : 0.f;
              }
            }
#pragma unroll
            for (int k = 0; k < 16; k += 4)
              *etile_at(eb, r, c + k) = make_float4(v[k], v[k + 1], v[k + 2], v[k + 3]);
          }
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        epi_bar();
        if (lead) {
          if (geglu) {
            const int jb = q >> 1, h = q & 1;
            tma_store_2d(&P.tc, eb, t.n0 + 128 * jb + 32 * h, t.m0);
            tma_store_2d(&P.tc, eb + kWsSub, t.n0 + 128 * jb + 64 + 32 * h, t.m0);
            tma_store_2d(&P.tx0, eb + 2 * kWsSub, (t.n0 >> 1) + 64 * jb + 32 * h, t.m0);
          } else if (P.splits > 1) {
            tma_store_3d(&P.tc, eb, t.n0 + 32 * q, t.m0, t.split);
          } else {
            tma_store_2d(&P.tc, eb, t.n0 + 32 * q, t.m0);
          }
          asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        }
      }
      if (has) {
        // every tcgen05.ld of this tile has completed: hand the accumulator back
        tc_fence_before();
        epi_bar();
        if (lead) {
          if (PAIR == 2) mbar_arrive_remote(acce_leader + buf * 8);
          else mbar_arrive_local(&acce[buf]);
        }
        ++jj;
      }
    }
    if (lead) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
#ifdef FADE_PHASE_PROBE
    if (lead && BN == 256) g_phase[1024 + blockIdx.x][3] = gtimer();
#endif
  }
  tc_fence_before();
  __syncthreads();
  if (PAIR == 2) cluster_sync_all();
  if (warp == 1) {
    tc_fence_after();
    if (PAIR == 2)
      asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                   "r"(Cfg::kTmemCols));
    else
      asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                   "r"(Cfg::kTmemCols));
  }
}

}  // namespace fade
