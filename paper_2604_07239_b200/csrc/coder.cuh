// Integer path of FADE on the device: quantiser, range encoder, range decoder.
//
// Every state machine here is the reference's, bit for bit
// (pkg/src/dszip/kernels.py:26-233): 32-bit range coder with 16-bit
// frequencies, byte renormalisation below 2^24, carry cache with an unbounded
// run of pending 0xFF bytes, 5-shift flush, 4-byte prime.  One thread owns one
// stream (the reference's per-row loop body), so B streams run as B lanes.
#pragma once
#include "common.cuh"

namespace fade {

constexpr uint64_t kTop = 1ull << 24;
constexpr uint64_t kMask32 = 0xFFFFFFFFull;
constexpr int kTotal = 65536;
constexpr int kAlphabet = 256;
constexpr int kCumLd = 260;   // u32 cum rows padded to 16 bytes (257 used)

struct EncLane {
  uint64_t low;    // < 2^33 transiently
  uint64_t rng;
  int32_t cache;
  int64_t ncache;
  int64_t n;       // bytes written
};

// one renormalisation shift through the carry cache (kernels.py:133-147)
__device__ __forceinline__ void enc_shift(EncLane& s, uint8_t* out) {
  if (s.low < 0xFF000000ull || s.low > kMask32) {
    const uint32_t carry = (uint32_t)(s.low >> 32);
    if (s.ncache > 0) {
      out[s.n++] = (uint8_t)((s.cache + carry) & 0xFF);
      const uint8_t fill = (uint8_t)((0xFF + carry) & 0xFF);
      for (int64_t j = 1; j < s.ncache; ++j) out[s.n++] = fill;
    }
    s.cache = (int32_t)((s.low >> 24) & 0xFF);
    s.ncache = 0;
  }
  s.ncache += 1;
  s.low = (s.low << 8) & kMask32;
}

// kernels.py:123-155 body for one stream; c0 < c1 guaranteed by the caller
__device__ __forceinline__ void enc_symbol(EncLane& s, uint32_t c0, uint32_t c1, uint8_t* out) {
  const uint64_t r = s.rng >> 16;
  s.low += (uint64_t)c0 * r;
  uint64_t rg = (uint64_t)(c1 - c0) * r;
  while (rg < kTop) {
    enc_shift(s, out);
    rg <<= 8;
  }
  s.rng = rg;
}

// kernels.py:158-183
__device__ __forceinline__ void enc_flush(EncLane& s, uint8_t* out) {
#pragma unroll 1
  for (int j = 0; j < 5; ++j) enc_shift(s, out);
}

struct DecLane {
  uint64_t code;
  uint64_t rng;
  int64_t pos;
};

// kernels.py:200-233 for one stream.  cum: 257 ascending entries.
// Returns 0 ok, 1 invalid code, 2 truncated; sym receives the symbol.
template <typename CumT>   // CumT: pointer/array of 257 entries or an indexable functor
__device__ __forceinline__ int dec_symbol(DecLane& s, const CumT& cum, const uint8_t* data,
                                          int64_t dlen, int* sym) {
  const uint64_t r = s.rng >> 16;
  const uint64_t dv = s.code / r;
  if (dv >= (uint64_t)kTotal) return 1;
  int lo = 0, hi = kAlphabet;
  while (hi - lo > 1) {
    const int mid = (lo + hi) >> 1;
    if ((uint64_t)cum[mid] <= dv) lo = mid; else hi = mid;
  }
  const uint64_t c0 = (uint64_t)cum[lo], c1 = (uint64_t)cum[lo + 1];
  uint64_t cd = s.code - c0 * r;
  uint64_t rg = (c1 - c0) * r;
  int64_t p = s.pos;
  while (rg < kTop) {
    if (p >= dlen) return 2;
    cd = ((cd << 8) | data[p]) & kMask32;
    ++p;
    rg <<= 8;
  }
  s.pos = p;
  s.code = cd;
  s.rng = rg;
  *sym = lo;
  return 0;
}

// ---------------------------------------------------------------------------
// quantiser for one row, 256 threads, thread i owns symbol i
// (kernels.py:48-85).  Returns the final frequency of symbol i; *bad is set
// (block-uniform) when the row is not a distribution.  Exactly reproduces the
// reference: p*65536 and frac*2^40 are exact power-of-two scalings, so the
// integer keys -- and hence the largest-remainder order -- are identical.
struct QuantSmem {
  int hist[kAlphabet];   // radix-select digit histogram
  int sel[3];            // selected digit, its count, remaining k
  int ired[8];
  int ired2[8];
};

__device__ __forceinline__ int block_isum256(int v, int* red) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  if (lane == 0) red[w] = v;
  __syncthreads();
  int t = lane < 8 ? red[lane] : 0;
#pragma unroll
  for (int o = 4; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
  t = __shfl_sync(0xffffffffu, t, 0);
  __syncthreads();
  return t;
}
__device__ __forceinline__ int block_imax256(int v, int* red) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = max(v, __shfl_xor_sync(0xffffffffu, v, o));
  if (lane == 0) red[w] = v;
  __syncthreads();
  int t = lane < 8 ? red[lane] : INT_MIN;
#pragma unroll
  for (int o = 4; o > 0; o >>= 1) t = max(t, __shfl_xor_sync(0xffffffffu, t, o));
  t = __shfl_sync(0xffffffffu, t, 0);
  __syncthreads();
  return t;
}

__device__ __forceinline__ int quantize_sym(double p, QuantSmem& sm, bool* bad) {
  const int i = threadIdx.x;
  const double t = p * 65536.0;
  int v = (int)(long long)t;     // t >= 0: truncation == floor (kernels.py:56)
  const int deficit = kTotal - block_isum256(v, sm.ired);
  if (deficit < 0 || deficit > kAlphabet) {
    *bad = true;
    return 0;
  }
  if (deficit > 0) {
    const double fr = t - (double)(long long)t;
    const long long key = (long long)(fr * 1099511627776.0) * 256 + (kAlphabet - 1 - i);
    // The reference bumps the `deficit` largest keys (rank >= 256 - deficit in
    // its argsort; keys are distinct: index in the low byte).  Select them by
    // an MSB-first radix select over the 48-bit keys, 8-bit digits: each pass
    // histograms the remaining candidates' digit, one warp finds the digit
    // holding the k-th largest, larger digits are selected, smaller dropped.
    // It stops as soon as every remaining candidate is selected (usually
    // after two passes) -- no 256 x 256 comparison sweep.
    bool cand = true, sel = false;
    for (int shift = 40; shift >= 0; shift -= 8) {
      sm.hist[i] = 0;
      if (i == 0 && shift == 40) sm.sel[2] = deficit;
      __syncthreads();
      const int dg = (int)((key >> shift) & 255);
      if (cand) atomicAdd(&sm.hist[dg], 1);
      __syncthreads();
      if (i < 32) {
        // lane L owns digits 8L..8L+7; suffix sums from the top digit down
        const int kk = sm.sel[2];
        int h[8], s8 = 0;
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          h[q] = sm.hist[8 * i + q];
          s8 += h[q];
        }
        int x = s8;   // inclusive suffix sum over lanes >= i
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const int y = __shfl_down_sync(0xffffffffu, x, o);
          if (i + o < 32) x += y;
        }
        const unsigned hit = __ballot_sync(0xffffffffu, x >= kk);
        if (i == 31 - __clz(hit)) {
          int c = x - s8;    // candidates with a larger digit than this lane's range
#pragma unroll
          for (int q = 7; q >= 0; --q) {
            if (c + h[q] >= kk) {
              sm.sel[0] = 8 * i + q;
              sm.sel[1] = h[q];
              sm.sel[2] = kk - c;
              break;
            }
            c += h[q];
          }
        }
      }
      __syncthreads();
      const int dsel = sm.sel[0], cnt = sm.sel[1], kk = sm.sel[2];
      if (cand) {
        if (dg > dsel) {
          sel = true;
          cand = false;
        } else if (dg < dsel) {
          cand = false;
        }
      }
      if (cnt == kk) {            // every candidate left is among the largest
        if (cand) sel = true;
        break;
      }
    }
    if (sel) v += 1;
    __syncthreads();
  }
  const int zeros = block_isum256(v == 0 ? 1 : 0, sm.ired);
  if (zeros > 0) {
    // first maximum: max of v*256 + (255-i) picks the lowest index on ties
    const int best = block_imax256(v * 256 + (kAlphabet - 1 - i), sm.ired2);
    const int vmax = best >> 8, imax = kAlphabet - 1 - (best & 0xFF);
    if (vmax - zeros < 1) {
      *bad = true;
      return 0;
    }
    if (i == imax) v = vmax - zeros;
    if (v == 0) v = 1;
  }
  *bad = false;
  return v;
}

// exclusive prefix sum of 256 ints (cum[i] = sum_{j<i} f[j]); block-uniform
__device__ __forceinline__ int block_excl_scan256(int f, int* wsum) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  int x = f;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) wsum[w] = x;
  __syncthreads();
  int base = 0;
  for (int k = 0; k < w; ++k) base += wsum[k];
  __syncthreads();
  return base + x - f;
}

}  // namespace fade
