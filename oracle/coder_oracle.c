/*
 * TEST INFRASTRUCTURE ONLY -- CPU oracle for the FADE integer path.
 *
 * Plain-C restatement of the reference's quantiser and range coder
 * (/root/reference/pkg/src/dszip/kernels.py). Only tests/, the smoke check in
 * __graft_entry__.py and bench.py's cpu_baseline leg may load this library;
 * the product path (paper_2604_07239_b200/) never does.
 *
 * Parity is pinned by tests/test_oracle.py against golden vectors that
 * tests/golden/make_golden.py produced by running the reference itself.
 *
 * Every function follows the reference argument convention: caller-owned
 * int64 arrays mutated in place, row range [r0, r1), return -1 on success or
 * the first failing row.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define TOP (1LL << 24)
#define MASK32 0xFFFFFFFFLL
#define TOTAL 65536LL
#define KEYSCALE 1099511627776.0 /* 2^40, kernels.py:31 */

static int cmp_i64(const void *a, const void *b) {
  int64_t x = *(const int64_t *)a, y = *(const int64_t *)b;
  return (x > y) - (x < y);
}

/* kernels.py:48-85: floor(p*2^16), largest remainder with index tie-break,
 * zeros raised to 1 taken from the first maximum. */
int64_t oracle_quantize_rows(const double *probs, int64_t *freq, int64_t a,
                             int64_t r0, int64_t r1) {
  double *t = (double *)malloc(sizeof(double) * a);
  int64_t *keys = (int64_t *)malloc(sizeof(int64_t) * a);
  int64_t *sorted = (int64_t *)malloc(sizeof(int64_t) * a);
  int64_t bad = -1;
  for (int64_t k = r0; k < r1 && bad < 0; ++k) {
    const double *p = probs + k * a;
    int64_t *f = freq + k * a;
    int64_t deficit = TOTAL;
    for (int64_t i = 0; i < a; ++i) {
      t[i] = p[i] * 65536.0;
      f[i] = (int64_t)t[i];
      deficit -= f[i];
    }
    if (deficit < 0 || deficit > a) { bad = k; break; }
    if (deficit > 0) {
      for (int64_t i = 0; i < a; ++i) {
        double fr = t[i] - (double)(int64_t)t[i];
        keys[i] = (int64_t)(fr * KEYSCALE) * 256 + (a - 1 - i);
      }
      /* keys are distinct, so a threshold on the sorted copy selects exactly
       * the top `deficit` entries -- same set as argsort order[a-deficit:] */
      memcpy(sorted, keys, sizeof(int64_t) * a);
      qsort(sorted, (size_t)a, sizeof(int64_t), cmp_i64);
      int64_t thr = sorted[a - deficit];
      for (int64_t i = 0; i < a; ++i)
        if (keys[i] >= thr) f[i] += 1;
    }
    int64_t zeros = 0, imax = 0, vmax = -1;
    for (int64_t i = 0; i < a; ++i) {
      if (f[i] > vmax) { vmax = f[i]; imax = i; }
      if (f[i] == 0) zeros++;
    }
    if (zeros > 0) {
      if (vmax - zeros < 1) { bad = k; break; }
      f[imax] = vmax - zeros;
      for (int64_t i = 0; i < a; ++i)
        if (f[i] == 0) f[i] = 1;
    }
  }
  free(t); free(keys); free(sorted);
  return bad;
}

/* one renormalisation shift through the carry cache (kernels.py:133-147) */
static inline void shift_low(int64_t *lo, int64_t *ca, int64_t *nc,
                             uint8_t *out, int64_t *n) {
  if (*lo < 0xFF000000LL || *lo > MASK32) {
    int64_t carry = *lo >> 32;
    if (*nc > 0) {
      out[(*n)++] = (uint8_t)((*ca + carry) & 0xFF);
      for (int64_t j = 0; j < *nc - 1; ++j)
        out[(*n)++] = (uint8_t)((0xFF + carry) & 0xFF);
    }
    *ca = (*lo >> 24) & 0xFF;
    *nc = 0;
  }
  *nc += 1;
  *lo = (*lo << 8) & MASK32;
}

/* kernels.py:123-155 */
int64_t oracle_encode_step(const int64_t *cum, int64_t cum_stride,
                           const int64_t *syms, int64_t *low, int64_t *rng,
                           int64_t *cache, int64_t *ncache, uint8_t *buf,
                           int64_t cap, int64_t *blen, int64_t r0, int64_t r1) {
  for (int64_t k = r0; k < r1; ++k) {
    int64_t s = syms[k];
    int64_t c0 = cum[k * cum_stride + s], c1 = cum[k * cum_stride + s + 1];
    if (c1 <= c0) return k;
    int64_t r = rng[k] >> 16;
    int64_t lo = low[k] + c0 * r;
    int64_t rg = (c1 - c0) * r;
    int64_t ca = cache[k], nc = ncache[k], n = blen[k];
    while (rg < TOP) {
      shift_low(&lo, &ca, &nc, buf + k * cap, &n);
      rg <<= 8;
    }
    low[k] = lo; rng[k] = rg; cache[k] = ca; ncache[k] = nc; blen[k] = n;
  }
  return -1;
}

/* kernels.py:158-183: five shifts push every live bit of low out */
int64_t oracle_flush(int64_t *low, int64_t *cache, int64_t *ncache,
                     uint8_t *buf, int64_t cap, int64_t *blen, int64_t r0,
                     int64_t r1) {
  for (int64_t k = r0; k < r1; ++k) {
    int64_t lo = low[k], ca = cache[k], nc = ncache[k], n = blen[k];
    for (int j = 0; j < 5; ++j) shift_low(&lo, &ca, &nc, buf + k * cap, &n);
    low[k] = lo; cache[k] = ca; ncache[k] = nc; blen[k] = n;
  }
  return -1;
}

/* kernels.py:186-197 */
int64_t oracle_prime(const uint8_t *payload, const int64_t *off,
                     const int64_t *dlen, int64_t *pos, int64_t *code,
                     int64_t *rng, int64_t r0, int64_t r1) {
  for (int64_t k = r0; k < r1; ++k) {
    if (dlen[k] < 4) return k;
    int64_t cd = 0;
    for (int j = 0; j < 4; ++j) cd = (cd << 8) | payload[off[k] + j];
    code[k] = cd;
    pos[k] = 4;
    rng[k] = MASK32;
  }
  return -1;
}

/* kernels.py:200-233; returns k and writes why (1 invalid code, 2 truncated) */
int64_t oracle_decode_step(const int64_t *cum, int64_t cum_stride,
                           const uint8_t *payload, const int64_t *off,
                           const int64_t *dlen, int64_t *pos, int64_t *code,
                           int64_t *rng, int64_t *out, int64_t r0, int64_t r1,
                           int64_t *why) {
  *why = 0;
  for (int64_t k = r0; k < r1; ++k) {
    const int64_t *c = cum + k * cum_stride;
    int64_t r = rng[k] >> 16;
    int64_t cd = code[k];
    int64_t dv = cd / r;
    if (dv >= TOTAL) { *why = 1; return k; }
    int64_t lo = 0, hi = 256;
    while (hi - lo > 1) {
      int64_t mid = (lo + hi) >> 1;
      if (c[mid] <= dv) lo = mid; else hi = mid;
    }
    int64_t c0 = c[lo], c1 = c[lo + 1];
    cd -= c0 * r;
    int64_t rg = (c1 - c0) * r;
    int64_t p = pos[k];
    while (rg < TOP) {
      if (p >= dlen[k]) { *why = 2; return k; }
      cd = ((cd << 8) | payload[off[k] + p]) & MASK32;
      p++;
      rg <<= 8;
    }
    pos[k] = p; code[k] = cd; rng[k] = rg; out[k] = lo;
  }
  return -1;
}
