// Kernel-table entries (include/fade_b200.h section 1): the five integer
// kernels of pkg/src/dszip/kernels.py:236-254 on device arrays, with the
// reference's exact error protocol (rows after the first failing row are left
// untouched, the first failing row index is returned).
#include <climits>

#include "../../include/fade_b200.h"
#include "coder.cuh"

namespace fade {

// -- quantize_rows ------------------------------------------------------------
__global__ void __launch_bounds__(256) k_quantize_rows(const double* __restrict__ probs,
                                                       long long* __restrict__ freq,
                                                       long long r0, long long r1,
                                                       unsigned long long* first_bad) {
  __shared__ QuantSmem sm;
  const long long row = r0 + blockIdx.x;
  if (row >= r1) return;
  bool bad;
  const int v = quantize_sym(probs[row * kAlphabet + threadIdx.x], sm, &bad);
  if (bad) {
    if (threadIdx.x == 0) atomicMin(first_bad, (unsigned long long)row);
    return;
  }
  freq[row * kAlphabet + threadIdx.x] = v;
}

// Rows after the first failing one must keep their old contents
// (kernels.py:57-58 returns immediately).  The kernel above writes every good
// row, so undo is needed only for rows > first_bad: restore them from a copy.
__global__ void k_restore_rows(long long* freq, const long long* saved, long long from,
                               long long r1) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long n = (r1 - from) * kAlphabet;
  if (i < n) freq[from * kAlphabet + i] = saved[from * kAlphabet + i];
}

// -- encode_step ----------------------------------------------------------------
__global__ void k_check_zero_width(const long long* cum, long long ld, const long long* syms,
                                   long long r0, long long r1, unsigned long long* first_bad) {
  const long long k = r0 + (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= r1) return;
  const long long s = syms[k];
  if (cum[k * ld + s + 1] <= cum[k * ld + s]) atomicMin(first_bad, (unsigned long long)k);
}

__global__ void k_encode_step(const long long* cum, long long ld, const long long* syms,
                              long long* low, long long* rng, long long* cache,
                              long long* ncache, uint8_t* buf, long long buf_ld,
                              long long* blen, long long r0, const unsigned long long* stop) {
  const long long k = r0 + (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= (long long)*stop) return;
  EncLane s{(uint64_t)low[k], (uint64_t)rng[k], (int32_t)cache[k], ncache[k], blen[k]};
  const long long sym = syms[k];
  enc_symbol(s, (uint32_t)cum[k * ld + sym], (uint32_t)cum[k * ld + sym + 1], buf + k * buf_ld);
  low[k] = (long long)s.low;
  rng[k] = (long long)s.rng;
  cache[k] = s.cache;
  ncache[k] = s.ncache;
  blen[k] = s.n;
}

__global__ void k_flush(long long* low, long long* cache, long long* ncache, uint8_t* buf,
                        long long buf_ld, long long* blen, long long r0, long long r1) {
  const long long k = r0 + (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= r1) return;
  EncLane s{(uint64_t)low[k], 0, (int32_t)cache[k], ncache[k], blen[k]};
  enc_flush(s, buf + k * buf_ld);
  low[k] = (long long)s.low;
  cache[k] = s.cache;
  ncache[k] = s.ncache;
  blen[k] = s.n;
}

// -- prime / decode_step --------------------------------------------------------
__global__ void k_prime_check(const long long* dlen, long long r0, long long r1,
                              unsigned long long* first_bad) {
  const long long k = r0 + (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (k < r1 && dlen[k] < 4) atomicMin(first_bad, (unsigned long long)k);
}

__global__ void k_prime(const uint8_t* payload, const long long* off, long long* pos,
                        long long* code, long long* rng, long long r0,
                        const unsigned long long* stop) {
  const long long k = r0 + (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= (long long)*stop) return;
  const uint8_t* p = payload + off[k];
  code[k] = ((long long)p[0] << 24) | ((long long)p[1] << 16) | ((long long)p[2] << 8) | p[3];
  pos[k] = 4;
  rng[k] = (long long)kMask32;
}

// pass 1: find the first failing row without touching state
__global__ void k_decode_probe(const long long* cum, long long ld, const uint8_t* payload,
                               const long long* off, const long long* dlen, const long long* pos,
                               const long long* code, const long long* rng, long long r0,
                               long long r1, unsigned long long* first_bad, int* why) {
  const long long k = r0 + (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= r1) return;
  DecLane s{(uint64_t)code[k], (uint64_t)rng[k], pos[k]};
  int sym;
  const int w = dec_symbol(s, cum + k * ld, payload + off[k], dlen[k], &sym);
  if (w) {
    why[k - r0] = w;
    atomicMin(first_bad, (unsigned long long)k);
  }
}

// pass 2: commit rows before the first failure
__global__ void k_decode_commit(const long long* cum, long long ld, const uint8_t* payload,
                                const long long* off, const long long* dlen, long long* pos,
                                long long* code, long long* rng, long long* out, long long r0,
                                const unsigned long long* stop) {
  const long long k = r0 + (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= (long long)*stop) return;
  DecLane s{(uint64_t)code[k], (uint64_t)rng[k], pos[k]};
  int sym = 0;
  dec_symbol(s, cum + k * ld, payload + off[k], dlen[k], &sym);
  pos[k] = s.pos;
  code[k] = (long long)s.code;
  rng[k] = (long long)s.rng;
  out[k] = sym;
}

// small helper: a device u64 scratch initialised to `init`
struct Scratch {
  unsigned long long* p = nullptr;
  cudaStream_t st;
  explicit Scratch(cudaStream_t s) : st(s) {}
  bool init(unsigned long long v, size_t extra_bytes = 0) {
    if (cudaMallocAsync(&p, sizeof(unsigned long long) + extra_bytes, st) != cudaSuccess) return false;
    return cudaMemcpyAsync(p, &v, sizeof(v), cudaMemcpyHostToDevice, st) == cudaSuccess;
  }
  long long read() {
    unsigned long long v = 0;
    cudaMemcpyAsync(&v, p, sizeof(v), cudaMemcpyDeviceToHost, st);
    cudaStreamSynchronize(st);
    return (long long)v;
  }
  ~Scratch() {
    if (p) cudaFreeAsync(p, st);
  }
};

static int64_t fail_cuda(const char* what) {
  cudaError_t e = cudaGetLastError();
  char b[256];
  snprintf(b, sizeof(b), "%s: %s", what, cudaGetErrorString(e));
  set_last_error(b);
  return -2;  // never a valid row index
}

}  // namespace fade

using namespace fade;

extern "C" {

int64_t fade_quantize_rows(const double* probs, int64_t* freq, int64_t r0, int64_t r1,
                           void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  if (r1 <= r0) return -1;
  Scratch bad(st);
  long long* saved = nullptr;
  const size_t bytes = (size_t)(r1 - r0) * kAlphabet * sizeof(long long);
  if (!bad.init((unsigned long long)LLONG_MAX)) return fail_cuda("quantize_rows alloc");
  if (cudaMallocAsync(&saved, bytes, st) != cudaSuccess) return fail_cuda("quantize_rows alloc");
  cudaMemcpyAsync(saved, freq + r0 * kAlphabet, bytes, cudaMemcpyDeviceToDevice, st);
  k_quantize_rows<<<(unsigned)(r1 - r0), 256, 0, st>>>(probs, (long long*)freq, r0, r1, bad.p);
  const long long k = bad.read();
  if (k != LLONG_MAX && k + 1 < r1) {
    const long long n = (r1 - (k + 1)) * kAlphabet;
    k_restore_rows<<<cdiv(n, 256), 256, 0, st>>>((long long*)freq, saved - r0 * kAlphabet, k + 1, r1);
  }
  cudaFreeAsync(saved, st);
  if (cudaStreamSynchronize(st) != cudaSuccess) return fail_cuda("quantize_rows");
  return k == LLONG_MAX ? -1 : k;
}

int64_t fade_encode_step(const int64_t* cum, int64_t cum_ld, const int64_t* syms, int64_t* low,
                         int64_t* rng, int64_t* cache, int64_t* ncache, uint8_t* buf,
                         int64_t buf_ld, int64_t* blen, int64_t r0, int64_t r1, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  if (r1 <= r0) return -1;
  Scratch stop(st);
  if (!stop.init((unsigned long long)r1)) return fail_cuda("encode_step alloc");
  const int nb = cdiv(r1 - r0, 128);
  k_check_zero_width<<<nb, 128, 0, st>>>((const long long*)cum, cum_ld, (const long long*)syms,
                                         r0, r1, stop.p);
  k_encode_step<<<nb, 128, 0, st>>>((const long long*)cum, cum_ld, (const long long*)syms,
                                    (long long*)low, (long long*)rng, (long long*)cache,
                                    (long long*)ncache, buf, buf_ld, (long long*)blen, r0, stop.p);
  const long long k = stop.read();
  if (cudaGetLastError() != cudaSuccess) return fail_cuda("encode_step");
  return k < r1 ? k : -1;
}

int64_t fade_flush(int64_t* low, int64_t* cache, int64_t* ncache, uint8_t* buf, int64_t buf_ld,
                   int64_t* blen, int64_t r0, int64_t r1, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  if (r1 <= r0) return -1;
  k_flush<<<cdiv(r1 - r0, 128), 128, 0, st>>>((long long*)low, (long long*)cache,
                                               (long long*)ncache, buf, buf_ld,
                                               (long long*)blen, r0, r1);
  if (cudaStreamSynchronize(st) != cudaSuccess) return fail_cuda("flush");
  return -1;
}

int64_t fade_prime(const uint8_t* payload, const int64_t* off, const int64_t* dlen, int64_t* pos,
                   int64_t* code, int64_t* rng, int64_t r0, int64_t r1, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  if (r1 <= r0) return -1;
  Scratch stop(st);
  if (!stop.init((unsigned long long)r1)) return fail_cuda("prime alloc");
  const int nb = cdiv(r1 - r0, 128);
  k_prime_check<<<nb, 128, 0, st>>>((const long long*)dlen, r0, r1, stop.p);
  k_prime<<<nb, 128, 0, st>>>(payload, (const long long*)off, (long long*)pos, (long long*)code,
                              (long long*)rng, r0, stop.p);
  const long long k = stop.read();
  if (cudaGetLastError() != cudaSuccess) return fail_cuda("prime");
  return k < r1 ? k : -1;
}

int64_t fade_decode_step(const int64_t* cum, int64_t cum_ld, const uint8_t* payload,
                         const int64_t* off, const int64_t* dlen, int64_t* pos, int64_t* code,
                         int64_t* rng, int64_t* out, int64_t r0, int64_t r1, int64_t* why,
                         void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  *why = 0;
  if (r1 <= r0) return -1;
  Scratch stop(st);
  const size_t nrow = (size_t)(r1 - r0);
  if (!stop.init((unsigned long long)r1, nrow * sizeof(int))) return fail_cuda("decode alloc");
  int* whys = (int*)(stop.p + 1);
  cudaMemsetAsync(whys, 0, nrow * sizeof(int), st);
  const int nb = cdiv(r1 - r0, 128);
  k_decode_probe<<<nb, 128, 0, st>>>((const long long*)cum, cum_ld, payload,
                                     (const long long*)off, (const long long*)dlen,
                                     (const long long*)pos, (const long long*)code,
                                     (const long long*)rng, r0, r1, stop.p, whys);
  k_decode_commit<<<nb, 128, 0, st>>>((const long long*)cum, cum_ld, payload,
                                      (const long long*)off, (const long long*)dlen,
                                      (long long*)pos, (long long*)code, (long long*)rng,
                                      (long long*)out, r0, stop.p);
  const long long k = stop.read();
  if (cudaGetLastError() != cudaSuccess) return fail_cuda("decode_step");
  if (k < r1) {
    int w = 0;
    cudaMemcpy(&w, whys + (k - r0), sizeof(int), cudaMemcpyDeviceToHost);
    *why = w;
    return k;
  }
  return -1;
}

}  // extern "C"
