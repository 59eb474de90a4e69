// On-device range coding for the executors (pipeline.py:197-396): lane per
// stream, bit-exact with pkg/src/dszip/kernels.py.
#include "stream_coder.cuh"

namespace fade {

constexpr int kCoderThreads = 128;

__device__ __forceinline__ EncLane load_lane(const EncState& e, int b) {
  return EncLane{e.low[b], e.rng[b], e.cache[b], e.ncache[b], e.blen[b]};
}
__device__ __forceinline__ void store_lane(const EncState& e, int b, const EncLane& s) {
  e.low[b] = s.low;
  e.rng[b] = s.rng;
  e.cache[b] = s.cache;
  e.ncache[b] = s.ncache;
  e.blen[b] = s.n;
}

__global__ void k_enc_init(EncState e, int B) {
  pdl_enter();
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b == 0) {
    *e.col = 0;
    *e.done_blocks = 0;
  }
  if (b >= B) return;
  store_lane(e, b, EncLane{0ull, 0xFFFFFFFFull, 0, 0, 0});   // coder.py:57-63
}

void launch_enc_init(const EncState& e, int B, cudaStream_t s) {
  launch_pdl(k_enc_init, dim3(cdiv(B, kCoderThreads)), dim3(kCoderThreads), 0, s, e, B);
}

__global__ void k_encode_warm(EncState e, int B, const uint8_t* data, long long ld,
                              long long warm) {
  pdl_enter();
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b < B) {
    EncLane s = load_lane(e, b);
    uint8_t* out = e.buf + (long long)b * e.cap;
    for (long long c = 0; c < warm; ++c) {
      const unsigned sym = data[(long long)b * ld + c];
      enc_symbol(s, sym * 256u, sym * 256u + 256u, out);   // uniform_cum (coder.py:46-49)
    }
    store_lane(e, b, s);
  }
  if (b == 0) *e.col = warm;
}

void launch_encode_warm(const EncState& e, int B, const uint8_t* data, long long ld, long long warm,
                        cudaStream_t s) {
  launch_pdl(k_encode_warm, dim3(cdiv(B, kCoderThreads)), dim3(kCoderThreads), 0, s, e, B, data, ld, warm);
}

__global__ void k_encode_col(EncState e, int B, const uint8_t* data, long long ld,
                             const unsigned* cum) {
  pdl_enter();
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  const long long col = *e.col;
  if (e.tape && b == 0) e.tape[kTapeSlots * (col - e.tape_base) + 2] = gtimer_ns();
  if (b < B) {
    const unsigned* row = cum + ((col & 1) * (long long)B + b) * kCumLd;
    const unsigned sym = data[(long long)b * ld + col];
    EncLane s = load_lane(e, b);
    unsigned c0 = row[sym], c1 = row[sym + 1];
    // memory safety only: every quantised table has freq >= 1, so a
    // zero-width interval means the step already failed (error recorded);
    // code the uniform interval instead of renormalising without bound
    if (c1 <= c0) c0 = sym * 256u, c1 = c0 + 256u;
    enc_symbol(s, c0, c1, e.buf + (long long)b * e.cap);
    store_lane(e, b, s);
  }
  // the last block to finish advances the column (every block has read it)
  __syncthreads();
  if (threadIdx.x == 0) {
    if (e.tape) atomicMax(e.tape + kTapeSlots * (col - e.tape_base) + 3, gtimer_ns());
    __threadfence();
    const unsigned prev = atomicAdd(e.done_blocks, 1u);
    if (prev == gridDim.x - 1) {
      *e.done_blocks = 0;
      *e.col = col + 1;
      __threadfence();
    }
  }
}

void launch_encode_col(const EncState& e, int B, const uint8_t* data, long long ld,
                       const unsigned* cum, cudaStream_t s) {
  launch_pdl(k_encode_col, dim3(cdiv(B, kCoderThreads)), dim3(kCoderThreads), 0, s, e, B, data, ld, cum);
}

__global__ void k_encode_flush(EncState e, int B) {
  pdl_enter();
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= B) return;
  EncLane s = load_lane(e, b);
  enc_flush(s, e.buf + (long long)b * e.cap);
  store_lane(e, b, s);
}

void launch_encode_flush(const EncState& e, int B, cudaStream_t s) {
  launch_pdl(k_encode_flush, dim3(cdiv(B, kCoderThreads)), dim3(kCoderThreads), 0, s, e, B);
}

__global__ void k_compact(EncState e, const long long* off, uint8_t* out) {
  pdl_enter();
  const int b = blockIdx.x;
  const long long n = e.blen[b];
  const uint8_t* src = e.buf + (long long)b * e.cap;
  uint8_t* dst = out + off[b];
  for (long long i = threadIdx.x; i < n; i += blockDim.x) dst[i] = src[i];
}

void launch_compact(const EncState& e, int B, const long long* off, uint8_t* out, cudaStream_t s) {
  launch_pdl(k_compact, dim3(B), dim3(256), 0, s, e, off, out);
}

__device__ __forceinline__ void dec_error(unsigned long long* key, long long step, long long stream,
                                          int code) {
  const unsigned long long k = ((unsigned long long)step << 24) |
                               ((unsigned long long)stream << 3) | (unsigned long long)code;
  atomicMin(key, k);
}

// kernels.py:186-197; a stream shorter than the 4-byte tail is corrupt (coder.py:117-118)
__global__ void k_dec_prime(DecState d, int B, unsigned long long* err_key) {
  pdl_enter();
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= B) return;
  if (d.dlen[b] < 4) {
    // step -1 is encoded as 0 with code 6 ("stream shorter than coder tail")
    dec_error(err_key, 0, b, 6);
    d.pos[b] = 0;
    d.code[b] = 0;
    d.rng[b] = kMask32;
    return;
  }
  const uint8_t* p = d.payload + d.off[b];
  d.code[b] = ((unsigned long long)p[0] << 24) | ((unsigned long long)p[1] << 16) |
              ((unsigned long long)p[2] << 8) | p[3];
  d.pos[b] = 4;
  d.rng[b] = kMask32;
}

void launch_dec_prime(const DecState& d, int B, unsigned long long* err_key, cudaStream_t s) {
  launch_pdl(k_dec_prime, dim3(cdiv(B, kCoderThreads)), dim3(kCoderThreads), 0, s, d, B, err_key);
}

struct UniformCum {
  __device__ unsigned operator[](int i) const { return (unsigned)i * 256u; }
};

__global__ void k_decode_warm(DecState d, int B, uint8_t* out, long long ld, long long warm,
                              unsigned long long* err_key) {
  pdl_enter();
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= B) return;
  DecLane s{d.code[b], d.rng[b], d.pos[b]};
  const uint8_t* src = d.payload + d.off[b];
  const long long lim = d.dlen[b];
  const UniformCum ucum;
  for (long long c = 0; c < warm; ++c) {
    int sym = 0;
    const int why = dec_symbol(s, ucum, src, lim, &sym);
    if (why) {
      dec_error(err_key, c, b, why);
      break;
    }
    out[(long long)b * ld + c] = (uint8_t)sym;
  }
  d.code[b] = s.code;
  d.rng[b] = s.rng;
  d.pos[b] = s.pos;
}

void launch_decode_warm(const DecState& d, int B, uint8_t* out, long long ld, long long warm,
                        unsigned long long* err_key, cudaStream_t s) {
  launch_pdl(k_decode_warm, dim3(cdiv(B, kCoderThreads)), dim3(kCoderThreads), 0, s, d, B, out, ld, warm, err_key);
}

}  // namespace fade
