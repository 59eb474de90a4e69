// Per-stream range coder state for the on-device executors (one lane per
// stream).  Same state machine as coder.cuh; the column being coded is read
// from a device counter so a captured CUDA graph replays every timestep.
#pragma once
#include "coder.cuh"

namespace fade {

struct EncState {
  unsigned long long* low;
  unsigned long long* rng;
  int* cache;
  long long* ncache;
  long long* blen;
  uint8_t* buf;            // [B][cap]
  long long cap;
  long long* col;          // column the next encode launch codes
  unsigned* done_blocks;   // last-block-done counter for advancing *col
  unsigned long long* tape; // executor event tape (model.cuh kTapeSlots), or null
  long long tape_base;      // column of tape row 0
};

struct DecState {
  const uint8_t* payload;
  const long long* off;
  const long long* dlen;
  long long* pos;
  unsigned long long* code;
  unsigned long long* rng;
};

// uniform-coded warm-up columns [0, warm) of every stream (pipeline.py:212-213)
void launch_encode_warm(const EncState& e, int B, const uint8_t* data, long long ld, long long warm,
                        cudaStream_t s);
// one column from the CSPP slot (col & 1) of `cum` ([2][B][kCumLd])
void launch_encode_col(const EncState& e, int B, const uint8_t* data, long long ld,
                       const unsigned* cum, cudaStream_t s);
void launch_encode_flush(const EncState& e, int B, cudaStream_t s);
void launch_enc_init(const EncState& e, int B, cudaStream_t s);
// gather per-stream bytes into one payload at offsets off[b]
void launch_compact(const EncState& e, int B, const long long* off, uint8_t* out, cudaStream_t s);

void launch_dec_prime(const DecState& d, int B, unsigned long long* err_key, cudaStream_t s);
void launch_decode_warm(const DecState& d, int B, uint8_t* out, long long ld, long long warm,
                        unsigned long long* err_key, cudaStream_t s);

}  // namespace fade
