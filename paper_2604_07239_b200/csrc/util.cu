// ABI housekeeping: error strings, version, and a GEMM test hook.
#include <cstring>
#include <string>

#include "../../include/fade_b200.h"
#include "gemm.cuh"

namespace fade {
static thread_local std::string g_last_error;
void set_last_error(const std::string& msg) { g_last_error = msg; }
const char* last_error() { return g_last_error.c_str(); }
}  // namespace fade

using namespace fade;

extern "C" {

const char* fade_last_error(void) { return last_error(); }

int fade_abi_version(void) { return 3; }

int fade_device_count(void) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) return 0;
  return n;
}

int fade_device_arch(int device, int* major, int* minor, char* name, int name_len) {
  cudaDeviceProp prop;
  if (cudaGetDeviceProperties(&prop, device) != cudaSuccess) {
    set_last_error("fade_device_arch: no such device");
    return FADE_ERR_CUDA;
  }
  *major = prop.major;
  *minor = prop.minor;
  if (name && name_len > 0) {
    strncpy(name, prop.name, (size_t)name_len - 1);
    name[name_len - 1] = 0;
  }
  return FADE_OK;
}

// Test hook for the tcgen05 GEMM (device pointers, fp32 in/out, TF32 math):
//   C[M,N] = A . B  with a_trans / b_trans as in GemmDesc; splits > 1 writes
//   `splits` partial slices at C + s*M*ldc.
int fade_debug_gemm(const float* A, long long lda, int a_trans, const float* B, long long ldb,
                    int b_trans, float* C, long long ldc, int M, int N, int K, int splits, int bn,
                    int pair, void* stream) {
  GemmParams G;
  memset(&G, 0, sizeof(G));
  G.pair = pair & 3;
  G.ws = (pair & 4) ? 1 : 0;     // bit 2: the persistent kernel
  GemmDesc d{};
  d.pair = pair & 3;
  d.A = A; d.lda = lda; d.a_trans = a_trans;
  d.B = B; d.ldb = ldb; d.b_trans = b_trans;
  d.M = M; d.N = N; d.K = K;
  d.splits = splits;
  d.epi = EPI_STORE;
  d.C = C; d.ldc = ldc;
  if (int s = gemm_setup(&G.prob[0], d, bn)) return s;
  G.nprob = 1;
  return gemm_launch(G, bn, (cudaStream_t)stream);
}

}  // extern "C"
