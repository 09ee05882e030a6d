// Shared device helpers for the featlsq B200 kernels (sm_100a, fp64).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/featlsq_b200.h"

namespace fl {

// true the first time it is called for the current device with this flag
// word (per-device one-time setup such as cudaFuncSetAttribute)
inline bool first_on_device(unsigned long long& seen) {
  int dev = 0;
  cudaGetDevice(&dev);
  const unsigned long long bit = 1ull << (dev & 63);
  if (seen & bit) return false;
  seen |= bit;
  return true;
}

// thread-local description of the last failure (fl_last_error)
void set_error(const char* file, int line, cudaError_t e);
}  // namespace fl

#define FL_CHECK_LAUNCH()                                     \
  do {                                                        \
    cudaError_t e_ = cudaGetLastError();                      \
    if (e_ != cudaSuccess) {                                  \
      fl::set_error(__FILE__, __LINE__, e_);                  \
      return FL_ERR_CUDA;                                     \
    }                                                         \
  } while (0)

#define FL_CUDA(call)                                         \
  do {                                                        \
    cudaError_t e_ = (call);                                  \
    if (e_ != cudaSuccess) {                                  \
      fl::set_error(__FILE__, __LINE__, e_);                  \
      return FL_ERR_CUDA;                                     \
    }                                                         \
  } while (0)

namespace fl {

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Warp sums of N (a power of two <= 32) per-lane values with N - 1 + log2(32/N)
// shuffles instead of 5 N: the first log2(N) butterfly levels halve the live
// values per lane; afterwards every lane l holds the full sum of value
// l / (32 / N). Fixed order, so results are run-to-run reproducible.
template <int N>
__device__ __forceinline__ double warp_multi_sum(const double (&in)[N]) {
  const int lane = threadIdx.x & 31;
  double v[N];
#pragma unroll
  for (int c = 0; c < N; ++c) v[c] = in[c];
#pragma unroll
  for (int half = N / 2, o = 16; half >= 1; half /= 2, o /= 2) {
    const bool up = (lane & o) != 0;
#pragma unroll
    for (int c = 0; c < half; ++c) {
      const double send = up ? v[c] : v[c + half];
      const double recv = __shfl_xor_sync(0xffffffffu, send, o);
      v[c] = (up ? v[c + half] : v[c]) + recv;
    }
  }
  double s = v[0];
#pragma unroll
  for (int o = 32 / N / 2; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  return s;
}

// Deterministic CTA-wide sum (fixed shuffle tree, fixed warp order). Every
// thread gets the result. `sh` needs blockDim.x/32 doubles.
__device__ __forceinline__ double block_sum(double v, double* sh) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  v = warp_sum(v);
  __syncthreads();
  if (lane == 0) sh[wid] = v;
  __syncthreads();
  double t = 0.0;
  if (wid == 0) {
    t = lane < nw ? sh[lane] : 0.0;
    t = warp_sum(t);
    if (lane == 0) sh[0] = t;
  }
  __syncthreads();
  t = sh[0];
  __syncthreads();
  return t;
}

// Grid-level deterministic reduction: each CTA deposits `partial` at
// slots[blockIdx.x]; the last CTA to arrive sums all slots in index order
// and returns true (with `total` set) in every thread of that CTA.
__device__ __forceinline__ bool grid_sum_last(double partial, double* slots, unsigned int* counter,
                                              double* total, double* sh) {
  __shared__ bool is_last;
  if (threadIdx.x == 0) {
    slots[blockIdx.x] = partial;
    __threadfence();
    unsigned int prev = atomicAdd(counter, 1u);
    is_last = (prev == gridDim.x - 1);
  }
  __syncthreads();
  if (!is_last) return false;
  __threadfence();
  double acc = 0.0;
  // fixed assignment of slots to threads + fixed tree => deterministic
  for (int i = threadIdx.x; i < (int)gridDim.x; i += blockDim.x) acc += ((volatile double*)slots)[i];
  acc = block_sum(acc, sh);
  *total = acc;
  if (threadIdx.x == 0) *counter = 0u;
  return true;
}

__host__ __device__ __forceinline__ int64_t round_up(int64_t a, int64_t b) { return (a + b - 1) / b * b; }

}  // namespace fl
