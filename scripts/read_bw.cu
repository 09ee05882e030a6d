// Streaming-read ceiling on this GPU: sum of a large fp64 buffer with
// 16-byte loads (nvcc -gencode arch=compute_100a,code=sm_100a -O3 read_bw.cu).
#include <cstdio>
#include <cuda_runtime.h>

template <int U>
__global__ void rd(const double2* __restrict__ a, size_t n2, double* out) {
  double s = 0.0;
  size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x, st = (size_t)gridDim.x * blockDim.x;
  for (; i + (U - 1) * st < n2; i += U * st) {
    double2 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) v[u] = __ldcs(a + i + u * st);
#pragma unroll
    for (int u = 0; u < U; ++u) s += v[u].x + v[u].y;
  }
  for (; i < n2; i += st) s += a[i].x + a[i].y;
  if (s == 123.456) out[0] = s;
}

int main() {
  const size_t bytes = 9ull << 30, n2 = bytes / 16;
  double2* a;
  double* o;
  cudaMalloc(&a, bytes);
  cudaMalloc(&o, 8);
  cudaMemset(a, 0, bytes);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int bpsm : {2, 4, 8, 16}) {
    for (int thr : {256, 512, 1024}) {
      if (bpsm * thr > 2048) continue;
      float best = 1e9;
      for (int r = 0; r < 5; ++r) {
        cudaEventRecord(e0);
        rd<4><<<148 * bpsm, thr>>>(a, n2, o);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (ms < best) best = ms;
      }
      printf("{\"blocks_per_sm\": %d, \"threads\": %d, \"read_GBs\": %.1f}\n", bpsm, thr, bytes / best / 1e6);
    }
  }
  return 0;
}
