// Streaming-read ceiling on this GPU: sum of a large fp64 buffer with
// 16-byte loads, (a) grid-stride (adjacent CTAs read adjacent lines) and
// (b) one contiguous region per CTA (the LSQR kernels' pattern: every CTA
// streams its own block), plus (c) per-CTA regions through TMA bulk copies
// into a shared-memory ring.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o read_bw read_bw.cu
#include <cstdint>
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

// each CTA: contiguous chunk of `per` double2, U loads in flight per thread
template <int U>
__global__ void rd_chunk(const double2* __restrict__ a, size_t per, int nchunks, double* out) {
  double s = 0.0;
  for (int c = blockIdx.x; c < nchunks; c += gridDim.x) {
    const double2* p = a + (size_t)c * per;
    size_t i = threadIdx.x;
    for (; i + (U - 1) * blockDim.x < per; i += U * blockDim.x) {
      double2 v[U];
#pragma unroll
      for (int u = 0; u < U; ++u) v[u] = __ldcs(p + i + u * blockDim.x);
#pragma unroll
      for (int u = 0; u < U; ++u) s += v[u].x + v[u].y;
    }
    for (; i < per; i += blockDim.x) s += p[i].x + p[i].y;
  }
  if (s == 123.456) out[0] = s;
}

// each CTA: contiguous chunk streamed by TMA bulk copies (tile bytes each)
// into an ST-stage ring; consumers sum the stage
__global__ void rd_tma(const char* __restrict__ a, size_t per_bytes, int nchunks, int tile, int ST, double* out) {
  extern __shared__ __align__(128) char smc[];
  __shared__ __align__(8) uint64_t bars[8];
  if (threadIdx.x == 0) {
    for (int s = 0; s < ST; ++s)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"((unsigned)__cvta_generic_to_shared(&bars[s])));
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  double s = 0.0;
  const int ntile = (int)(per_bytes / tile);
  int phase_base = 0;
  for (int c = blockIdx.x; c < nchunks; c += gridDim.x) {
    const char* p = a + (size_t)c * per_bytes;
    auto issue = [&](int t) {
      if (threadIdx.x != 0 || t >= ntile) return;
      const int g = phase_base + t;
      const unsigned bar = (unsigned)__cvta_generic_to_shared(&bars[g % ST]);
      asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(bar), "r"(tile) : "memory");
      const unsigned dst = (unsigned)__cvta_generic_to_shared(smc + (size_t)(g % ST) * tile);
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(dst),
                   "l"(p + (size_t)t * tile), "r"(tile), "r"(bar) : "memory");
    };
    for (int t = 0; t < ST - 1; ++t) issue(t);
    for (int t = 0; t < ntile; ++t) {
      const int g = phase_base + t;
      const unsigned bar = (unsigned)__cvta_generic_to_shared(&bars[g % ST]);
      const unsigned par = (unsigned)((g / ST) & 1);
      unsigned ok = 0;
      while (!ok)
        asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }\n"
                     : "=r"(ok) : "r"(bar), "r"(par) : "memory");
      const double2* sp = (const double2*)(smc + (size_t)(g % ST) * tile);
      for (int i = threadIdx.x; i < tile / 16; i += blockDim.x) s += sp[i].x + sp[i].y;
      __syncthreads();
      issue(t + ST - 1);
    }
    phase_base += ntile;
  }
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
  auto timeit = [&](auto launch) {
    float best = 1e9;
    for (int r = 0; r < 5; ++r) {
      cudaEventRecord(e0);
      launch();
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      if (ms < best) best = ms;
    }
    return bytes / best / 1e6;
  };
  for (int bpsm : {2, 4}) {
    for (int thr : {256, 512}) {
      double g = timeit([&] { rd<4><<<148 * bpsm, thr>>>(a, n2, o); });
      printf("{\"pattern\": \"grid-stride\", \"ctas_per_sm\": %d, \"threads\": %d, \"read_GBs\": %.1f}\n", bpsm, thr, g);
    }
  }
  // per-CTA contiguous chunks of ~4.7 MB (a half block of cfg4's Q)
  const size_t per = (size_t)(4700000 / 16);
  const int nchunks = (int)(n2 / per);
  for (int bpsm : {2, 3, 4}) {
    double g = timeit([&] { rd_chunk<8><<<148 * bpsm, 256>>>(a, per, nchunks, o); });
    printf("{\"pattern\": \"chunk-per-cta\", \"ctas_per_sm\": %d, \"threads\": 256, \"read_GBs\": %.1f}\n", bpsm,
           g * (double)(nchunks * per * 16) / bytes);
  }
  for (int tile : {22528, 45056}) {
    for (int ST : {3, 4}) {
      for (int bpsm : {2, 3}) {
        const int smem = tile * ST;
        if (smem * bpsm > 220000) continue;
        cudaFuncSetAttribute(rd_tma, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        const size_t pb = (size_t)per * 16 / tile * tile;
        const int nch = (int)(bytes / pb);
        double g = timeit([&] { rd_tma<<<148 * bpsm, 256, smem>>>((const char*)a, pb, nch, tile, ST, o); });
        printf("{\"pattern\": \"tma-ring\", \"tile\": %d, \"stages\": %d, \"ctas_per_sm\": %d, \"read_GBs\": %.1f}\n",
               tile, ST, bpsm, g * (double)(nch * pb) / bytes);
      }
    }
  }
  return 0;
}
