// FP64 throughput probes (diagnostic entry point, used by bench.py to state
// the FP64 roofline denominator: MEASURED_PEAKS.json carries HBM and bf16
// only). mode 0: independent DFMA chains on the CUDA cores; mode 1: legacy
// FP64 tensor MMA (mma.sync m8n8k4 f64, SASS DMMA). tcgen05 has no f64 kind.
#include "common.cuh"

namespace {

__global__ void __launch_bounds__(256) dfma_probe(int iters, double* out) {
  double a[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) a[k] = threadIdx.x * 1e-3 + k;
  const double b = 1.0000001, c = -1e-9;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k) a[k] = fma(a[k], b, c);
  }
  double s = 0.0;
#pragma unroll
  for (int k = 0; k < 8; ++k) s += a[k];
  if (s == 12345.678) out[0] = s;  // keep the chains alive
}

__global__ void __launch_bounds__(256) dmma_probe(int iters, double* out) {
  double c[4][2];
#pragma unroll
  for (int k = 0; k < 4; ++k) c[k][0] = c[k][1] = 0.0;
  const double a = 1e-3 * (threadIdx.x & 7), b = 1e-3 * (threadIdx.x >> 3);
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      asm volatile(
          "mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
          : "+d"(c[k][0]), "+d"(c[k][1])
          : "d"(a), "d"(b));
    }
  }
  double s = 0.0;
#pragma unroll
  for (int k = 0; k < 4; ++k) s += c[k][0] + c[k][1];
  if (s == 12345.678) out[0] = s;
}

}  // namespace

// flops per call: mode 0: grid*256*iters*8*2; mode 1: grid*8 warps*iters*4*512
extern "C" int fl_probe_fp64(int32_t mode, int32_t grid, int32_t iters, double* out, void* stream) {
  cudaStream_t s = (cudaStream_t)stream;
  if (mode == 0)
    dfma_probe<<<grid, 256, 0, s>>>(iters, out);
  else
    dmma_probe<<<grid, 256, 0, s>>>(iters, out);
  FL_CHECK_LAUNCH();
  return FL_OK;
}
