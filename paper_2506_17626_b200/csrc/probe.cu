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

// DMMA with CH independent accumulator chains per warp; LDSOP: the A operand
// of every DMMA is a fresh shared-memory load (the pattern of the WY kernels)
template <int CH, bool LDSOP>
__global__ void __launch_bounds__(512) dmma_chain_probe(int iters, double* out) {
  __shared__ double sa[1024];
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) sa[i] = 1e-3 * i;
  __syncthreads();
  double c[CH][2];
#pragma unroll
  for (int k = 0; k < CH; ++k) c[k][0] = c[k][1] = 0.0;
  const double a0 = 1e-3 * (threadIdx.x & 7), b = 1e-3 * (threadIdx.x >> 3);
  const int lane = threadIdx.x & 31;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < CH; ++k) {
      const double a = LDSOP ? sa[((i * CH + k) * 36 + lane) & 1023] : a0;
      asm volatile(
          "mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
          : "+d"(c[k][0]), "+d"(c[k][1])
          : "d"(a), "d"(b));
    }
  }
  double s = 0.0;
#pragma unroll
  for (int k = 0; k < CH; ++k) s += c[k][0] + c[k][1];
  if (s == 12345.678) out[0] = s;
}

// streaming read of n doubles with 16-byte loads, four in flight per thread
__global__ void __launch_bounds__(256) read_probe(const double2* __restrict__ a, int64_t n2, double* out) {
  double s = 0.0;
  const int64_t st = (int64_t)gridDim.x * blockDim.x;
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  for (; i + 3 * st < n2; i += 4 * st) {
    const double2 v0 = __ldcs(a + i), v1 = __ldcs(a + i + st), v2 = __ldcs(a + i + 2 * st),
                  v3 = __ldcs(a + i + 3 * st);
    s += (v0.x + v0.y) + (v1.x + v1.y) + (v2.x + v2.y) + (v3.x + v3.y);
  }
  for (; i < n2; i += st) s += a[i].x + a[i].y;
  if (s == 123.456) out[0] = s;  // keeps the loads alive
}

}  // namespace

// HBM streaming-read ceiling (the LSQR kernel's traffic is read-dominated;
// MEASURED_PEAKS.json's figure is a copy, read + write): bytes = 8 * n
extern "C" int fl_probe_read(const double* buf, int64_t n, double* out, void* stream) {
  if (n < 2) return FL_ERR_INVALID;
  read_probe<<<148 * 4, 256, 0, (cudaStream_t)stream>>>(reinterpret_cast<const double2*>(buf), n / 2, out);
  FL_CHECK_LAUNCH();
  return FL_OK;
}

// flops per call: mode 0: grid*256*iters*8*2; mode 1: grid*8 warps*iters*4*512
extern "C" int fl_probe_fp64(int32_t mode, int32_t grid, int32_t iters, double* out, void* stream) {
  cudaStream_t s = (cudaStream_t)stream;
  switch (mode) {
    case 0: dfma_probe<<<grid, 256, 0, s>>>(iters, out); break;
    case 1: dmma_probe<<<grid, 256, 0, s>>>(iters, out); break;
    // diagnostic: 512-thread CTAs, flops = grid*16 warps*iters*CH*512
    case 11: dmma_chain_probe<1, false><<<grid, 512, 0, s>>>(iters, out); break;
    case 12: dmma_chain_probe<2, false><<<grid, 512, 0, s>>>(iters, out); break;
    case 14: dmma_chain_probe<4, false><<<grid, 512, 0, s>>>(iters, out); break;
    case 18: dmma_chain_probe<8, false><<<grid, 512, 0, s>>>(iters, out); break;
    case 21: dmma_chain_probe<1, true><<<grid, 512, 0, s>>>(iters, out); break;
    case 22: dmma_chain_probe<2, true><<<grid, 512, 0, s>>>(iters, out); break;
    case 24: dmma_chain_probe<4, true><<<grid, 512, 0, s>>>(iters, out); break;
    case 28: dmma_chain_probe<8, true><<<grid, 512, 0, s>>>(iters, out); break;
    default: return FL_ERR_INVALID;
  }
  FL_CHECK_LAUNCH();
  return FL_OK;
}
