// Batched compact-WY block reflector application (see wy.cuh).
#include "wy.cuh"

namespace {

constexpr int NB = 32;            // reflectors per panel
constexpr int TN = 64;            // C columns per CTA
constexpr int RC = 64;            // rows per staged chunk
constexpr int NT = 256;           // 8 warps
constexpr int LDS = RC + 4;       // padded column length of a staged chunk (conflict-free fragments)
constexpr int LDW = TN + 4;       // padded row length of W

__device__ __forceinline__ void load_chunk(const double* __restrict__ V, int vld, const double* __restrict__ C,
                                           int cld, int ncol, int rbase, double* vs, double* cs) {
  for (int p = threadIdx.x; p < NB * (RC / 2); p += NT) {
    const int col = p / (RC / 2), rr = (p % (RC / 2)) * 2, row = rbase + rr;
    double* dst = vs + col * LDS + rr;
    if (row < vld) fl::cp_async16(dst, V + (int64_t)col * vld + row);
    else dst[0] = dst[1] = 0.0;
  }
  for (int p = threadIdx.x; p < TN * (RC / 2); p += NT) {
    const int col = p / (RC / 2), rr = (p % (RC / 2)) * 2, row = rbase + rr;
    double* dst = cs + col * LDS + rr;
    if (col < ncol && row < cld) fl::cp_async16(dst, C + (int64_t)col * cld + row);
    else dst[0] = dst[1] = 0.0;
  }
  fl::cp_async_commit();
}

// unit lower-trapezoidal mask of the first NB rows of V (chunk 0 only)
__device__ __forceinline__ void mask_unit(double* vs) {
  for (int p = threadIdx.x; p < NB * NB; p += NT) {
    const int col = p / NB, row = p % NB;
    if (row <= col) vs[col * LDS + row] = (row == col) ? 1.0 : 0.0;
  }
}

__global__ void __launch_bounds__(NT, 1) wy_apply_kernel(fl::WyArgs a) {
  extern __shared__ double sm[];
  double* Vs = sm;                       // [2][NB][LDS]
  double* Cs = Vs + 2 * NB * LDS;        // [2][TN][LDS]
  double* Ws = Cs + 2 * TN * LDS;        // [NB][LDW]   W, then op(T) W
  double* Ts = Ws + NB * LDW;            // [NB][NB]    column-major T

  int j, c0;
  if (a.tiles) {
    j = a.tiles[2 * blockIdx.x];
    c0 = a.tiles[2 * blockIdx.x + 1];
  } else {
    j = blockIdx.x / a.tiles_per_block;
    c0 = (blockIdx.x % a.tiles_per_block) * TN;
  }
  const int mj = a.m[j];
  const int r0 = a.row0;
  const int ncol = min(TN, (a.ncols ? a.ncols[j] - a.ncols_sub : a.ncols_const) - c0);
  if (mj <= r0 || ncol <= 0) return;
  const int vld = a.vld ? a.vld[j] : a.vld_const, cld = a.cld ? a.cld[j] : a.cld_const;
  const double* V = a.V + (a.voff ? a.voff[j] : j * a.vstride) + a.v_col0 * (int64_t)vld;
  double* C = a.C + (a.coff ? a.coff[j] : j * a.cstride) + (a.c_col0 + c0) * (int64_t)cld;
  const int nchunks = (mj - r0 + RC - 1) / RC;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, g = lane >> 2, t = lane & 3;

  for (int i = threadIdx.x; i < NB * NB; i += NT) Ts[i] = a.T[(int64_t)j * a.tstride + i];

  // ---------------- phase 1: W = V^T C  (W is NB x TN) ----------------
  const int mt = w & 3, ntb = (w >> 2) * 4;
  double acc[4][2];
#pragma unroll
  for (int n = 0; n < 4; ++n) acc[n][0] = acc[n][1] = 0.0;
  load_chunk(V, vld, C, cld, ncol, r0, Vs, Cs);
  for (int ch = 0; ch < nchunks; ++ch) {
    const int b = ch & 1;
    if (ch + 1 < nchunks)
      load_chunk(V, vld, C, cld, ncol, r0 + (ch + 1) * RC, Vs + (b ^ 1) * NB * LDS, Cs + (b ^ 1) * TN * LDS);
    else
      fl::cp_async_commit();
    fl::cp_async_wait<1>();
    __syncthreads();
    if (ch == 0) {
      mask_unit(Vs);
      __syncthreads();
    }
    const double* vs = Vs + b * NB * LDS;
    const double* cs = Cs + b * TN * LDS;
#pragma unroll 4
    for (int k0 = 0; k0 < RC; k0 += 4) {
      const double av = vs[(mt * 8 + g) * LDS + k0 + t];
#pragma unroll
      for (int n = 0; n < 4; ++n) fl::dmma(acc[n][0], acc[n][1], av, cs[((ntb + n) * 8 + g) * LDS + k0 + t]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int n = 0; n < 4; ++n) {
    Ws[(mt * 8 + g) * LDW + (ntb + n) * 8 + 2 * t] = acc[n][0];
    Ws[(mt * 8 + g) * LDW + (ntb + n) * 8 + 2 * t + 1] = acc[n][1];
  }
  // prefetch the first chunk for phase 3 while phase 2 runs
  load_chunk(V, vld, C, cld, ncol, r0, Vs, Cs);
  __syncthreads();

  // ---------------- phase 2: W <- op(T) W ----------------
#pragma unroll
  for (int n = 0; n < 4; ++n) acc[n][0] = acc[n][1] = 0.0;
#pragma unroll
  for (int k0 = 0; k0 < NB; k0 += 4) {
    const int ar = mt * 8 + g, ac = k0 + t;
    const double av = a.transT ? Ts[ar * NB + ac] : Ts[ac * NB + ar];  // op(T)[ar][ac]
#pragma unroll
    for (int n = 0; n < 4; ++n) fl::dmma(acc[n][0], acc[n][1], av, Ws[(k0 + t) * LDW + (ntb + n) * 8 + g]);
  }
  __syncthreads();
#pragma unroll
  for (int n = 0; n < 4; ++n) {
    Ws[(mt * 8 + g) * LDW + (ntb + n) * 8 + 2 * t] = acc[n][0];
    Ws[(mt * 8 + g) * LDW + (ntb + n) * 8 + 2 * t + 1] = acc[n][1];
  }
  __syncthreads();

  // ---------------- phase 3: C -= V W'  ----------------
  // warp tile: rows 16*(w&3) .. +16 (two 8-row m-tiles), cols 32*(w>>2) .. +32
  const int mrow = (w & 3) * 16, ncb = (w >> 2) * 4;
  double bw[NB / 4][4];
#pragma unroll
  for (int k = 0; k < NB / 4; ++k)
#pragma unroll
    for (int n = 0; n < 4; ++n) bw[k][n] = Ws[(4 * k + t) * LDW + (ncb + n) * 8 + g];
  for (int ch = 0; ch < nchunks; ++ch) {
    const int b = ch & 1;
    const int rbase = r0 + ch * RC;
    if (ch + 1 < nchunks)
      load_chunk(V, vld, C, cld, ncol, rbase + RC, Vs + (b ^ 1) * NB * LDS, Cs + (b ^ 1) * TN * LDS);
    else
      fl::cp_async_commit();
    fl::cp_async_wait<1>();
    __syncthreads();
    if (ch == 0) {
      mask_unit(Vs);
      __syncthreads();
    }
    const double* vs = Vs + b * NB * LDS;
    const double* cs = Cs + b * TN * LDS;
    double c[2][4][2];
#pragma unroll
    for (int mi = 0; mi < 2; ++mi)
#pragma unroll
      for (int n = 0; n < 4; ++n) {
        const int row = mrow + mi * 8 + g, col = (ncb + n) * 8 + 2 * t;
        c[mi][n][0] = cs[col * LDS + row];
        c[mi][n][1] = cs[(col + 1) * LDS + row];
      }
#pragma unroll
    for (int k = 0; k < NB / 4; ++k) {
#pragma unroll
      for (int mi = 0; mi < 2; ++mi) {
        const double av = -vs[(4 * k + t) * LDS + mrow + mi * 8 + g];
#pragma unroll
        for (int n = 0; n < 4; ++n) fl::dmma(c[mi][n][0], c[mi][n][1], av, bw[k][n]);
      }
    }
#pragma unroll
    for (int mi = 0; mi < 2; ++mi) {
      const int row = rbase + mrow + mi * 8 + g;
      if (row < mj) {
#pragma unroll
        for (int n = 0; n < 4; ++n) {
          const int col = (ncb + n) * 8 + 2 * t;
          if (col < ncol) C[(int64_t)col * cld + row] = c[mi][n][0];
          if (col + 1 < ncol) C[(int64_t)(col + 1) * cld + row] = c[mi][n][1];
        }
      }
    }
    __syncthreads();
  }
}

}  // namespace

namespace fl {
size_t wy_smem_bytes() { return (size_t)(2 * NB * LDS + 2 * TN * LDS + NB * LDW + NB * NB) * sizeof(double); }

int wy_apply(const WyArgs& a, cudaStream_t s) {
  if (a.ntiles == 0) return FL_OK;
  static bool attr = false;
  if (!attr) {
    FL_CUDA(cudaFuncSetAttribute(wy_apply_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)wy_smem_bytes()));
    attr = true;
  }
  wy_apply_kernel<<<a.ntiles, NT, wy_smem_bytes(), s>>>(a);
  FL_CHECK_LAUNCH();
  return FL_OK;
}
int wy_nb() { return NB; }
int wy_tn() { return TN; }
}  // namespace fl

// Diagnostic entry point: one launch of the block reflector kernel over
// caller-built tables (all device pointers), for kernel-level tests.
extern "C" int fl_dev_wy_apply(const double* V, const int64_t* voff, const int32_t* vld, double* C,
                               const int64_t* coff, const int32_t* cld, const int32_t* m, const double* T,
                               int64_t tstride, int32_t row0, int32_t transT, const int32_t* ncols,
                               const int32_t* tiles, int32_t ntiles, void* stream) {
  fl::WyArgs a{};
  a.V = V;
  a.voff = voff;
  a.vld = vld;
  a.C = C;
  a.coff = coff;
  a.cld = cld;
  a.m = m;
  a.T = T;
  a.tstride = tstride;
  a.v_col0 = 0;
  a.c_col0 = 0;
  a.row0 = row0;
  a.transT = transT;
  a.ncols = ncols;
  a.ncols_sub = 0;
  a.tiles = tiles;
  a.ntiles = ntiles;
  return fl::wy_apply(a, (cudaStream_t)stream);
}
