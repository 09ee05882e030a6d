// K2 (route R) — batched truncated RRQR of every block, BLAS-3 where the
// work is a genuine GEMM (hard part 1):
//
//   K2a  unpivoted blocked Householder QR  A_j = Q0_j R0_j      (panel.cu + wy.cu, DMMA)
//   K2b  truncated QRCP on R0_j (LAPACK dlaqps rule)  -> perm, r_j, R_j   (qrcp.cu)
//   Q1   thin Q1_j = H'_0 .. H'_{r-1} [S; 0]  (K x r_j, signs S = sign(diag R))   (wy.cu)
//   K2c  Q_j = Q0_j [Q1_j; 0]  (m_j x r_j), reflector panels in reverse   (wy.cu)
//
// Pivots of QRCP(R0_j) equal those of QRCP(A_j) in exact arithmetic (partial
// column norms are invariant under Q0_j). No host synchronisation: every
// per-block size that depends on the rank is read by the kernels from device
// memory (tiles past r_j exit immediately).
#include <float.h>

#include "wy.cuh"

namespace fl {
int panel_factor(double* A, const int64_t* off, const int32_t* ld, const int32_t* m, int J, int K, int P0,
                 double* tau, double* T, cudaStream_t s, const double* src = nullptr);
int qrcp_r0(double* R0, int K, const int32_t* kmax, int J, double sigma, double* tau, int32_t* perm,
            int32_t* rank, double* diag, cudaStream_t s);
int wy_apply(const WyArgs& a, cudaStream_t s);
int wy_nb();
int wy_tn();
int qform_fused(const double* V, const int64_t* voff, const int32_t* vld, const int32_t* m, double* C,
                const int64_t* coff, const int32_t* cld, const int32_t* rank, const double* T64, int K, int J,
                cudaStream_t s);
}  // namespace fl

namespace {

constexpr int NB = 32;
constexpr int NT = 256;

// R0w[j] (K x K, ld K) = upper triangle of the factored work block's top K rows.
// bad[j] != 0 when R0_j holds a non-finite entry: a NaN/Inf anywhere in A_j
// reaches R0_j (every reflector dot product over a non-finite column is
// non-finite, 0 * Inf included), so this is the `_check_matrix` test of
// linalg.py:49-55 for the blocked route.
__global__ void extract_r0_kernel(const double* __restrict__ W, const int64_t* __restrict__ off,
                                  const int32_t* __restrict__ ld, const int32_t* __restrict__ m, int K,
                                  double* __restrict__ R0, int32_t* __restrict__ kmax, int32_t* __restrict__ bad) {
  const int j = blockIdx.y;
  const int64_t n = (int64_t)K * K;
  const int mj = m[j];
  const int km = mj < K ? mj : K;
  if (blockIdx.x == 0 && threadIdx.x == 0) kmax[j] = km;
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < n; p += (int64_t)gridDim.x * blockDim.x) {
    const int c = (int)(p / K), r = (int)(p % K);
    const double v = (r <= c && r < km) ? W[off[j] + (int64_t)c * ld[j] + r] : 0.0;
    if (!isfinite(v)) bad[j] = 1;
    R0[(int64_t)j * n + p] = v;
  }
}

// blocks with a non-finite entry report rank -1 (the host raises InvalidInputError)
__global__ void mark_nonfinite_kernel(const int32_t* __restrict__ bad, int J, int32_t* __restrict__ rank) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j < J && bad[j]) rank[j] = -1;
}

// per (block, panel of the QRCP reflectors): T from G = V^T V (V unit lower in
// R0w columns p0..p0+31, rows p0..kmax-1); reflectors past the rank have tau 0.
__global__ void __launch_bounds__(NT) build_t_kernel(const double* __restrict__ R0, int K,
                                                     const int32_t* __restrict__ kmax,
                                                     const double* __restrict__ tau, const int32_t* __restrict__ rank,
                                                     double* __restrict__ T) {
  constexpr int GC = 64, GLD = GC + 4;
  __shared__ double Vs[NB * GLD];
  __shared__ double Gs[NB * NB];
  __shared__ double Tl[NB * NB];
  const int j = blockIdx.y, p = blockIdx.x, p0 = p * NB;
  const int npan = K / NB;
  double* Tp = T + ((int64_t)j * npan + p) * NB * NB;
  const int r = rank[j];
  if (p0 >= r) return;
  const double* A = R0 + (int64_t)j * K * K;
  const double* tj = tau + (int64_t)j * K;
  const int M = kmax[j] - p0;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, g = lane >> 2, t4 = lane & 3;
  // 10 upper 8x8 tiles over 8 warps: warps 0,1 take two tiles
  double acc[2][2] = {{0.0, 0.0}, {0.0, 0.0}};
  int ta[2], tb[2], nt = 0;
  {
    int cnt = 0;
    for (int x = 0; x < 4; ++x)
      for (int y = x; y < 4; ++y) {
        if (cnt % 8 == w && nt < 2) {
          ta[nt] = x;
          tb[nt] = y;
          ++nt;
        }
        ++cnt;
      }
  }
  for (int r0 = 0; r0 < M; r0 += GC) {
    for (int q = threadIdx.x; q < NB * GC; q += NT) {
      const int col = q / GC, rr = q % GC, row = r0 + rr;
      double v = 0.0;
      if (row < M && p0 + col < r) {
        if (row > col) v = A[(int64_t)(p0 + col) * K + p0 + row];
        else if (row == col) v = 1.0;
      }
      Vs[col * GLD + rr] = v;
    }
    __syncthreads();
    for (int u = 0; u < nt; ++u)
#pragma unroll 4
      for (int k0 = 0; k0 < GC; k0 += 4)
        fl::dmma(acc[u][0], acc[u][1], Vs[(ta[u] * 8 + g) * GLD + k0 + t4], Vs[(tb[u] * 8 + g) * GLD + k0 + t4]);
    __syncthreads();
  }
  for (int u = 0; u < nt; ++u) {
    Gs[(ta[u] * 8 + g) * NB + tb[u] * 8 + 2 * t4] = acc[u][0];
    Gs[(ta[u] * 8 + g) * NB + tb[u] * 8 + 2 * t4 + 1] = acc[u][1];
  }
  __syncthreads();
  if (w == 0) {
    for (int i = 0; i < NB; ++i) {
      const double ti = (p0 + i < r) ? tj[p0 + i] : 0.0;
      double z = 0.0;
      if (lane < i)
        for (int b = lane; b < i; ++b) z += Tl[b * NB + lane] * Gs[b * NB + i];
      __syncwarp();
      Tl[i * NB + lane] = (lane < i) ? -ti * z : (lane == i ? ti : 0.0);
      __syncwarp();
    }
    for (int i = lane; i < NB * NB; i += 32) Tp[i] = Tl[i];
  }
}

// Q1[j] (K x K, ld K) = [S_r; 0]; R[j] = S R0w[0:r, 0:r] (upper), zero elsewhere
__global__ void init_q1_r_kernel(const double* __restrict__ R0, int K, const int32_t* __restrict__ rank,
                                 double* __restrict__ Q1, double* __restrict__ R) {
  const int j = blockIdx.y;
  const int64_t n = (int64_t)K * K;
  const int rk = rank[j];
  const double* A = R0 + (int64_t)j * n;
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < n; p += (int64_t)gridDim.x * blockDim.x) {
    const int c = (int)(p / K), r = (int)(p % K);
    const double sr = A[(int64_t)r * K + r] < 0.0 ? -1.0 : 1.0;  // sign(R_rr), 0 -> +1
    Q1[(int64_t)j * n + p] = (r == c && c < rk) ? sr : 0.0;
    R[(int64_t)j * n + p] = (r <= c && c < rk) ? sr * A[p] : 0.0;
  }
}

// Qhat[j] (ld_j x K): rows < K, cols < r: Q1; everything else 0
// Q store <- [Q1; 0]. sparse = 1 (fused K2c): only the first rank columns,
// rows < K and the padding rows m..ld-1 are written; qform writes rows
// K..m-1 itself and treats them as zero until then.
__global__ void init_qhat_kernel(const double* __restrict__ Q1, int K, const int32_t* __restrict__ rank,
                                 const int64_t* __restrict__ off, const int32_t* __restrict__ ld,
                                 const int32_t* __restrict__ m, int sparse, double* __restrict__ Q) {
  const int j = blockIdx.y;
  const int ldj = ld[j], rk = rank[j], mj = m[j];
  // rows written per column: all ld, or (sparse) rows < K plus the padding
  const int lo = min(K, mj);
  const int per = sparse ? lo + (ldj - mj) : ldj;
  const int64_t n = (int64_t)per * (sparse ? rk : K);
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < n; p += (int64_t)gridDim.x * blockDim.x) {
    const int c = (int)(p / per), rr = (int)(p % per);
    const int r = (sparse && rr >= lo) ? mj + (rr - lo) : rr;
    Q[off[j] + (int64_t)c * ldj + r] = (r < K && c < rk) ? Q1[(int64_t)j * K * K + (int64_t)c * K + r] : 0.0;
  }
}

// Two consecutive 32-reflector panels (P0 = 64 q) -> one 64-wide compact WY:
// T = [[T1, -T1 (V1^T V2) T2], [0, T2]] with V1 = columns P0..P0+31 (unit
// diagonal from row P0), V2 = columns P0+32..P0+63 (unit diagonal from row
// P0+32). X = V1^T V2 only involves rows >= P0+32 (V2 vanishes above).
__global__ void __launch_bounds__(NT) combine_t_kernel(const double* __restrict__ W, const int64_t* __restrict__ off,
                                                       const int32_t* __restrict__ ld,
                                                       const int32_t* __restrict__ m, int K,
                                                       const double* __restrict__ T32, double* __restrict__ T64,
                                                       int q) {
  constexpr int GC = 48, GLD = GC + 4;  // static smem <= 48 KB
  __shared__ double V1s[NB * GLD];
  __shared__ double V2s[NB * GLD];
  __shared__ double Xs[NB * NB];
  __shared__ double Ys[NB * NB];
  const int j = blockIdx.y, P0 = 64 * q;
  const int npan32 = K / NB, npan64 = K / 64;
  const double* A = W + off[j];
  const int64_t ldj = ld[j];
  const int M = m[j] - (P0 + NB);  // rows of V2's support
  const double* T1 = T32 + ((int64_t)j * npan32 + 2 * q) * NB * NB;
  const double* T2 = T1 + NB * NB;
  double* T = T64 + ((int64_t)j * npan64 + q) * 64 * 64;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, g = lane >> 2, t4 = lane & 3;
  // X = V1^T V2: 16 tiles of 8x8, 2 per warp
  double acc[2][2] = {{0.0, 0.0}, {0.0, 0.0}};
  // the next chunk is loaded into registers while this one is multiplied
  constexpr int PER = NB * GC / NT;
  static_assert(PER * NT == NB * GC, "chunk must split evenly over the CTA");
  double n1[PER], n2[PER];
  auto fetch = [&](int r0) {
#pragma unroll
    for (int u = 0; u < PER; ++u) {
      const int p = threadIdx.x + u * NT, col = p / GC, rr = p % GC, row = r0 + rr;  // row relative to P0 + 32
      double v1 = 0.0, v2 = 0.0;
      if (row < M) {
        v1 = A[(int64_t)(P0 + col) * ldj + P0 + NB + row];  // below V1's diagonal block
        if (row > col) v2 = A[(int64_t)(P0 + NB + col) * ldj + P0 + NB + row];
        else if (row == col) v2 = 1.0;
      }
      n1[u] = v1;
      n2[u] = v2;
    }
  };
  fetch(0);
  for (int r0 = 0; r0 < M; r0 += GC) {
#pragma unroll
    for (int u = 0; u < PER; ++u) {
      const int p = threadIdx.x + u * NT, col = p / GC, rr = p % GC;
      V1s[col * GLD + rr] = n1[u];
      V2s[col * GLD + rr] = n2[u];
    }
    if (r0 + GC < M) fetch(r0 + GC);
    __syncthreads();
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const int tile = 2 * w + u, ta = tile & 3, tb = tile >> 2;
#pragma unroll 4
      for (int k0 = 0; k0 < GC; k0 += 4)
        fl::dmma(acc[u][0], acc[u][1], V1s[(ta * 8 + g) * GLD + k0 + t4], V2s[(tb * 8 + g) * GLD + k0 + t4]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int u = 0; u < 2; ++u) {
    const int tile = 2 * w + u, ta = tile & 3, tb = tile >> 2;
    Xs[(ta * 8 + g) * NB + tb * 8 + 2 * t4] = acc[u][0];
    Xs[(ta * 8 + g) * NB + tb * 8 + 2 * t4 + 1] = acc[u][1];
  }
  __syncthreads();
  // Y = X T2 (row-major Xs/Ys; T2 column-major: T2[b][c] at T2[c*NB + b])
  for (int p = threadIdx.x; p < NB * NB; p += NT) {
    const int a = p / NB, c = p % NB;
    double s = 0.0;
    for (int b = 0; b <= c; ++b) s += Xs[a * NB + b] * T2[c * NB + b];
    Ys[a * NB + c] = s;
  }
  __syncthreads();
  // T (column-major 64 x 64)
  for (int p = threadIdx.x; p < 64 * 64; p += NT) {
    const int c = p / 64, r = p % 64;
    double val = 0.0;
    if (r < NB && c < NB) val = T1[c * NB + r];
    else if (r >= NB && c >= NB) val = T2[(c - NB) * NB + (r - NB)];
    else if (r < NB && c >= NB) {
      double s = 0.0;
      for (int b = r; b < NB; ++b) s += T1[b * NB + r] * Ys[b * NB + (c - NB)];
      val = -s;
    }
    T[p] = val;
  }
}

// rows m_j..ld_j-1 of every column of block j set to zero
__global__ void zero_pad_kernel(double* __restrict__ W, const int64_t* __restrict__ off,
                                const int32_t* __restrict__ ld, const int32_t* __restrict__ m, int K) {
  const int j = blockIdx.x;
  const int ldj = ld[j], mj = m[j], pad = ldj - mj;
  if (pad <= 0) return;
  for (int p = threadIdx.x; p < K * pad; p += blockDim.x) W[off[j] + (int64_t)(p / pad) * ldj + mj + p % pad] = 0.0;
}

// zero tau past the rank (reflectors that were never generated)
__global__ void clamp_tau_kernel(double* tau, int K, const int32_t* rank) {
  const int j = blockIdx.x;
  for (int c = threadIdx.x; c < K; c += blockDim.x)
    if (c >= rank[j]) tau[(int64_t)j * K + c] = 0.0;
}

}  // namespace

namespace {
struct Workspace {
  double *fac, *R0, *Q1, *T0, *T1, *T64, *tau0, *tau1;
  int32_t *kmax, *bad;
};

Workspace carve(void* base, int J, int K, int64_t store_elems, size_t* total) {
  const int npan = K / NB;
  char* w = (char*)base;
  size_t used = 0;
  auto take = [&](size_t bytes) {
    char* p = w ? w + used : nullptr;
    used += (bytes + 255) / 256 * 256;
    return p;
  };
  Workspace ws;
  ws.fac = (double*)take((size_t)store_elems * 8);
  ws.R0 = (double*)take((size_t)J * K * K * 8);
  ws.Q1 = (double*)take((size_t)J * K * K * 8);
  ws.T0 = (double*)take((size_t)J * npan * NB * NB * 8);
  ws.T1 = (double*)take((size_t)J * npan * NB * NB * 8);
  ws.T64 = (double*)take((size_t)J * (K / 64 + 1) * 64 * 64 * 8);
  ws.tau0 = (double*)take((size_t)J * K * 8);
  ws.tau1 = (double*)take((size_t)J * K * 8);
  ws.kmax = (int32_t*)take((size_t)J * 4);
  ws.bad = (int32_t*)take((size_t)J * 4);
  if (total) *total = used;
  return ws;
}

// C_j[:, c_col0 : c_col0 + ncols] of the factor copy -= its own reflector panel at v_col0
fl::WyArgs self_args(const fl_blockop* A, double* fac, int J, int v_col0, int c_col0, int ncols,
                     const double* T, int64_t tstride, int transT) {
  fl::WyArgs a{};
  a.V = fac;
  a.voff = A->off;
  a.vld = A->ld;
  a.C = fac;
  a.coff = A->off;
  a.cld = A->ld;
  a.m = A->m;
  a.T = T;
  a.tstride = tstride;
  a.v_col0 = v_col0;
  a.c_col0 = c_col0;
  a.row0 = v_col0;
  a.transT = transT;
  a.ncols_const = ncols;
  a.tiles_per_block = (ncols + fl::wy_tn() - 1) / fl::wy_tn();
  a.ntiles = J * a.tiles_per_block;
  return a;
}
}  // namespace

extern "C" int64_t fl_rrqr_blocked_workspace(int32_t nblocks, int32_t K, int64_t store_elems) {
  size_t total = 0;
  carve(nullptr, nblocks, K, store_elems, &total);
  return (int64_t)total;
}

namespace {
// The whole route for the J blocks of one store.
int run_route(const fl_blockop* A, const fl_blockop* Q, int K, double sigma, double* R, int32_t* perm,
              int32_t* rank, double* diag, const Workspace& ws, int J, cudaStream_t s) {
  const int npan = K / NB;
  const int TN = fl::wy_tn();
  const bool wide = (K % 64) == 0;  // 64-wide compact-WY updates
  const int64_t t32s = (int64_t)npan * NB * NB, t64s = (int64_t)(K / 64) * 64 * 64;
  double* fac = ws.fac;

  // ---- K2a: unpivoted blocked Householder QR ----
  // the factor copy is written by the first panel step (rows < m_j); its
  // padding rows m_j..ld_j-1, which the WY kernels stream, are zeroed here
  zero_pad_kernel<<<J, 256, 0, s>>>(fac, A->off, A->ld, A->m, K);
  FL_CHECK_LAUNCH();
  int e;
  if (wide) {
    for (int q = 0; q < K / 64; ++q) {
      const int P0 = 64 * q;
      // q = 0 reads the raw blocks and writes the factor copy (no separate copy)
      const double* src = q == 0 ? (const double*)A->vals : nullptr;
      if ((e = fl::panel_factor(fac, A->off, A->ld, A->m, J, K, P0, ws.tau0, ws.T0, s, src))) return e;
      fl::WyArgs a = self_args(A, fac, J, P0, P0 + NB, NB, ws.T0 + (int64_t)(2 * q) * NB * NB, t32s, 1);
      a.Csrc = src;
      if ((e = fl::wy_apply_nb(a, 32, s))) return e;
      if ((e = fl::panel_factor(fac, A->off, A->ld, A->m, J, K, P0 + NB, ws.tau0, ws.T0, s))) return e;
      combine_t_kernel<<<dim3(1, J), NT, 0, s>>>(fac, A->off, A->ld, A->m, K, ws.T0, ws.T64, q);
      FL_CHECK_LAUNCH();
      const int ntrail = K - P0 - 64;
      if (ntrail > 0) {
        a = self_args(A, fac, J, P0, P0 + 64, ntrail, ws.T64 + (int64_t)q * 64 * 64, t64s, 1);
        a.Csrc = src;
        if ((e = fl::wy_apply_nb(a, 64, s))) return e;
      }
    }
  } else {
    for (int p = 0; p < npan; ++p) {
      const int P0 = p * NB;
      const double* src = p == 0 ? (const double*)A->vals : nullptr;
      if ((e = fl::panel_factor(fac, A->off, A->ld, A->m, J, K, P0, ws.tau0, ws.T0, s, src))) return e;
      const int ntrail = K - P0 - NB;
      if (ntrail > 0) {
        fl::WyArgs a = self_args(A, fac, J, P0, P0 + NB, ntrail, ws.T0 + (int64_t)p * NB * NB, t32s, 1);
        a.Csrc = src;
        if ((e = fl::wy_apply_nb(a, 32, s))) return e;
      }
    }
  }
  // ---- K2b: truncated QRCP of R0 ----
  FL_CUDA(cudaMemsetAsync(ws.bad, 0, (size_t)J * sizeof(int32_t), s));
  extract_r0_kernel<<<dim3(64, J), 256, 0, s>>>(fac, A->off, A->ld, A->m, K, ws.R0, ws.kmax, ws.bad);
  FL_CHECK_LAUNCH();
  if ((e = fl::qrcp_r0(ws.R0, K, ws.kmax, J, sigma, ws.tau1, perm, rank, diag, s))) return e;
  clamp_tau_kernel<<<J, 256, 0, s>>>(ws.tau1, K, rank);
  build_t_kernel<<<dim3(npan, J), NT, 0, s>>>(ws.R0, K, ws.kmax, ws.tau1, rank, ws.T1);
  init_q1_r_kernel<<<dim3(64, J), 256, 0, s>>>(ws.R0, K, rank, ws.Q1, R);
  FL_CHECK_LAUNCH();
  // ---- Q1 = H'_0 .. H'_{r-1} [S; 0]: 32-wide panels in reverse, columns >= P0 ----
  // (measured: 64-wide blocks with combined T's 9.95 ms per filter incl. the
  // combine, the fused qform sweep 12.7 ms, vs 8.3 for these launches on the
  // 512-row factors, whose passes are too short for the wider kernels)
  for (int p = npan - 1; p >= 0; --p) {
    const int P0 = p * NB;
    fl::WyArgs a{};
    a.V = ws.R0;
    a.vstride = (int64_t)K * K;
    a.vld_const = K;
    a.C = ws.Q1;
    a.cstride = (int64_t)K * K;
    a.cld_const = K;
    a.m = ws.kmax;
    a.T = ws.T1 + (int64_t)p * NB * NB;
    a.tstride = t32s;
    a.v_col0 = P0;
    a.c_col0 = P0;
    a.row0 = P0;
    a.transT = 0;
    a.ncols = rank;
    a.ncols_sub = P0;
    a.tiles_per_block = (K - P0 + TN - 1) / TN;
    a.ntiles = J * a.tiles_per_block;
    if ((e = fl::wy_apply_nb(a, 32, s))) return e;
  }
  // ---- K2c: Qhat = Q0 [Q1; 0], reflector blocks of Q0 in reverse ----
  init_qhat_kernel<<<dim3(128, J), 256, 0, s>>>(ws.Q1, K, rank, Q->off, Q->ld, Q->m, wide ? 1 : 0,
                                                (double*)Q->vals);
  FL_CHECK_LAUNCH();
  if (wide) {
    // one fused sweep per 64-column tile of Qhat (qform.cu)
    if ((e = fl::qform_fused(fac, A->off, A->ld, A->m, (double*)Q->vals, Q->off, Q->ld, rank, ws.T64, K, J, s)))
      return e;
  } else {
    for (int p = K / NB - 1; p >= 0; --p) {
      const int P0 = p * NB;
      fl::WyArgs a{};
      a.V = fac;
      a.voff = A->off;
      a.vld = A->ld;
      a.C = (double*)Q->vals;
      a.coff = Q->off;
      a.cld = Q->ld;
      a.m = A->m;
      a.T = ws.T0 + (int64_t)p * NB * NB;
      a.tstride = t32s;
      a.v_col0 = P0;
      a.c_col0 = 0;
      a.row0 = P0;
      a.transT = 0;
      a.ncols = rank;
      a.ncols_sub = 0;
      a.tiles_per_block = (K + TN - 1) / TN;
      a.ntiles = J * a.tiles_per_block;
      if ((e = fl::wy_apply_nb(a, NB, s))) return e;
    }
  }
  mark_nonfinite_kernel<<<(J + 255) / 256, 256, 0, s>>>(ws.bad, J, rank);
  FL_CHECK_LAUNCH();
  return FL_OK;
}
}  // namespace

extern "C" int fl_rrqr_blocked(const fl_blockop* A, const fl_blockop* Q, int32_t K, int64_t store_elems,
                               double sigma, double* R, int32_t* perm, int32_t* rank, double* diag,
                               void* workspace, void* stream) {
  if (!(sigma >= 0.0 && sigma < 1.0) || K < NB || K % NB) return FL_ERR_INVALID;
  const int J = A->nblocks;
  if (J == 0) return FL_OK;
  // shared-memory bound of K2b (F panel). Blocks taller than
  // FL_RRQR_BLOCKED_MAX_ROWS are handled too: their inner panels are factored
  // in place instead of staged (panel.cu)
  if (K > FL_RRQR_BLOCKED_MAX_K) return FL_ERR_INVALID;
  Workspace ws = carve(workspace, J, K, store_elems, nullptr);
  // the raw blocks stay intact: the first K2a step reads them and writes the
  // factor copy (same layout, absolute offsets)
  return run_route(A, Q, K, sigma, R, perm, rank, diag, ws, J, (cudaStream_t)stream);
}
