// K2b — truncated column-pivoted QR of the triangular factor R0_j of every
// block (route R: QRCP(A_j) and QRCP(R0_j) choose the same pivots in exact
// arithmetic because partial column norms are invariant under the
// orthogonal Q0_j). One CTA per block, R0_j (K x K,
// column-major, ld K) in HBM/L2.
//
// Pivot rule and norm bookkeeping follow LAPACK's blocked dlaqps (what
// dgeqp3 runs on the leading columns): first maximum of the partial norms
// over current positions (IDAMAX, swap semantics), the panel F matrix
// (F[:, k] = tau_k A^T v_k with the incremental correction), row updates of
// the current row, downdate temp = max(0, (1 + t)(1 - t)), t = |a_rj|/vn1_j,
// columns with temp * (vn1/vn2)^2 <= sqrt(eps) flagged and the panel closed
// early, their norms recomputed after the block update. Truncation: the
// first step with |R_ii| < sigma |R_00| stops everything (linalg.py:75-85).
#include <float.h>

#include "wy.cuh"

namespace {

constexpr int NT = 512;
constexpr int NW = NT / 32;
constexpr int PB = 32;  // panel width

struct QrcpArgs {
  double* R0;          // (J, K, K) column-major, ld K; on exit: R above, reflectors below
  int K;
  const int32_t* kmax; // (J,) min(m_j, K)
  double sigma;
  double* tau;         // (J, K)
  int32_t* perm;       // (J, K)
  int32_t* rank;       // (J,)
  double* diag;        // (J, K) |R_ii| / |R_00|
};

__device__ __forceinline__ void argmax_lowest(double& v, int& i) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const double ov = __shfl_xor_sync(0xffffffffu, v, o);
    const int oi = __shfl_xor_sync(0xffffffffu, i, o);
    if (ov > v || (ov == v && oi < i)) {
      v = ov;
      i = oi;
    }
  }
}

__device__ __forceinline__ double blk_sum(double x, double* red) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  x = fl::warp_sum(x);
  if (lane == 0) red[wid] = x;
  __syncthreads();
  double s = 0.0;
  for (int w = 0; w < NW; ++w) s += red[w];
  __syncthreads();
  return s;
}

__global__ void __launch_bounds__(NT, 1) qrcp_kernel(QrcpArgs q) {
  extern __shared__ double sm[];
  const int K = q.K;
  const int j = blockIdx.x;
  const int M = q.kmax[j];   // rows of R0 that matter
  const int N = K;
  double* F = sm;                    // [PB][K]  (column-major: F[k*K + c])
  double* vn1 = F + PB * K;
  double* vn2 = vn1 + K;
  double* v = vn2 + K;               // current reflector rows i..M-1 (v[0] = 1)
  double* rowi = v + K;              // A(i, offset..offset+k) with the trailing 1
  int* piv = (int*)(rowi + PB + 1);
  int* flag = piv + K;               // recompute flags
  __shared__ double red[NW];
  __shared__ double redv[NW];
  __shared__ int redi[NW];
  __shared__ double auxv[PB];
  __shared__ int s_stop, s_rank, s_flagged;

  double* A = q.R0 + (int64_t)j * K * K;
  double* tau = q.tau + (int64_t)j * K;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const double tol3z = sqrt(DBL_EPSILON * 0.5);

  for (int c = threadIdx.x; c < N; c += NT) {
    piv[c] = c;
    flag[c] = 0;
  }
  for (int c = wid; c < N; c += NW) {
    double ss = 0.0;
    for (int r = lane; r < M; r += 32) ss += A[(int64_t)c * K + r] * A[(int64_t)c * K + r];
    ss = fl::warp_sum(ss);
    if (lane == 0) vn1[c] = vn2[c] = sqrt(ss);
  }
  if (threadIdx.x == 0) {
    s_stop = 0;
    s_rank = M;
  }
  __syncthreads();

  double lead = 0.0;
  int offset = 0;
  while (offset < M && !s_stop) {
    const int nbp = min(PB, M - offset);
    for (int p = threadIdx.x; p < PB * N; p += NT) F[p] = 0.0;
    if (threadIdx.x == 0) s_flagged = 0;
    __syncthreads();
    int k = 0;
    while (k < nbp && !s_flagged) {
      const int i = offset + k;
      // ---- pivot: first max of vn1 over current positions i..N-1 ----
      double bv = -1.0;
      int bi = N;
      for (int c = i + threadIdx.x; c < N; c += NT) {
        const double x = vn1[c];
        if (x > bv) {
          bv = x;
          bi = c;
        }
      }
      argmax_lowest(bv, bi);
      if (lane == 0) {
        redv[wid] = bv;
        redi[wid] = bi;
      }
      __syncthreads();
      if (wid == 0) {
        bv = lane < NW ? redv[lane] : -1.0;
        bi = lane < NW ? redi[lane] : N;
        argmax_lowest(bv, bi);
        if (lane == 0) redi[0] = bi;
      }
      __syncthreads();
      const int p = redi[0];
      if (p != i) {
        double* ci = A + (int64_t)i * K;
        double* cp = A + (int64_t)p * K;
        for (int r = threadIdx.x; r < M; r += NT) {
          const double t = ci[r];
          ci[r] = cp[r];
          cp[r] = t;
        }
        if (threadIdx.x < k) {
          const double t = F[threadIdx.x * K + i];
          F[threadIdx.x * K + i] = F[threadIdx.x * K + p];
          F[threadIdx.x * K + p] = t;
        }
        if (threadIdx.x == 0) {
          const int t = piv[p];
          piv[p] = piv[i];
          piv[i] = t;
          vn1[p] = vn1[i];
          vn2[p] = vn2[i];
          const int f = flag[p];
          flag[p] = flag[i];
          flag[i] = f;
        }
      }
      __syncthreads();
      // ---- A(i:M, i) -= A(i:M, offset:i) F(i, 0:k)^T ; load into v ----
      double* col = A + (int64_t)i * K;
      for (int r = i + threadIdx.x; r < M; r += NT) {
        double x = col[r];
        for (int kk = 0; kk < k; ++kk) x -= A[(int64_t)(offset + kk) * K + r] * F[kk * K + i];
        v[r - i] = x;
      }
      __syncthreads();
      // ---- dlarfg ----
      double ss = 0.0;
      for (int r = i + 1 + threadIdx.x; r < M; r += NT) ss += v[r - i] * v[r - i];
      const double alpha = v[0];
      ss = blk_sum(ss, red);
      const double xnorm = sqrt(ss);
      double beta, t;
      if (xnorm == 0.0) {
        t = 0.0;
        beta = alpha;
      } else {
        beta = -copysign(hypot(alpha, xnorm), alpha);
        t = (beta - alpha) / beta;
        const double scal = 1.0 / (alpha - beta);
        for (int r = i + 1 + threadIdx.x; r < M; r += NT) v[r - i] *= scal;
      }
      if (i == 0) lead = fabs(beta);
      if (q.sigma > 0.0 && (lead == 0.0 || fabs(beta) < q.sigma * lead)) {
        if (threadIdx.x == 0) {
          s_stop = 1;
          s_rank = i;
        }
        __syncthreads();
        break;
      }
      __syncthreads();
      if (threadIdx.x == 0) {
        v[0] = 1.0;
        tau[i] = t;
        q.diag[(int64_t)j * K + i] = fabs(beta);
      }
      // write the reflector (below the diagonal) and R_ii = beta
      for (int r = i + 1 + threadIdx.x; r < M; r += NT) col[r] = v[r - i];
      if (threadIdx.x == 0) col[i] = beta;
      __syncthreads();
      // ---- F(i+1:N, k) = t * A(i:M, i+1:N)^T v  (trailing columns, un-updated) ----
      for (int c = i + 1 + wid; c < N; c += NW) {
        const double* cc = A + (int64_t)c * K;
        double d = 0.0;
        for (int r = i + lane; r < M; r += 32) d += cc[r] * v[r - i];
        d = fl::warp_sum(d);
        if (lane == 0) F[k * K + c] = t * d;
      }
      // ---- auxv = -t * A(i:M, offset:i)^T v ----
      for (int kk = wid; kk < k; kk += NW) {
        const double* cc = A + (int64_t)(offset + kk) * K;
        double d = 0.0;
        for (int r = i + lane; r < M; r += 32) d += cc[r] * v[r - i];
        d = fl::warp_sum(d);
        if (lane == 0) auxv[kk] = -t * d;
      }
      __syncthreads();
      // ---- F(:, k) += F(:, 0:k) auxv ; F(offset..i, k) = 0 ----
      for (int c = offset + threadIdx.x; c < N; c += NT) {
        double f = (c <= i) ? 0.0 : F[k * K + c];
        for (int kk = 0; kk < k; ++kk) f += F[kk * K + c] * auxv[kk];
        F[k * K + c] = f;
      }
      // row i of the panel columns: A(i, offset+kk) (reflector entries), 1 at k
      if (threadIdx.x <= k) rowi[threadIdx.x] = (threadIdx.x == k) ? 1.0 : A[(int64_t)(offset + threadIdx.x) * K + i];
      __syncthreads();
      // ---- A(i, i+1:N) -= A(i, offset:i+1) F(i+1:N, 0:k+1)^T ; downdate ----
      for (int c = i + 1 + threadIdx.x; c < N; c += NT) {
        double x = A[(int64_t)c * K + i];
        for (int kk = 0; kk <= k; ++kk) x -= rowi[kk] * F[kk * K + c];
        A[(int64_t)c * K + i] = x;
        if (i + 1 < M && vn1[c] != 0.0) {
          double tt = fabs(x) / vn1[c];
          tt = fmax(0.0, (1.0 + tt) * (1.0 - tt));
          const double rr = vn1[c] / vn2[c];
          if (tt * rr * rr <= tol3z) {
            flag[c] = 1;
            s_flagged = 1;
          } else {
            vn1[c] *= sqrt(tt);
          }
        }
      }
      __syncthreads();
      ++k;
    }
    if (s_stop) break;
    const int kb = k;
    const int rk = offset + kb;  // first row/col of the trailing block
    // ---- block update: A(rk:M, rk:N) -= A(rk:M, offset:rk) F(rk:N, 0:kb)^T  (DMMA) ----
    if (rk < M && rk < N) {
      const int g = lane >> 2, t4 = lane & 3;
      const int nrt = (M - rk + 7) / 8, nct = (N - rk + 7) / 8;
      for (int tile = wid; tile < nrt * nct; tile += NW) {
        const int r8 = rk + (tile % nrt) * 8, c8 = rk + (tile / nrt) * 8;
        const int row = r8 + g, c0 = c8 + 2 * t4;
        double d0 = (row < M && c0 < N) ? A[(int64_t)c0 * K + row] : 0.0;
        double d1 = (row < M && c0 + 1 < N) ? A[(int64_t)(c0 + 1) * K + row] : 0.0;
        for (int k0 = 0; k0 < kb; k0 += 4) {
          const int kk = k0 + t4;
          const double av = (row < M && kk < kb) ? -A[(int64_t)(offset + kk) * K + row] : 0.0;
          const int cb = c8 + g;
          const double bv = (cb < N && kk < kb) ? F[kk * K + cb] : 0.0;
          fl::dmma(d0, d1, av, bv);
        }
        if (row < M && c0 < N) A[(int64_t)c0 * K + row] = d0;
        if (row < M && c0 + 1 < N) A[(int64_t)(c0 + 1) * K + row] = d1;
      }
    }
    __syncthreads();
    // ---- recompute flagged norms over rows rk..M-1 ----
    for (int c = rk + wid; c < N; c += NW) {
      if (!flag[c]) continue;
      double ss = 0.0;
      for (int r = rk + lane; r < M; r += 32) ss += A[(int64_t)c * K + r] * A[(int64_t)c * K + r];
      ss = fl::warp_sum(ss);
      if (lane == 0) {
        vn1[c] = vn2[c] = (rk < M) ? sqrt(ss) : 0.0;
        flag[c] = 0;
      }
    }
    __syncthreads();
    offset = rk;
  }
  __syncthreads();
  const int rank = s_rank;
  for (int c = threadIdx.x; c < K; c += NT) {
    q.perm[(int64_t)j * K + c] = piv[c];
    if (c >= rank) q.diag[(int64_t)j * K + c] = 0.0;
  }
  __syncthreads();
  if (threadIdx.x == 0) q.rank[j] = rank;
  // diag ratios |R_ii| / |R_00|
  for (int c = threadIdx.x; c < rank; c += NT)
    q.diag[(int64_t)j * K + c] = lead > 0.0 ? q.diag[(int64_t)j * K + c] / lead : 0.0;
}

}  // namespace

namespace fl {
int qrcp_r0(double* R0, int K, const int32_t* kmax, int J, double sigma, double* tau, int32_t* perm,
            int32_t* rank, double* diag, cudaStream_t s) {
  const size_t smem = (size_t)(PB * K + 3 * K + PB + 1) * sizeof(double) + (size_t)2 * K * sizeof(int);
  if (smem > 220 * 1024) return FL_ERR_INVALID;
  FL_CUDA(cudaFuncSetAttribute(qrcp_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  QrcpArgs a{R0, K, kmax, sigma, tau, perm, rank, diag};
  qrcp_kernel<<<J, NT, smem, s>>>(a);
  FL_CHECK_LAUNCH();
  return FL_OK;
}
}  // namespace fl
