// K2 — batched truncated column-pivoted Householder QR (reference:
// featlsq filtering.py:92-115 -> linalg.py:58-97, LAPACK dgeqp3 + dorgqr).
//
// One CTA per subdomain block, the block living in HBM/L2 (column-major,
// ld multiple of 16). Pivot rule = LAPACK dlaqp2: first maximum of the
// partial column norms over the *current* (swapped) positions (IDAMAX),
// swap semantics for the norm arrays, reflector by dlarfg
// (beta = -sign(alpha) * hypot(alpha, ||x||), tau = (beta - alpha)/beta),
// norm downdate temp = max(0, 1 - (|r_ij|/vn1)^2), recomputed from the
// column when temp * (vn1/vn2)^2 <= sqrt(eps). The reference's truncation
// (|R_tt| < sigma |R_00|, strict; sigma = 0 keeps min(m, K); R_00 = 0 keeps
// nothing unless sigma = 0) is applied on the fly: the first r steps of QRCP
// do not depend on later ones, so stopping at r gives the same kept
// sequence, R and Q columns as the full factorisation followed by slicing.
// The thin Q (r columns) is then formed in place from the kept reflectors
// (dorg2r order) and sign-normalised with R so diag(R) > 0 (linalg.py:92-96).
//
// Reductions (column norms, dots, argmax) use fixed warp-shuffle trees and
// a fixed warp order, so the factorisation is run-to-run deterministic.
#include <float.h>

#include "common.cuh"

namespace {

constexpr int NT = 512;
constexpr int NW = NT / 32;

__device__ __forceinline__ void argmax_lowest(double& v, int& i) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    double ov = __shfl_xor_sync(0xffffffffu, v, o);
    int oi = __shfl_xor_sync(0xffffffffu, i, o);
    if (ov > v || (ov == v && oi < i)) {
      v = ov;
      i = oi;
    }
  }
}

__global__ void __launch_bounds__(NT) rrqr_kernel(fl_blockop b, int K, double sigma, double* __restrict__ Rout,
                                                  int32_t* __restrict__ perm_out,
                                                  int32_t* __restrict__ rank_out,
                                                  double* __restrict__ diag_out, int mmax) {
  extern __shared__ double smem[];
  double* vn1 = smem;
  double* vn2 = vn1 + K;
  double* tau = vn2 + K;
  double* bet = tau + K;
  double* vref = bet + K;                 // reflector, mmax doubles
  int* piv = (int*)(vref + mmax);
  __shared__ double red[NW];
  __shared__ int redi[NW];
  __shared__ int s_rank;

  const int j = blockIdx.x;
  const int m = b.m[j];
  const int64_t ld = b.ld[j];
  double* A = const_cast<double*>(b.vals) + b.off[j];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const double tol3z = sqrt(DBL_EPSILON * 0.5);
  const int kmax = m < K ? m : K;

  for (int c = threadIdx.x; c < K; c += NT) piv[c] = c;
  // initial column norms (dgeqp3: dnrm2 of every free column)
  for (int c = wid; c < K; c += NW) {
    const double* col = A + c * ld;
    double ss = 0.0;
    for (int r = lane; r < m; r += 32) ss += col[r] * col[r];
    ss = fl::warp_sum(ss);
    if (lane == 0) {
      vn1[c] = sqrt(ss);
      vn2[c] = vn1[c];
    }
  }
  if (threadIdx.x == 0) s_rank = kmax;
  __syncthreads();
  // linalg.py:51-55: non-finite entries are an input error (rank = -1)
  {
    int bad = 0;
    for (int c = threadIdx.x; c < K; c += NT) bad |= !isfinite(vn1[c]);
    if (__syncthreads_or(bad)) {
      if (threadIdx.x == 0) rank_out[j] = -1;
      return;
    }
  }

  double lead = 0.0;
  for (int i = 0; i < kmax; ++i) {
    // ---- pivot: first max over current positions i..K-1 (IDAMAX) ----
    double bv = -1.0;
    int bi = K;
    for (int c = i + threadIdx.x; c < K; c += NT) {
      double x = vn1[c];
      if (x > bv) {  // strictly greater keeps the lowest index per thread
        bv = x;
        bi = c;
      }
    }
    argmax_lowest(bv, bi);
    if (lane == 0) {
      red[wid] = bv;
      redi[wid] = bi;
    }
    __syncthreads();
    if (wid == 0) {
      bv = lane < NW ? red[lane] : -1.0;
      bi = lane < NW ? redi[lane] : K;
      argmax_lowest(bv, bi);
      if (lane == 0) redi[0] = bi;
    }
    __syncthreads();
    const int p = redi[0];
    if (p != i) {
      double* ci = A + i * ld;
      double* cp = A + p * ld;
      for (int r = threadIdx.x; r < m; r += NT) {
        double t = ci[r];
        ci[r] = cp[r];
        cp[r] = t;
      }
      __syncthreads();
      if (threadIdx.x == 0) {
        int t = piv[p];
        piv[p] = piv[i];
        piv[i] = t;
        vn1[p] = vn1[i];
        vn2[p] = vn2[i];
      }
    }
    __syncthreads();

    // ---- dlarfg on A[i:m, i] ----
    double* col = A + i * ld;
    const double alpha = col[i];  // read before block_sum's barriers: thread 0 overwrites it below
    double ss = 0.0;
    for (int r = i + 1 + threadIdx.x; r < m; r += NT) {
      double x = col[r];
      vref[r - i] = x;
      ss += x * x;
    }
    ss = fl::block_sum(ss, red);
    const double xnorm = sqrt(ss);
    double beta, t;
    if (xnorm == 0.0) {
      t = 0.0;
      beta = alpha;
    } else {
      beta = -copysign(hypot(alpha, xnorm), alpha);
      t = (beta - alpha) / beta;
      const double scal = 1.0 / (alpha - beta);
      for (int r = i + 1 + threadIdx.x; r < m; r += NT) {
        double x = vref[r - i] * scal;
        vref[r - i] = x;
        col[r] = x;
      }
    }
    if (threadIdx.x == 0) {
      col[i] = beta;
      vref[0] = 1.0;
      tau[i] = t;
      bet[i] = beta;
    }
    if (i == 0) lead = fabs(beta);
    // ---- truncation (linalg.py:75-85), decided at step i ----
    if (sigma > 0.0 && (lead == 0.0 || fabs(beta) < sigma * lead)) {
      if (threadIdx.x == 0) s_rank = i;
      __syncthreads();
      break;
    }
    __syncthreads();

    // ---- apply H_i to A[i:m, i+1:K] and downdate the partial norms ----
    for (int c = i + 1 + wid; c < K; c += NW) {
      double* cc = A + c * ld;
      double dot = 0.0;
      if (t != 0.0) {
        for (int r = i + lane; r < m; r += 32) dot += vref[r - i] * cc[r];
        dot = fl::warp_sum(dot) * t;
      }
      double sst = 0.0;  // sum of squares of the updated A[i+1:m, c]
      for (int r = i + lane; r < m; r += 32) {
        double x = cc[r];
        if (t != 0.0) {
          x -= dot * vref[r - i];
          cc[r] = x;
        }
        if (r > i) sst += x * x;
      }
      sst = fl::warp_sum(sst);
      if (lane == 0) {
        const double v1 = vn1[c];
        if (v1 != 0.0) {
          const double q = fabs(cc[i]) / v1;
          double temp = 1.0 - q * q;
          temp = temp > 0.0 ? temp : 0.0;
          const double rr = v1 / vn2[c];
          const double temp2 = temp * rr * rr;
          if (temp2 <= tol3z) {
            const double nv = (i + 1 < m) ? sqrt(sst) : 0.0;
            vn1[c] = nv;
            vn2[c] = nv;
          } else {
            vn1[c] = v1 * sqrt(temp);
          }
        }
      }
    }
    __syncthreads();
  }
  __syncthreads();
  const int rank = s_rank;

  // ---- outputs: perm, |R_tt|/|R_00|, R (sign-normalised), then thin Q ----
  for (int c = threadIdx.x; c < K; c += NT) {
    perm_out[(int64_t)j * K + c] = piv[c];
    diag_out[(int64_t)j * K + c] = (c < rank && lead > 0.0) ? fabs(bet[c]) / lead : 0.0;
  }
  double* Rj = Rout + (int64_t)j * K * K;
  for (int c = wid; c < rank; c += NW) {
    for (int r = lane; r < rank; r += 32) {
      double x = 0.0;
      if (r <= c) {
        double sg = bet[r] < 0.0 ? -1.0 : 1.0;
        x = A[c * ld + r] * sg;
      }
      Rj[(int64_t)c * K + r] = x;
    }
  }
  __syncthreads();

  // dorg2r: Q = H_0 ... H_{rank-1} E_rank, in place over columns 0..rank-1
  for (int i = rank - 1; i >= 0; --i) {
    double* col = A + i * ld;
    for (int r = i + 1 + threadIdx.x; r < m; r += NT) vref[r - i] = col[r];
    if (threadIdx.x == 0) vref[0] = 1.0;
    __syncthreads();
    const double t = tau[i];
    if (t != 0.0) {
      for (int c = i + 1 + wid; c < rank; c += NW) {
        double* cc = A + c * ld;
        double dot = 0.0;
        for (int r = i + lane; r < m; r += 32) dot += vref[r - i] * cc[r];
        dot = fl::warp_sum(dot) * t;
        for (int r = i + lane; r < m; r += 32) cc[r] -= dot * vref[r - i];
      }
    }
    for (int r = threadIdx.x; r < m; r += NT) {
      double x;
      if (r < i) x = 0.0;
      else if (r == i) x = 1.0 - t;
      else x = -t * vref[r - i];
      col[r] = x;
    }
    __syncthreads();
  }
  // sign normalisation of Q's columns
  for (int c = wid; c < rank; c += NW) {
    if (bet[c] < 0.0) {
      double* cc = A + c * ld;
      for (int r = lane; r < m; r += 32) cc[r] = -cc[r];
    }
  }
  if (threadIdx.x == 0) rank_out[j] = rank;
}

}  // namespace

extern "C" int fl_rrqr(const fl_blockop* blocks, int32_t K, int32_t max_rows, double sigma, double* R,
                       int32_t* perm, int32_t* rank, double* diag, void* stream) {
  if (!(sigma >= 0.0 && sigma < 1.0) || K < 1 || max_rows < 0) return FL_ERR_INVALID;
  if (blocks->nblocks == 0) return FL_OK;
  const int mmax = max_rows < 1 ? 1 : max_rows;
  size_t smem = (size_t)K * 4 * sizeof(double) + (size_t)mmax * sizeof(double) + (size_t)K * sizeof(int);
  if (smem > 220 * 1024) return FL_ERR_INVALID;
  cudaFuncSetAttribute(rrqr_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  rrqr_kernel<<<blocks->nblocks, NT, smem, (cudaStream_t)stream>>>(*blocks, K, sigma, R, perm, rank, diag, mmax);
  FL_CHECK_LAUNCH();
  return FL_OK;
}
