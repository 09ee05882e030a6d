// N4 — additive-Schwarz setup (reference: featlsq solvers.py:178-192):
// per block the Gramian G_j = A_j^T A_j, its eigendecomposition and the
// pseudo-inverse sum_{lambda_i > cutoff * lambda_max} v_i v_i^T / lambda_i,
// plus the "cutoff bit" (degenerate) flag. One CTA per block with G and the
// eigenvector matrix V in shared memory (K <= FL_AS_MAX_K).
//
// Eigensolver: cyclic two-sided Jacobi with the parallel round-robin
// ("circle") ordering — in every round the K/2 pairs are disjoint, so all
// rotations of a round are computed from the round's start values (the
// 2x2 block of a pair is touched by its own rotation only) and applied as
// one column pass (G J, V J) and one row pass (J^T G). Rotation angles
// follow Rutishauser (t = sgn(theta) / (|theta| + sqrt(theta^2 + 1))), a
// pair is skipped when |g_pq| <= eps sqrt(|g_pp g_qq|) (the relative
// criterion that keeps small eigenvalues accurate), sweeps stop when a
// whole sweep skipped every pair (at most 40 sweeps). The Gramian pass is
// HBM-light (the block is read once); the sweeps run from shared memory.
#include <float.h>

#include "common.cuh"

namespace {

constexpr int NT = 256;
constexpr int KMAX = FL_AS_MAX_K;
constexpr int LDG = KMAX + 1;  // padded row length of G and V in shared memory
constexpr int RC = 16;         // rows of A staged per Gramian chunk

__global__ void __launch_bounds__(NT) as_setup_kernel(fl_blockop A, double cutoff, double* __restrict__ inv,
                                                      int32_t* __restrict__ degenerate) {
  extern __shared__ double sm[];
  const int j = blockIdx.x;
  const int n = A.ncols[j];
  const int m = A.m[j], ld = A.ld[j];
  const double* a = A.vals + A.off[j];
  double* G = sm;                // n x n, row stride LDG
  double* V = G + KMAX * LDG;    // n x n, row stride LDG
  double* st = V + KMAX * LDG;   // RC x n staged rows of A
  double* cs = st + RC * KMAX;   // (c, s) per pair
  int* pr = reinterpret_cast<int*>(cs + KMAX);  // pair (p, q) per slot
  __shared__ int s_rot;
  __shared__ double s_top;

  // ---- G = A^T A (column-major A: entry (r, c) at a[c * ld + r]) ----
  constexpr int NU = (KMAX * (KMAX + 1) / 2 + NT - 1) / NT;  // upper-triangle entries per thread
  const int npairs_g = n * (n + 1) / 2;
  double acc[NU];
  int erow[NU], ecol[NU];
#pragma unroll
  for (int u = 0; u < NU; ++u) {
    acc[u] = 0.0;
    // entry e -> (row, col) of the upper triangle, row <= col
    int row = 0, rem = threadIdx.x + u * NT;
    while (row < n && rem >= n - row) {
      rem -= n - row;
      ++row;
    }
    erow[u] = row;
    ecol[u] = row + rem;
  }
  for (int r0 = 0; r0 < m; r0 += RC) {
    const int nr = min(RC, m - r0);
    __syncthreads();
    for (int p = threadIdx.x; p < RC * n; p += NT) {
      const int c = p / RC, r = p % RC;
      st[r * KMAX + c] = r < nr ? a[(int64_t)c * ld + r0 + r] : 0.0;
    }
    __syncthreads();
#pragma unroll
    for (int u = 0; u < NU; ++u) {
      if (threadIdx.x + u * NT < npairs_g) {
        double s = acc[u];
#pragma unroll 4
        for (int r = 0; r < RC; ++r) s += st[r * KMAX + erow[u]] * st[r * KMAX + ecol[u]];
        acc[u] = s;
      }
    }
  }
#pragma unroll
  for (int u = 0; u < NU; ++u) {
    if (threadIdx.x + u * NT < npairs_g) {
      G[erow[u] * LDG + ecol[u]] = acc[u];
      G[ecol[u] * LDG + erow[u]] = acc[u];
    }
  }
  for (int p = threadIdx.x; p < n * n; p += NT) V[(p / n) * LDG + p % n] = (p / n == p % n) ? 1.0 : 0.0;
  __syncthreads();

  // ---- cyclic Jacobi, round-robin ordering over n' = n rounded up to even ----
  const int np = n + (n & 1);
  const int half = np / 2;
  for (int sweep = 0; sweep < 40; ++sweep) {
    if (threadIdx.x == 0) s_rot = 0;
    __syncthreads();
    for (int round = 0; round < np - 1; ++round) {
      // circle method: position 0 fixed, the others rotate by `round`
      for (int k = threadIdx.x; k < half; k += NT) {
        auto member = [&](int pos) { return pos == 0 ? 0 : 1 + (pos - 1 + round) % (np - 1); };
        int p = member(k), q = member(np - 1 - k);
        if (p > q) {
          const int t = p;
          p = q;
          q = t;
        }
        double c = 1.0, s = 0.0;
        if (q < n) {
          const double gpp = G[p * LDG + p], gqq = G[q * LDG + q], gpq = G[p * LDG + q];
          if (fabs(gpq) > DBL_EPSILON * sqrt(fabs(gpp)) * sqrt(fabs(gqq)) && gpq != 0.0) {
            const double theta = (gqq - gpp) / (2.0 * gpq);
            const double t = copysign(1.0, theta) / (fabs(theta) + sqrt(theta * theta + 1.0));
            c = 1.0 / sqrt(t * t + 1.0);
            s = t * c;
            s_rot = 1;
          }
        }
        pr[2 * k] = p;
        pr[2 * k + 1] = q;
        cs[2 * k] = c;
        cs[2 * k + 1] = s;
      }
      __syncthreads();
      // columns: G <- G J, V <- V J  (pair k owns columns p, q)
      for (int e = threadIdx.x; e < half * n; e += NT) {
        const int k = e / n, row = e % n;
        const int p = pr[2 * k], q = pr[2 * k + 1];
        const double c = cs[2 * k], s = cs[2 * k + 1];
        if (q >= n || s == 0.0) continue;
        const double gp = G[row * LDG + p], gq = G[row * LDG + q];
        G[row * LDG + p] = c * gp - s * gq;
        G[row * LDG + q] = s * gp + c * gq;
        const double vp = V[row * LDG + p], vq = V[row * LDG + q];
        V[row * LDG + p] = c * vp - s * vq;
        V[row * LDG + q] = s * vp + c * vq;
      }
      __syncthreads();
      // rows: G <- J^T G
      for (int e = threadIdx.x; e < half * n; e += NT) {
        const int k = e / n, col = e % n;
        const int p = pr[2 * k], q = pr[2 * k + 1];
        const double c = cs[2 * k], s = cs[2 * k + 1];
        if (q >= n || s == 0.0) continue;
        const double gp = G[p * LDG + col], gq = G[q * LDG + col];
        G[p * LDG + col] = c * gp - s * gq;
        G[q * LDG + col] = s * gp + c * gq;
      }
      __syncthreads();
      // the rotated pair's off-diagonal entries are zero in exact arithmetic
      for (int k = threadIdx.x; k < half; k += NT) {
        const int p = pr[2 * k], q = pr[2 * k + 1];
        if (q < n && cs[2 * k + 1] != 0.0) G[p * LDG + q] = G[q * LDG + p] = 0.0;
      }
      __syncthreads();
    }
    if (!s_rot) break;
  }

  // ---- pseudo-inverse with the reference's cutoff (solvers.py:183-189) ----
  if (threadIdx.x == 0) {
    double top = -DBL_MAX;
    for (int i = 0; i < n; ++i) top = fmax(top, G[i * LDG + i]);
    s_top = n ? top : 0.0;
    int deg = 0;
    for (int i = 0; i < n; ++i) {
      const bool keep = s_top > 0.0 && G[i * LDG + i] > cutoff * s_top;
      cs[i] = keep ? 1.0 / G[i * LDG + i] : 0.0;
      deg |= !keep;
    }
    degenerate[j] = deg;
  }
  __syncthreads();
  double* out = inv + (int64_t)j * n * n;  // row-major n x n (fl_block_precond)
  for (int e = threadIdx.x; e < n * n; e += NT) {
    const int r = e / n, c = e % n;
    double s = 0.0;
    for (int i = 0; i < n; ++i) s += V[r * LDG + i] * cs[i] * V[c * LDG + i];
    out[e] = s;
  }
}

}  // namespace

extern "C" int fl_as_setup(const fl_blockop* A, double cutoff, double* inv, int32_t* degenerate, void* stream) {
  if (A->nblocks == 0) return FL_OK;
  if (A->max_ncols > FL_AS_MAX_K || A->max_ncols < 1) return FL_ERR_INVALID;
  const size_t smem = (size_t)(2 * KMAX * LDG + RC * KMAX + KMAX) * sizeof(double) + 2 * KMAX * sizeof(int);
  FL_CUDA(cudaFuncSetAttribute(as_setup_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  as_setup_kernel<<<A->nblocks, NT, smem, (cudaStream_t)stream>>>(*A, cutoff, inv, degenerate);
  FL_CHECK_LAUNCH();
  return FL_OK;
}
