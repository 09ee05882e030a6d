// K2b — truncated column-pivoted QR of the triangular factor R0_j of every
// block (route R: QRCP(A_j) and QRCP(R0_j) choose the same pivots in exact
// arithmetic because partial column norms are invariant under the
// orthogonal Q0_j). One CTA per block (384 threads, one CTA
// per SM), R0_j (K x K, column-major, ld K) streamed from HBM/L2.
//
// Pivot rule and norm bookkeeping follow LAPACK's blocked dlaqps (what
// dgeqp3 runs on the leading columns): first maximum of the partial norms
// over current positions (IDAMAX, swap semantics), the panel F matrix
// (F[:, k] = tau_k A^T v_k with the incremental correction), row updates of
// the current row, downdate temp = max(0, (1 + t)(1 - t)), t = |a_rj|/vn1_j,
// columns with temp * (vn1/vn2)^2 <= sqrt(eps) flagged; their norms are
// recomputed at once from the panel-updated values (dlaqps closes the panel
// and recomputes after the block update: same exact-arithmetic value,
// DESIGN.md §3 K2). Truncation: the first step with |R_ii| < sigma |R_00|
// stops everything (linalg.py:75-85).
//
// Measured and removed variants (cfg4, one filter): dlaqps's literal early
// panel close (96.6 vs 91.3 ms then, 4x more block updates), an L2 bulk
// prefetch of the step's trailing columns behind the argmax (115.7 vs 89.6
// ms: evicted again before use), the reflector scaled by its readers instead
// of once in shared memory (72.6 vs 67.5 ms), gemv column groups from a
// shared counter (68.1 vs 67.6 ms), two 256-thread CTAs per SM (85-90 vs
// 67.5 ms: DRAM reads 327-351 vs 230 GB, round 2).
//
// 256-bit loads in the F-gemv (round 2): 72.9 vs 63.5 ms and 309 vs 235 GB of
// DRAM reads — LDG.E.ENL2.256 does not keep its lines in L1, so the
// evict_last reuse across a panel's steps is lost; they are used only in
// the block update, which streams.
//
// The step's critical path is a handful of dependent memory round trips, so
// the kernel is organised for memory-level parallelism: the column swap is
// fused with the pivot column's panel update (whose k panel values per row
// are loaded together), the F-gemv keeps eight columns x two 64-row chunks
// in flight per warp with 16-byte loads (the columns nearest the pivot with
// an L1 evict_last hint, since every step of a panel re-reads the same
// panel-start matrix), and the auxv dots issue eight loads per lane at a
// time.
#include <float.h>
#include <stdio.h>

#include <type_traits>

#include "wy.cuh"

namespace {

// measured on cfg4 (ncu, one filter): 256 threads x 2 CTAs/SM 89.0 ms;
// one CTA/SM: 384 threads 80.8 ms (166 registers), 512 81.6, 448 106.7,
// 320 129.6, 640 117.3; 512 with a 32-column panel 92.3 (spills)
constexpr int NT = 384;
constexpr int NW = NT / 32;
constexpr int QRCP_CU = 8;  // gemv: columns in flight per warp
constexpr int QRCP_UT = 4;  // block update: 8-column tiles loaded per trip (measured: 4 / 6 / 8 -> 64.6 / 65.0 / 65.2 ms)
// F-gemv loads: column groups starting < QRCP_L1KEEP trailing columns past the
// pivot use L1::evict_last, the rest L1::no_allocate. Measured on cfg4 (one
// filter): plain loads 80.8 ms; all no_allocate 79.7; keep 32 / 64 / 96 / 128
// / 160 / 192 / 256: 76.4 / 74.8 / 74.6 / 73.2 / 74.3 / 76.0 / 78.4; all
// evict_last 81.6. A keep width scaled to the panel's height (96 to 512 KB
// of trailing columns, 128 to 512 columns wide) measured 64.2 to 67.0 ms
// against 64.5 for the fixed 128 (round 2)
constexpr int QRCP_L1KEEP = 128;
constexpr int QRCP_MB = 1;
constexpr int PB = 16;  // panel width (F has PB columns)

struct QrcpArgs {
  double* R0;          // (J, K, K) column-major, ld K; on exit: R above, reflectors below
  int K;
  const int32_t* kmax; // (J,) min(m_j, K)
  double sigma;
  double* tau;         // (J, K)
  int32_t* perm;       // (J, K)
  int32_t* rank;       // (J,)
  double* diag;        // (J, K) |R_ii| / |R_00|
  int J;
};

__device__ __forceinline__ double2 ld_keep(const double* p) {
  double2 v;
  asm volatile("ld.global.L1::evict_last.v2.f64 {%0, %1}, [%2];\n" : "=d"(v.x), "=d"(v.y) : "l"(p));
  return v;
}
__device__ __forceinline__ double2 ld_stream(const double* p) {
  double2 v;
  asm volatile("ld.global.L1::no_allocate.v2.f64 {%0, %1}, [%2];\n" : "=d"(v.x), "=d"(v.y) : "l"(p));
  return v;
}

__device__ __forceinline__ fl::d4 ld_stream4(const double* p) {
  fl::d4 v;
  asm volatile("ld.global.L1::no_allocate.v4.f64 {%0, %1, %2, %3}, [%4];\n"
               : "=d"(v.a), "=d"(v.b), "=d"(v.c), "=d"(v.d)
               : "l"(p));
  return v;
}
__device__ __forceinline__ double ld_keep1(const double* p) {
  double v;
  asm volatile("ld.global.L1::evict_last.f64 %0, [%1];\n" : "=d"(v) : "l"(p));
  return v;
}
// panel columns (re-read by the auxv dots every step of the panel) kept in
// L1; the block update's once-per-panel read-modify-write streams past it
#define QRCP_LD_PANEL(p) ld_keep1(p)

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

#ifdef QRCP_PHASES  // diagnostic build: cycles per phase of the pivot step (thread 0's clock)
#define PH(n)                                  \
  do {                                         \
    if (threadIdx.x == 0) {                    \
      const long long t_ = clock64();          \
      ph_acc[n] += t_ - ph_last;               \
      ph_last = t_;                            \
    }                                          \
  } while (0)
#else
#define PH(n)
#endif

__global__ void __launch_bounds__(NT, QRCP_MB) qrcp_kernel(QrcpArgs q) {
  extern __shared__ double sm[];
#ifdef QRCP_PHASES
  long long ph_acc[10] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
  long long ph_last = clock64();
  int ph_steps = 0, ph_flag = 0;
#endif
  const int K = q.K;
  for (int j = blockIdx.x; j < q.J; j += gridDim.x) {
  const int M = q.kmax[j];
  const int N = K;
  double* F = sm;                    // [PB][K]  F[k*K + c]
  double* vn1 = F + PB * K;
  double* vn2 = vn1 + K;
  double* v = vn2 + K;               // pivot column rows i..M-1 (unscaled)
  double* rowA = v + K;              // prefetched A(i, c) of the trailing columns
  int* piv = (int*)(rowA + K);
  int* flag = piv + K;
  __shared__ double red[NW];
  __shared__ double redv[NW];
  __shared__ int redi[NW];
  __shared__ double auxv[PB];
  __shared__ double fred[8 * NW];
  __shared__ double rowi[PB + 1];
  __shared__ int s_stop, s_rank, s_flagged, s_p;
  __shared__ double s_alpha;

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
  int s_pl = 0;
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
      {
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
        // every warp reduces the NW candidates itself (no second barrier)
        bv = lane < NW ? redv[lane] : -1.0;
        bi = lane < NW ? redi[lane] : N;
        argmax_lowest(bv, bi);
        s_pl = bi;
      }
      PH(0);
      const int p = s_pl;
      // ---- swap columns i <-> p fused with the pivot column's panel update:
      //      v = A(i:M, p) - A(i:M, offset:i) F(p, 0:k)^T ----
      double* ci = A + (int64_t)i * K;
      double* cp = A + (int64_t)p * K;
      double ss = 0.0;  // dlarfg's ||v(i+1:M)||^2, summed as the column is formed
      auto form_row = [&](int r, double xi, double xp) {
        if (p != i) cp[r] = xi;
        if (r < i) {
          if (p != i) ci[r] = xp;
        } else {
          // the panel values are loaded together (one round trip, not k)
          double pa[PB];
#pragma unroll
          for (int kk = 0; kk < PB; ++kk) pa[kk] = (kk < k) ? QRCP_LD_PANEL(A + (int64_t)(offset + kk) * K + r) : 0.0;
#pragma unroll
          for (int kk = 0; kk < PB; ++kk)
            if (kk < k) xp -= pa[kk] * F[kk * K + p];
          v[r - i] = xp;
          if (r > i) ss += xp * xp;
          if (r == i) s_alpha = xp;
        }
      };
      // a thread's rows r and r + NT (M <= 2 NT for every K of this route):
      // both rows' column values are requested before either is used
      for (int r = threadIdx.x; r < M; r += 2 * NT) {
        const int r2 = r + NT;
        const double xi = ci[r], xp = cp[r];
        const double xi2 = r2 < M ? ci[r2] : 0.0, xp2 = r2 < M ? cp[r2] : 0.0;
        form_row(r, xi, xp);
        if (r2 < M) form_row(r2, xi2, xp2);
      }
      ss = fl::warp_sum(ss);
      if (lane == 0) red[wid] = ss;
      __syncthreads();
      PH(1);
      // row i of the trailing columns (final once the swap is done) and of
      // the panel columns: 8-byte cp.async into shared memory, waited for
      // only before the row update, so the round trip overlaps dlarfg and the
      // gemv without holding registers
      for (int c = i + 1 + threadIdx.x; c < N; c += NT)
        asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(
                         (unsigned)__cvta_generic_to_shared(rowA + c)),
                     "l"(A + (int64_t)c * K + i)
                     : "memory");
      if (threadIdx.x < k)
        asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(
                         (unsigned)__cvta_generic_to_shared(rowi + threadIdx.x)),
                     "l"(A + (int64_t)(offset + threadIdx.x) * K + i)
                     : "memory");
      if (p != i) {
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
      // ---- dlarfg (the norm's warp partials are in red) ----
      ss = 0.0;
#pragma unroll
      for (int w = 0; w < NW; ++w) ss += red[w];
      const double alpha = s_alpha;
      const bool xzero = ss == 0.0;  // sqrt(ss) == 0 exactly when ss == 0
      double beta, t;
      if (xzero) {
        t = 0.0;
        beta = alpha;
      } else {
        // ||(alpha, x)|| from the sum of squares with one sqrt on the step's
        // critical path (dlapy2's scaled form only outside the safe range)
        const double n2 = fma(alpha, alpha, ss);
        const double nrm = (n2 > 1e-280 && n2 < 1e280 && ss > 1e-280) ? sqrt(n2) : hypot(alpha, sqrt(ss));
        beta = -copysign(nrm, alpha);
        t = (beta - alpha) / beta;
      }
      if (i == 0) lead = fabs(beta);
      if (q.sigma > 0.0 && (lead == 0.0 || fabs(beta) < q.sigma * lead)) {
        if (threadIdx.x == 0) {
          s_stop = 1;
          s_rank = i;
        }
        asm volatile("cp.async.wait_all;\n" ::: "memory");  // no copies in flight at exit
        __syncthreads();
        break;
      }
      // v = x * scal (dlarfg's dscal), v_i = 1, scaled once in shared memory
      // (one more barrier) and read as is below
      const double scal = xzero ? 1.0 : 1.0 / (alpha - beta);
      for (int r = i + 1 + threadIdx.x; r < M; r += NT) {
        const double x = v[r - i] * scal;
        v[r - i] = x;
        ci[r] = x;  // reflector below the diagonal
      }
      if (threadIdx.x == 0) v[0] = 1.0;
      __syncthreads();
      PH(2);
      if (threadIdx.x == 0) {
        tau[i] = t;
        ci[i] = beta;
        q.diag[(int64_t)j * K + i] = fabs(beta);
      }
      auto wv = [&](int r) { return v[r - i]; };
      // ---- F(i+1:N, k) = t A(i:M, i+1:N)^T v ; auxv = -t A(i:M, offset:i)^T v ----
      {
        const int ncol = N - i - 1;
        // 16-byte loads: lane owns rows (2l, 2l+1) of each 64-row chunk, starting at
        // the even row i0 <= i (row i-1 contributes v = 0); two chunks per trip
        constexpr int CU = QRCP_CU;  // columns in flight per warp
        const int i0 = i & ~1;
        for (int c0 = wid * CU; c0 < ncol; c0 += NW * CU) {
          double d[CU];
          const double* cc[CU];
#pragma unroll
          for (int u = 0; u < CU; ++u) {
            d[u] = 0.0;
            cc[u] = A + (int64_t)(i + 1 + min(c0 + u, ncol - 1)) * K;
          }
          // the first QRCP_L1KEEP trailing columns stay in L1 across the
          // panel's steps (the gemv re-reads the same panel-start matrix);
          // the rest stream past L1. One loop per load kind (no select).
          auto rows_loop = [&](auto keep_tag) {
            constexpr bool KEEPL1 = decltype(keep_tag)::value;
            for (int r = i0 + 2 * lane; r < M; r += 128) {
              const int r2 = r + 64;
              const double v0 = (r >= i) ? wv(r) : 0.0;
              const double v1 = (r + 1 < M) ? wv(r + 1) : 0.0;
              const bool two = r2 < M;
              const double w0 = two ? wv(r2) : 0.0;
              const double w1 = (r2 + 1 < M) ? wv(r2 + 1) : 0.0;
              double2 x[CU], y[CU];
#pragma unroll
              for (int u = 0; u < CU; ++u) {
                x[u] = KEEPL1 ? ld_keep(cc[u] + r) : ld_stream(cc[u] + r);
                y[u] = two ? (KEEPL1 ? ld_keep(cc[u] + r2) : ld_stream(cc[u] + r2)) : make_double2(0.0, 0.0);
              }
#pragma unroll
              for (int u = 0; u < CU; ++u) d[u] += x[u].x * v0 + x[u].y * v1 + y[u].x * w0 + y[u].y * w1;
            }
          };
          if (c0 < QRCP_L1KEEP) rows_loop(std::true_type{});
          else rows_loop(std::false_type{});
          {
            const double s = fl::warp_multi_sum<CU>(d);  // lane l: column u = l / (32 / CU)
            const int u = lane / (32 / CU);
            if ((lane & (32 / CU - 1)) == 0 && c0 + u < ncol) F[k * K + i + 1 + c0 + u] = t * s;
          }
        }
        PH(3);
        for (int kk = wid; kk < k; kk += NW) {
          const double* cc = A + (int64_t)(offset + kk) * K;
          double dd = 0.0;
          for (int r0 = i + lane; r0 < M; r0 += 32 * 8) {  // 8 loads in flight per lane
            double x[8];
#pragma unroll
            for (int q = 0; q < 8; ++q) x[q] = (r0 + 32 * q < M) ? QRCP_LD_PANEL(cc + r0 + 32 * q) : 0.0;
#pragma unroll
            for (int q = 0; q < 8; ++q)
              if (r0 + 32 * q < M) dd += x[q] * wv(r0 + 32 * q);
          }
          dd = fl::warp_sum(dd);
          if (lane == 0) auxv[kk] = -t * dd;
        }
        if (threadIdx.x == k) rowi[k] = 1.0;
        PH(4);
        asm volatile("cp.async.wait_all;\n" ::: "memory");
      }
      __syncthreads();
      PH(5);
      // ---- F(:, k) += F(:, 0:k) auxv (F(offset..i, k) = 0 first);
      //      A(i, i+1:N) -= A(i, offset:i+1) F(i+1:N, 0:k+1)^T ; downdate ----
      for (int c = offset + threadIdx.x; c < N; c += NT) {
        double f = (c <= i) ? 0.0 : F[k * K + c];
        for (int kk = 0; kk < k; ++kk) f += F[kk * K + c] * auxv[kk];
        F[k * K + c] = f;
        if (c > i) {
          double x = rowA[c];
          for (int kk = 0; kk <= k; ++kk) x -= rowi[kk] * F[kk * K + c];
          A[(int64_t)c * K + i] = x;
          if (i + 1 < M && vn1[c] != 0.0) {
            double tt = fabs(x) / vn1[c];
            tt = fmax(0.0, (1.0 + tt) * (1.0 - tt));
            const double rr = vn1[c] / vn2[c];
            if (tt * rr * rr <= tol3z) {
              flag[atomicAdd(&s_flagged, 1)] = c;
            } else {
              vn1[c] *= sqrt(tt);
            }
          }
        }
      }
      __syncthreads();
      PH(6);
      // ---- flagged columns: instead of closing the panel (dlaqps), their
      //      norms are recomputed now from the panel-updated values
      //      A(i+1:M, c) - A(i+1:M, offset:i+1) F(c, 0:k+1)^T, which are what
      //      the block update would leave there (same exact-arithmetic value,
      //      no extra pass over the trailing matrix) ----
      if (s_flagged) {
        // all threads share the rows; the panel values of a row are loaded
        // once for up to FB flagged columns, warp partials summed in order
        constexpr int FB = 4;
        const int nf = s_flagged;
        for (int f0 = 0; f0 < nf; f0 += FB) {
          const int nb = min(FB, nf - f0);
          double s2[FB];
#pragma unroll
          for (int f = 0; f < FB; ++f) s2[f] = 0.0;
          for (int r = i + 1 + threadIdx.x; r < M; r += NT) {
            double pa[PB];
#pragma unroll
            for (int kk = 0; kk < PB; ++kk) pa[kk] = (kk <= k) ? QRCP_LD_PANEL(A + (int64_t)(offset + kk) * K + r) : 0.0;
            double x[FB];
#pragma unroll
            for (int f = 0; f < FB; ++f) x[f] = (f < nb) ? A[(int64_t)flag[f0 + f] * K + r] : 0.0;
#pragma unroll
            for (int f = 0; f < FB; ++f) {
              if (f < nb) {
                const int c = flag[f0 + f];
#pragma unroll
                for (int kk = 0; kk < PB; ++kk)
                  if (kk <= k) x[f] -= pa[kk] * F[kk * K + c];
                s2[f] += x[f] * x[f];
              }
            }
          }
#pragma unroll
          for (int f = 0; f < FB; ++f) {
            if (f < nb) {
              const double w = fl::warp_sum(s2[f]);
              if (lane == 0) fred[f * NW + wid] = w;
            }
          }
          __syncthreads();
          if (threadIdx.x < nb) {
            double t2 = 0.0;
#pragma unroll
            for (int w = 0; w < NW; ++w) t2 += fred[threadIdx.x * NW + w];
            const int c = flag[f0 + threadIdx.x];
            vn1[c] = vn2[c] = (i + 1 < M) ? sqrt(t2) : 0.0;
          }
          __syncthreads();
        }
        if (threadIdx.x == 0) s_flagged = 0;
        __syncthreads();
#ifdef QRCP_PHASES
        ++ph_flag;
#endif
      }
      PH(7);
#ifdef QRCP_PHASES
      ++ph_steps;
#endif
      ++k;
    }
    if (s_stop) break;
    const int kb = k;
    const int rk = offset + kb;
    // ---- block update: A(rk:M, rk:N) -= A(rk:M, offset:rk) F(rk:N, 0:kb)^T  (DMMA) ----
    if (rk < M && rk < N) {
      // The MMA's m index is the trailing column and its n index the row. A
      // warp owns a 16-row strip (the panel values of its rows stay in
      // registers as B fragments, zero outside rk..M-1 so those rows are
      // rewritten unchanged) and walks 8-column tiles, UT at a time with all
      // their loads in flight. A lane's 256-bit access is rows rs + 4 t4 .. + 3
      // of its column (one full line per column and warp access): the pairs
      // (0, 1) and (2, 3) are the accumulators of two MMA tiles, tile h
      // holding rows rs + 4 (n / 2) + 2 h + n % 2.
      constexpr int KS = PB / 4, UT = QRCP_UT;
      const int g = lane >> 2, t4 = lane & 3;
      const int r0 = rk & ~15;
      const int nrs = (M - r0 + 15) / 16;
      const int ncg = nrs >= NW ? 1 : NW / nrs;
      const int nct = (N - rk + 7) / 8;
      for (int item = wid; item < nrs * ncg; item += NW) {
        const int rs = r0 + (item % nrs) * 16;
        double bq[2][KS];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int row = rs + 4 * (g >> 1) + 2 * h + (g & 1);
#pragma unroll
          for (int s2 = 0; s2 < KS; ++s2) {
            const int kk = 4 * s2 + t4;
            bq[h][s2] = (row >= rk && row < M && kk < kb) ? A[(int64_t)(offset + kk) * K + row] : 0.0;
          }
        }
        const int row = rs + 4 * t4;  // K is a multiple of 4: the lane's rows are inside the column together
        for (int ct0 = item / nrs; ct0 < nct; ct0 += ncg * UT) {
          fl::d4 cc[UT];
#pragma unroll
          for (int u = 0; u < UT; ++u) {
            const int col = rk + (ct0 + u * ncg) * 8 + g;
            cc[u] = (col < N && row < M) ? ld_stream4(A + (int64_t)col * K + row) : fl::d4{0.0, 0.0, 0.0, 0.0};
          }
#pragma unroll
          for (int u = 0; u < UT; ++u) {
            const int col = rk + (ct0 + u * ncg) * 8 + g;
#pragma unroll
            for (int s2 = 0; s2 < KS; ++s2) {
              const int kk = 4 * s2 + t4;
              const double af = (col < N && kk < kb) ? -F[kk * K + col] : 0.0;
              fl::dmma(cc[u].a, cc[u].b, af, bq[0][s2]);
              fl::dmma(cc[u].c, cc[u].d, af, bq[1][s2]);
            }
            if (col < N && row < M) fl::stg256(A + (int64_t)col * K + row, cc[u]);
          }
        }
      }
    }
    __syncthreads();
    PH(8);
    offset = rk;
  }
  __syncthreads();
  const int rank = s_rank;
  for (int c = threadIdx.x; c < K; c += NT) {
    q.perm[(int64_t)j * K + c] = piv[c];
    q.diag[(int64_t)j * K + c] =
        (c < rank && lead > 0.0) ? q.diag[(int64_t)j * K + c] / lead : 0.0;
  }
  if (threadIdx.x == 0) q.rank[j] = rank;
  __syncthreads();
#ifdef QRCP_PHASES
  PH(9);
  if (threadIdx.x == 0 && (j % 128) == 5)
    printf("QRCPPH j=%d steps=%d flagged=%d argmax=%lld pivcol=%lld dlarfg=%lld gemv=%lld auxv=%lld wait=%lld rowupd=%lld flag=%lld blockupd=%lld other=%lld\n",
           j, ph_steps, ph_flag, ph_acc[0], ph_acc[1], ph_acc[2], ph_acc[3], ph_acc[4], ph_acc[5], ph_acc[6],
           ph_acc[7], ph_acc[8], ph_acc[9]);
#endif
  }
}

}  // namespace

namespace fl {
int qrcp_r0(double* R0, int K, const int32_t* kmax, int J, double sigma, double* tau, int32_t* perm,
            int32_t* rank, double* diag, cudaStream_t s) {
  const size_t smem = (size_t)(PB * K + 4 * K) * sizeof(double) + (size_t)2 * K * sizeof(int);
  if (smem > (QRCP_MB > 1 ? 110 : 220) * 1024) return FL_ERR_INVALID;
  FL_CUDA(cudaFuncSetAttribute(qrcp_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  QrcpArgs a{R0, K, kmax, sigma, tau, perm, rank, diag, J};
  qrcp_kernel<<<J, NT, smem, s>>>(a);
  FL_CHECK_LAUNCH();
  return FL_OK;
}
}  // namespace fl
