// K2b, TMA-streamed variant — same algorithm and pivot rule as qrcp.cu
// (LAPACK dlaqps on R0_j, truncation at |R_ii| < sigma |R_00|), reorganised
// for memory-level parallelism: one CTA per block and per SM (16 consumer
// warps + 1 producer warp). The per-step F-gemv
//     F(i+1:N, k) = tau A(i:M, i+1:N)^T v
// streams every trailing column segment A(i0:M, c) (contiguous, i0 = i & ~1)
// through a ring of single-column shared-memory slots with cp.async.bulk:
// the producer starts streaming step i's columns as soon as the pivot swap of
// step i is done, so the reflector generation (dlarfg) overlaps the fetch and
// the consumers only wait for data. Row i of the trailing columns (needed by
// the row update) is taken from the streamed segments. Consumer-only phases
// synchronise with named barrier 1 (512 threads).
//
// Protocol (mbarriers): full[s] (TMA bytes), empty[s] (the consuming warp),
// go (consumer thread 0 publishes the step index after the swap; a negative
// index stops the producer). Column j of step i is global sequence number
// base_i + j, slot (base_i + j) % NS, issued by producer lane (base_i + j) %
// 32 and consumed by warp j % 16.
#include <float.h>

#include "wy.cuh"

namespace {

#ifndef QRCP2_NCW
#define QRCP2_NCW 16
#endif
#ifndef QRCP2_NS
#define QRCP2_NS 32
#endif
constexpr int NCW = QRCP2_NCW;       // consumer warps
constexpr int NTC = NCW * 32;        // consumer threads
constexpr int NT = NTC + 32;         // + producer warp
constexpr int PB = 16;               // panel width (F has PB columns)
constexpr int NS = QRCP2_NS;         // ring slots (one column segment each)
constexpr int MINB = NCW >= 16 ? 1 : 2;  // CTAs per SM
// a slot is reused NS columns later by the same consumer warp, so no warp
// ever waits on a slot's phase two ahead of its last completion
static_assert(NS % NCW == 0, "ring slots must be a multiple of the consumer warps");

struct QrcpArgs {
  double* R0;
  int K;
  const int32_t* kmax;
  double sigma;
  double* tau;
  int32_t* perm;
  int32_t* rank;
  double* diag;
};

__device__ __forceinline__ void csync() { asm volatile("bar.sync 1, %0;\n" ::"n"(NTC) : "memory"); }

__device__ __forceinline__ unsigned sa(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint64_t* b, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(sa(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(sa(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, unsigned parity) {
  unsigned ok = 0;
  while (!ok)
    asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }\n"
                 : "=r"(ok)
                 : "r"(sa(b)), "r"(parity)
                 : "memory");
}

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

__global__ void __launch_bounds__(NT, MINB) qrcp2_kernel(QrcpArgs q) {
  extern __shared__ __align__(128) double sm[];
  const int K = q.K;
  const int j = blockIdx.x;
  const int M = q.kmax[j];
  const int N = K;
  double* ring = sm;                 // [NS][K] column segments
  double* F = ring + NS * K;         // [PB][K]  F[k*K + c]
  double* vn1 = F + PB * K;
  double* vn2 = vn1 + K;
  double* v = vn2 + K;               // reflector, absolute rows (v[i-1] = 0)
  double* rowA = v + K;              // row i of the trailing columns
  int* piv = (int*)(rowA + K);
  int* flag = piv + K;
  __shared__ double red[NCW];
  __shared__ double redv[NCW];
  __shared__ int redi[NCW];
  __shared__ double auxv[PB];
  __shared__ double rowi[PB + 1];
  __shared__ int s_stop, s_rank, s_flagged, s_p, s_step;
  __shared__ __align__(8) uint64_t full[NS], empty[NS], go;

  double* A = q.R0 + (int64_t)j * K * K;
  double* tau = q.tau + (int64_t)j * K;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const double tol3z = sqrt(DBL_EPSILON * 0.5);

  if (threadIdx.x == 0) {
    for (int s = 0; s < NS; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(&go, 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();

  // ======================= producer warp =======================
  // lane l < NS owns ring slot l: it streams the columns whose global
  // sequence number is l mod NS, so NS copies are issued in parallel
  if (wid == NCW) {
    static_assert(NS <= 32, "one ring slot per producer lane");
    if (lane >= NS) return;
    int64_t base_p = 0;  // global sequence number of the step's first column
    for (unsigned step = 0;; ++step) {
      mbar_wait(&go, step & 1);
      const int i = *(volatile int*)&s_step;
      if (i < 0) return;
      const int i0 = i & ~1;
      const unsigned bytes = (unsigned)(M - i0) * 8u;
      const int ncol = N - i - 1;
      int64_t g = base_p + ((lane - base_p % NS) + NS) % NS;  // first g >= base_p with g % NS == lane
      for (; g < base_p + ncol; g += NS) {
        const int c = i + 1 + (int)(g - base_p);
        if (g >= NS) mbar_wait(&empty[lane], (unsigned)(((g / NS) - 1) & 1));
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(sa(&full[lane])), "r"(bytes)
                     : "memory");
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                sa(ring + (int64_t)lane * K)),
            "l"(A + (int64_t)c * K + i0), "r"(bytes), "r"(sa(&full[lane]))
            : "memory");
      }
      base_p += ncol;
    }
  }

  // ======================= consumers (512 threads) =======================
  const int tid = threadIdx.x;
  for (int c = tid; c < N; c += NTC) {
    piv[c] = c;
    flag[c] = 0;
  }
  for (int c = wid; c < N; c += NCW) {
    double ss = 0.0;
    for (int r = lane; r < M; r += 32) ss += A[(int64_t)c * K + r] * A[(int64_t)c * K + r];
    ss = fl::warp_sum(ss);
    if (lane == 0) vn1[c] = vn2[c] = sqrt(ss);
  }
  if (tid == 0) {
    s_stop = 0;
    s_rank = M;
  }
  csync();

  int64_t base = 0;       // global sequence number of this step's first column
  unsigned gostep = 0;    // steps published to the producer
  double lead = 0.0;
  int offset = 0;
  while (offset < M && !s_stop) {
    const int nbp = min(PB, M - offset);
    for (int p = tid; p < PB * N; p += NTC) F[p] = 0.0;
    if (tid == 0) s_flagged = 0;
    csync();
    int k = 0;
    while (k < nbp && !s_flagged) {
      const int i = offset + k;
      // ---- pivot: first max of vn1 over current positions i..N-1 ----
      {
        double bv = -1.0;
        int bi = N;
        for (int c = i + tid; c < N; c += NTC) {
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
        csync();
        if (wid == 0) {
          bv = lane < NCW ? redv[lane] : -1.0;
          bi = lane < NCW ? redi[lane] : N;
          argmax_lowest(bv, bi);
          if (lane == 0) s_p = bi;
        }
        csync();
      }
      const int p = s_p;
      // ---- swap columns i <-> p fused with the pivot column's panel update ----
      double* ci = A + (int64_t)i * K;
      double* cp = A + (int64_t)p * K;
      for (int r = tid; r < M; r += NTC) {
        const double xi = ci[r];
        double xp = cp[r];
        if (p != i) cp[r] = xi;
        if (r < i) {
          if (p != i) ci[r] = xp;
        } else {
          for (int kk = 0; kk < k; ++kk) xp -= A[(int64_t)(offset + kk) * K + r] * F[kk * K + p];
          v[r] = xp;
        }
      }
      // generic-proxy writes must be visible to the bulk copies that read them
      asm volatile("fence.proxy.async.global;\n" ::: "memory");
      csync();
      // the trailing columns are final for this step: start streaming them
      if (tid == 0) {
        s_step = i;
        mbar_arrive(&go);
      }
      ++gostep;
      if (p != i) {
        if (tid < k) {
          const double t = F[tid * K + i];
          F[tid * K + i] = F[tid * K + p];
          F[tid * K + p] = t;
        }
        if (tid == 0) {
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
      // ---- dlarfg ----
      double ss = 0.0;
      for (int r = i + 1 + tid; r < M; r += NTC) ss += v[r] * v[r];
      ss = fl::warp_sum(ss);
      if (lane == 0) red[wid] = ss;
      csync();
      ss = 0.0;
#pragma unroll
      for (int w = 0; w < NCW; ++w) ss += red[w];
      const double alpha = v[i];
      const double xnorm = sqrt(ss);
      double beta, t;
      if (xnorm == 0.0) {
        t = 0.0;
        beta = alpha;
      } else {
        beta = -copysign(hypot(alpha, xnorm), alpha);
        t = (beta - alpha) / beta;
      }
      if (i == 0) lead = fabs(beta);
      const int ncol = N - i - 1;
      const bool stop = q.sigma > 0.0 && (lead == 0.0 || fabs(beta) < q.sigma * lead);
      if (stop) {
        // drain this step's streamed columns, then stop
        for (int jj = wid; jj < ncol; jj += NCW) {
          const int64_t g = base + jj;
          mbar_wait(&full[g % NS], (unsigned)((g / NS) & 1));
          __syncwarp();
          if (lane == 0) mbar_arrive(&empty[g % NS]);
        }
        base += ncol;
        if (tid == 0) {
          s_stop = 1;
          s_rank = i;
        }
        csync();
        break;
      }
      {
        const double scal = (xnorm == 0.0) ? 1.0 : 1.0 / (alpha - beta);
        for (int r = i + 1 + tid; r < M; r += NTC) {
          const double x = v[r] * scal;
          v[r] = x;
          ci[r] = x;  // reflector below the diagonal
        }
      }
      csync();
      if (tid == 0) {
        v[i] = 1.0;
        if (i & 1) v[i - 1] = 0.0;
        tau[i] = t;
        ci[i] = beta;
        q.diag[(int64_t)j * K + i] = fabs(beta);
      }
      csync();
      // ---- F(i+1:N, k) = t A(i:M, i+1:N)^T v over the streamed segments;
      //      rowA = A(i, i+1:N) from the same segments ----
      {
        const int i0 = i & ~1;
        const int len = M - i0;
        for (int jj = wid; jj < ncol; jj += NCW) {
          const int64_t g = base + jj;
          const int s = (int)(g % NS);
          mbar_wait(&full[s], (unsigned)((g / NS) & 1));
          const double* seg = ring + (int64_t)s * K;
          double d = 0.0;
          for (int r = 2 * lane; r < len; r += 64) {
            const double2 x = *reinterpret_cast<const double2*>(seg + r);
            const double2 vv = *reinterpret_cast<const double2*>(v + i0 + r);
            d += x.x * vv.x + x.y * vv.y;
          }
          d = fl::warp_sum(d);
          const int c = i + 1 + jj;
          if (lane == 0) {
            F[k * K + c] = t * d;
            rowA[c] = seg[i - i0];
          }
          __syncwarp();
          if (lane == 0) mbar_arrive(&empty[s]);
        }
        base += ncol;
        for (int kk = wid; kk < k; kk += NCW) {
          const double* cc = A + (int64_t)(offset + kk) * K;
          double dd = 0.0;
          for (int r = i + lane; r < M; r += 32) dd += cc[r] * v[r];
          dd = fl::warp_sum(dd);
          if (lane == 0) auxv[kk] = -t * dd;
        }
        if (tid <= k) rowi[tid] = (tid == k) ? 1.0 : A[(int64_t)(offset + tid) * K + i];
      }
      csync();
      // ---- F(:, k) += F(:, 0:k) auxv; A(i, i+1:N) -= A(i, offset:i+1) F(i+1:N, 0:k+1)^T; downdate ----
      for (int c = offset + tid; c < N; c += NTC) {
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
              flag[c] = 1;
              s_flagged = 1;
            } else {
              vn1[c] *= sqrt(tt);
            }
          }
        }
      }
      csync();
      ++k;
    }
    if (s_stop) break;
    const int kb = k;
    const int rk = offset + kb;
    // ---- block update: A(rk:M, rk:N) -= A(rk:M, offset:rk) F(rk:N, 0:kb)^T  (DMMA) ----
    if (rk < M && rk < N) {
      const int g = lane >> 2, t4 = lane & 3;
      const int nrt = (M - rk + 7) / 8, nct = (N - rk + 7) / 8;
      for (int rt = wid; rt < nrt; rt += NCW) {
        const int row = rk + rt * 8 + g;
        const bool rok = row < M;
        double av[PB / 4];
#pragma unroll
        for (int s = 0; s < PB / 4; ++s) {
          const int kk = 4 * s + t4;
          av[s] = (rok && kk < kb) ? -A[(int64_t)(offset + kk) * K + row] : 0.0;
        }
        auto ld = [&](int ct, double& x0, double& x1) {
          const int c0 = rk + ct * 8 + 2 * t4;
          x0 = (rok && c0 < N) ? A[(int64_t)c0 * K + row] : 0.0;
          x1 = (rok && c0 + 1 < N) ? A[(int64_t)(c0 + 1) * K + row] : 0.0;
        };
        double d0, d1;
        ld(0, d0, d1);
        for (int ct = 0; ct < nct; ++ct) {
          double n0 = 0.0, n1 = 0.0;
          if (ct + 1 < nct) ld(ct + 1, n0, n1);
          const int cb = rk + ct * 8 + g;
#pragma unroll
          for (int s = 0; s < PB / 4; ++s) {
            const int kk = 4 * s + t4;
            const double bv = (cb < N && kk < kb) ? F[kk * K + cb] : 0.0;
            fl::dmma(d0, d1, av[s], bv);
          }
          const int c0 = rk + ct * 8 + 2 * t4;
          if (rok && c0 < N) A[(int64_t)c0 * K + row] = d0;
          if (rok && c0 + 1 < N) A[(int64_t)(c0 + 1) * K + row] = d1;
          d0 = n0;
          d1 = n1;
        }
      }
    }
    asm volatile("fence.proxy.async.global;\n" ::: "memory");
    csync();
    // ---- recompute flagged norms over rows rk..M-1 ----
    for (int c = rk + wid; c < N; c += NCW) {
      if (!flag[c]) continue;
      double s2 = 0.0;
      for (int r = rk + lane; r < M; r += 32) s2 += A[(int64_t)c * K + r] * A[(int64_t)c * K + r];
      s2 = fl::warp_sum(s2);
      if (lane == 0) {
        vn1[c] = vn2[c] = (rk < M) ? sqrt(s2) : 0.0;
        flag[c] = 0;
      }
    }
    __threadfence_block();
    csync();
    offset = rk;
  }
  // stop the producer (it is waiting for the next step)
  if (tid == 0) {
    s_step = -1;
    mbar_arrive(&go);
  }
  csync();
  const int rank = s_rank;
  for (int c = tid; c < K; c += NTC) {
    q.perm[(int64_t)j * K + c] = piv[c];
    q.diag[(int64_t)j * K + c] = (c < rank && lead > 0.0) ? q.diag[(int64_t)j * K + c] / lead : 0.0;
  }
  if (tid == 0) q.rank[j] = rank;
  (void)gostep;
}

}  // namespace

namespace fl {
bool qrcp2_ok(int K) {
  const size_t smem = (size_t)((NS + PB + 4) * K) * sizeof(double) + (size_t)2 * K * sizeof(int);
  return K % 2 == 0 && smem <= (MINB > 1 ? 112 : 220) * 1024;
}
int qrcp2_r0(double* R0, int K, const int32_t* kmax, int J, double sigma, double* tau, int32_t* perm,
             int32_t* rank, double* diag, cudaStream_t s) {
  const size_t smem = (size_t)((NS + PB + 4) * K) * sizeof(double) + (size_t)2 * K * sizeof(int);
  if (!qrcp2_ok(K)) return FL_ERR_INVALID;
  FL_CUDA(cudaFuncSetAttribute(qrcp2_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  QrcpArgs a{R0, K, kmax, sigma, tau, perm, rank, diag};
  qrcp2_kernel<<<J, NT, smem, s>>>(a);
  FL_CHECK_LAUNCH();
  return FL_OK;
}
}  // namespace fl
