// K2a panel factorisation: unpivoted Householder QR of one 32-column panel
// of every block (LAPACK dgeqr2 + dlarft semantics), batched one CTA per
// block. The panel rows P0..m-1 are factored in inner panels of w columns
// (w = 8, 4 or 2, the widest whose rows fit in shared memory); each inner
// panel is factored entirely in shared memory, then applied to the rest of
// the 32-column panel in compact-WY form, 4 columns at a time. Finally the
// panel's T factor (32 x 32, upper triangular) is built from the Gram matrix
// V^T V, computed with DMMA over shared-memory-staged row chunks.
//
// Reflector convention (dlarfg): beta = -sign(alpha) hypot(alpha, ||x||),
// tau = (beta - alpha) / beta, v = [1; x / (alpha - beta)], R_ii = beta.
#include "wy.cuh"

namespace {

constexpr int NB = 32;
#ifndef PANEL_NT
// measured on cfg4: 512 threads 2.11 ms per launch, 384 threads (160
// registers) 2.34 ms
#define PANEL_NT 512
#endif
constexpr int NT = PANEL_NT;
constexpr int NW = NT / 32;
// (measured on cfg4: 184 KB 2.09 ms per launch, 164 KB 2.14, 132 KB (W = 4) 2.50)
#ifndef PANEL_SMEM_KB
#define PANEL_SMEM_KB 184
#endif
constexpr int SMEM_S = PANEL_SMEM_KB * 1024;  // bytes for the inner-panel columns (+ ~14 KB static)
// (measured: 256 threads at two CTAs per SM, 84 KB panels, was slower: 2.80 vs 2.25 ms per launch)
constexpr int GC = (NB * 64) % NT == 0 ? 64 : 48;  // Gram pass row chunk (NB * GC divisible by NT)
constexpr int GLD = GC + 4;

// Sum N (a power of two <= 32) per-thread partials across the CTA; results
// in out[0..N). Within a warp a butterfly halves the live values per lane at
// each of the first log2(N) steps (N - 1 shuffles instead of 5 N), then the
// remaining steps sum the single value; lane (32 / N) c ends with value c.
template <int N>
__device__ __forceinline__ void block_sums(const double (&part)[N], double* red, double* out) {
  static_assert(N >= 1 && N <= 32 && (N & (N - 1)) == 0, "power of two <= 32");
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  double v[N];
#pragma unroll
  for (int c = 0; c < N; ++c) v[c] = part[c];
#pragma unroll
  for (int half = N / 2, o = 16; half >= 1; half /= 2, o /= 2) {
    const bool up = (lane & o) != 0;
#pragma unroll
    for (int c = 0; c < half; ++c) {
      const double send = up ? v[c] : v[c + half];
      const double recv = __shfl_xor_sync(0xffffffffu, send, o);
      v[c] = (up ? v[c + half] : v[c]) + recv;
    }
  }
  double sv = v[0];
#pragma unroll
  for (int o = 32 / N / 2; o > 0; o >>= 1) sv += __shfl_xor_sync(0xffffffffu, sv, o);
  if ((lane & (32 / N - 1)) == 0) red[wid * 32 + lane / (32 / N)] = sv;
  __syncthreads();
  if (threadIdx.x < N) {
    double s = 0.0;
    for (int w = 0; w < NW; ++w) s += red[w * 32 + threadIdx.x];
    out[threadIdx.x] = s;
  }
  __syncthreads();
}

struct PanelArgs {
  double* A;
  const int64_t* off;
  const int32_t* ld;
  const int32_t* m;
  int K;
  int P0;
  double* tau;     // (J, K)
  double* T;       // (J, K/NB, NB, NB) column-major per panel
  const double* src;  // null, or the store the panel's columns are read from (same layout; the
                      // first inner panel reads it and writes A, so A needs no prior copy)
};

template <int W>
__device__ void factor_inner(double* S, int Mq, double* red, double* sc, double* Tw, double* tau_j, int col0) {
  // S: W columns of Mq rows (column-major, stride Mq), rows relative to col0.
  // One pass over the rows per column: the pass that applies H_s to the
  // columns right of s also accumulates, for column s+1, its squared norm
  // and its UNSCALED dots x^T S[k] with the columns right of it and with the
  // earlier reflectors (rows > s+1). After one CTA reduction every thread
  // forms dlarfg's beta, tau and scal = 1 / (alpha - beta) itself, and the
  // dots of the scaled reflector as S[k][s+1] + scal * dot (the row-(s+1)
  // term, v = 1, stashed by the row's owner). Rows are owned by thread
  // r mod NT throughout, so each pass only reads values its own thread wrote.
  __shared__ double rowb[2][W];
  double acc[2 * W];
  auto accumulate = [&](int s1, int r) {  // rows r > s1 of column s1 (updated)
    const double x = S[s1 * Mq + r];
    acc[0] += x * x;
#pragma unroll
    for (int k = 0; k < W; ++k) {
      if (k > s1) acc[k] += x * S[k * Mq + r];
      if (k < s1) acc[W + k] += x * S[k * Mq + r];  // reflector k (r > s1 > k: stored)
    }
  };
  auto stash = [&](int s1) {  // row s1 of every column, by its owner
#pragma unroll
    for (int k = 0; k < W; ++k) rowb[s1 & 1][k] = S[k * Mq + s1];
  };
#pragma unroll
  for (int k = 0; k < 2 * W; ++k) acc[k] = 0.0;
  for (int r = threadIdx.x; r < Mq; r += NT) {
    if (r > 0) accumulate(0, r);
    else stash(0);
  }
  for (int s = 0; s < W; ++s) {
    block_sums<2 * W>(acc, red, sc);
    const double* rb = rowb[s & 1];
    const double alpha = rb[s];
    const double xnorm = sqrt(sc[0]);
    double beta, t, scal;
    if (xnorm == 0.0) {
      t = 0.0;
      beta = alpha;
      scal = 1.0;
    } else {
      beta = -copysign(hypot(alpha, xnorm), alpha);
      t = (beta - alpha) / beta;
      scal = 1.0 / (alpha - beta);
    }
    double pk[W];  // t * v_s^T S[k] for k > s
#pragma unroll
    for (int k = 0; k < W; ++k) pk[k] = (k > s) ? t * (rb[k] + scal * sc[k]) : 0.0;
    // T column s (dlarft forward, columnwise): T[0:s, s] = -t T[0:s,0:s] (V_prev^T v_s)
    if (threadIdx.x < s) {
      const int a = threadIdx.x;
      double z = 0.0;
      for (int b = a; b < s; ++b) z += Tw[b * W + a] * (rb[b] + scal * sc[W + b]);
      Tw[s * W + a] = -t * z;
    }
    if (threadIdx.x == 0) {
      tau_j[col0 + s] = t;
      Tw[s * W + s] = t;
    }
#pragma unroll
    for (int k = 0; k < 2 * W; ++k) acc[k] = 0.0;
    for (int r = threadIdx.x; r < Mq; r += NT) {
      if (r < s) continue;
      double v = 1.0;
      if (r == s) {
        S[s * Mq + s] = beta;
      } else {
        v = S[s * Mq + r] * scal;
        S[s * Mq + r] = v;
      }
      if (t != 0.0) {
#pragma unroll
        for (int k = 0; k < W; ++k)
          if (k > s) S[k * Mq + r] -= pk[k] * v;
      }
      if (s + 1 < W) {
        if (r > s + 1) accumulate(s + 1, r);
        else if (r == s + 1) stash(s + 1);
      }
    }
  }
  __syncthreads();
}

template <int W>
__device__ void panel_body(const PanelArgs& a, int j, double* S, double* red, double* sc, double* Tw,
                           double* Vs, double* Gs) {
  const int m = a.m[j];
  const int64_t ld = a.ld[j];
  double* Aj = a.A + a.off[j];
  double* tau_j = a.tau + (int64_t)j * a.K;
  const int P0 = a.P0;
  for (int q = 0; q < NB / W; ++q) {
    const int c = P0 + q * W;
    const int Mq = m - c;
    // columns right of the first inner panel are first read from src, later from A
    const double* Xj = (q == 0 && a.src) ? a.src + a.off[j] : Aj;
    // load inner panel rows c..m-1 (8-byte cp.async: every load in flight at once)
    for (int k = 0; k < W; ++k)
#pragma unroll 2
      for (int r = threadIdx.x; r < Mq; r += NT) {
        const unsigned dst = (unsigned)__cvta_generic_to_shared(S + k * Mq + r);
        asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(dst), "l"(Xj + (int64_t)(c + k) * ld + c + r)
                     : "memory");
      }
    asm volatile("cp.async.wait_all;\n" ::: "memory");
    __syncthreads();
    factor_inner<W>(S, Mq, red, sc, Tw, tau_j, c);
    for (int k = 0; k < W; ++k)
      for (int r = threadIdx.x; r < Mq; r += NT) Aj[(int64_t)(c + k) * ld + c + r] = S[k * Mq + r];
    // apply (I - V Tw V^T)^T to the panel columns right of this inner panel,
    // 4 at a time: one pass per group updates group g (with z(g) = Tw^T
    // V^T x(g)) and forms the dots V^T x(g+1) of the next group from the same
    // rows (thread r mod NT throughout), so the groups cost one pass and one
    // reduction each instead of two passes
    {
      const int ng = (P0 + NB - (c + W)) / 4;
      __shared__ double z[2][4 * 8];
      auto vvals = [&](int r, double (&vv)[W]) {
#pragma unroll
        for (int k = 0; k < W; ++k) vv[k] = (r < k) ? 0.0 : ((r == k) ? 1.0 : S[k * Mq + r]);
      };
      auto finish = [&](double (&p)[4 * W], int buf) {  // z(buf) = Tw^T (V^T x)
        block_sums<4 * W>(p, red, sc);
        if (threadIdx.x < 4 * W) {
          const int k = threadIdx.x / 4, u = threadIdx.x % 4;
          double s2 = 0.0;
          for (int b = 0; b <= k; ++b) s2 += Tw[k * W + b] * sc[b * 4 + u];  // Tw^T[k][b] = Tw[b][k]
          z[buf][k * 4 + u] = s2;
        }
        __syncthreads();
      };
      if (ng > 0) {
        double p[4 * W];
#pragma unroll
        for (int k = 0; k < 4 * W; ++k) p[k] = 0.0;
        const int x0 = c + W;
#pragma unroll 2
        for (int r = threadIdx.x; r < Mq; r += NT) {
          double vv[W], xv[4];
          vvals(r, vv);
#pragma unroll
          for (int u = 0; u < 4; ++u) xv[u] = Xj[(int64_t)(x0 + u) * ld + c + r];
#pragma unroll
          for (int k = 0; k < W; ++k)
#pragma unroll
            for (int u = 0; u < 4; ++u) p[k * 4 + u] += vv[k] * xv[u];
        }
        finish(p, 0);
      }
      for (int gi = 0; gi < ng; ++gi) {
        const int x0 = c + W + 4 * gi;
        const bool nxt = gi + 1 < ng;
        const volatile double* zg = z[gi & 1];  // re-read per row (hoisted it would pin 4W registers)
        double p[4 * W];
#pragma unroll
        for (int k = 0; k < 4 * W; ++k) p[k] = 0.0;
#pragma unroll 1
        for (int r = threadIdx.x; r < Mq; r += NT) {
          double vv[W], xn[4];
          vvals(r, vv);
#pragma unroll
          for (int u = 0; u < 4; ++u) xn[u] = nxt ? Xj[(int64_t)(x0 + 4 + u) * ld + c + r] : 0.0;
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            double s2 = 0.0;
#pragma unroll
            for (int k = 0; k < W; ++k) s2 += vv[k] * zg[k * 4 + u];
            Aj[(int64_t)(x0 + u) * ld + c + r] = Xj[(int64_t)(x0 + u) * ld + c + r] - s2;
          }
          if (nxt) {
#pragma unroll
            for (int k = 0; k < W; ++k)
#pragma unroll
              for (int u = 0; u < 4; ++u) p[k * 4 + u] += vv[k] * xn[u];
          }
        }
        if (nxt) finish(p, (gi + 1) & 1);
        else __syncthreads();
      }
    }
  }
  // ---- T for the 32-column panel from G = V^T V (DMMA over staged chunks) ----
  __syncthreads();  // every inner panel written back; S is reused as the staging buffer
  const int M = m - P0;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, g = lane >> 2, t4 = lane & 3;
  // upper-triangular 8x8 tiles (ta <= tb): 10 tiles, tile w and (with fewer
  // than 10 warps) tile w + NW per warp
  constexpr int NTW = (10 + NW - 1) / NW;
  int ta[NTW], tb[NTW];
#pragma unroll
  for (int q = 0; q < NTW; ++q) {
    ta[q] = tb[q] = -1;
    int idx = w + q * NW, cnt = 0;
    for (int x = 0; x < 4; ++x)
      for (int y = x; y < 4; ++y) {
        if (cnt == idx) {
          ta[q] = x;
          tb[q] = y;
        }
        ++cnt;
      }
  }
  double acc[NTW][2];
#pragma unroll
  for (int q = 0; q < NTW; ++q) acc[q][0] = acc[q][1] = 0.0;
  // the next chunk's V values are loaded into registers while this one is
  // multiplied (one round trip per chunk overlapped instead of exposed)
  constexpr int PER = NB * GC / NT;
  static_assert(PER * NT == NB * GC, "chunk must split evenly over the CTA");
  double nx[PER];
  auto fetch = [&](int r0) {
#pragma unroll
    for (int q = 0; q < PER; ++q) {
      const int p = threadIdx.x + q * NT, col = p / GC, rr = p % GC, row = r0 + rr;
      double v = 0.0;
      if (row < M) {
        if (row > col) v = Aj[(int64_t)(P0 + col) * ld + P0 + row];
        else if (row == col) v = 1.0;
      }
      nx[q] = v;
    }
  };
  fetch(0);
  for (int r0 = 0; r0 < M; r0 += GC) {
#pragma unroll
    for (int q = 0; q < PER; ++q) {
      const int p = threadIdx.x + q * NT;
      Vs[(p / GC) * GLD + p % GC] = nx[q];
    }
    if (r0 + GC < M) fetch(r0 + GC);
    __syncthreads();
#pragma unroll
    for (int q = 0; q < NTW; ++q) {
      if (ta[q] >= 0) {
#pragma unroll 4
        for (int k0 = 0; k0 < GC; k0 += 4)
          fl::dmma(acc[q][0], acc[q][1], Vs[(ta[q] * 8 + g) * GLD + k0 + t4], Vs[(tb[q] * 8 + g) * GLD + k0 + t4]);
      }
    }
    __syncthreads();
  }
#pragma unroll
  for (int q = 0; q < NTW; ++q) {
    if (ta[q] >= 0) {
      Gs[(ta[q] * 8 + g) * NB + tb[q] * 8 + 2 * t4] = acc[q][0];
      Gs[(ta[q] * 8 + g) * NB + tb[q] * 8 + 2 * t4 + 1] = acc[q][1];
    }
  }
  __syncthreads();
  if (w == 0) {
    // T (column-major) : T[i][i] = tau_i; T[0:i,i] = -tau_i T[0:i,0:i] G[0:i,i]
    double* Tp = a.T + ((int64_t)j * (a.K / NB) + P0 / NB) * NB * NB;
    double* Tl = S;  // the staging buffer is free once G is formed
    for (int i = 0; i < NB; ++i) {
      const double ti = tau_j[P0 + i];
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

__global__ void __launch_bounds__(NT, 1) panel_kernel(PanelArgs a) {
  extern __shared__ double sm[];
  double* S = sm;                                   // SMEM_S bytes
  double* Vs = sm;                                  // reuses S for the Gram pass
  __shared__ double red[NW * 32];
  __shared__ double sc[64];
  __shared__ double Tw[64];
  __shared__ double Gs[NB * NB];
  const int j = blockIdx.x;
  const int M = a.m[j] - a.P0;
  if (M <= 0) return;
  const int cap = SMEM_S / 8;
  if (8 * M <= cap) panel_body<8>(a, j, S, red, sc, Tw, Vs, Gs);
  else if (4 * M <= cap) panel_body<4>(a, j, S, red, sc, Tw, Vs, Gs);
  else if (2 * M <= cap) panel_body<2>(a, j, S, red, sc, Tw, Vs, Gs);
  else __trap();  // excluded by rrqr_route (filtering.py BLOCKED_MAX_ROWS) and panel_factor
}

}  // namespace

namespace fl {
int panel_factor(double* A, const int64_t* off, const int32_t* ld, const int32_t* m, int J, int K, int P0,
                 double* tau, double* T, cudaStream_t s, const double* src) {
  static unsigned long long attr = 0;
  if (fl::first_on_device(attr)) {
    FL_CUDA(cudaFuncSetAttribute(panel_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_S));
  }
  PanelArgs a{A, off, ld, m, K, P0, tau, T, src};
  panel_kernel<<<J, NT, SMEM_S, s>>>(a);
  FL_CHECK_LAUNCH();
  return FL_OK;
}
}  // namespace fl
