// K2a panel factorisation: unpivoted Householder QR of one 32-column panel
// of every block (LAPACK dgeqr2 + dlarft semantics), batched one CTA per
// block. The panel rows P0..m-1 are factored in inner panels of 8 columns,
// staged in shared memory when their rows fit (<= 2944), else in place in
// the block.
// Each inner panel is factored on chip, then applied to the rest of the
// 32-column panel in compact-WY form as two streaming DMMA passes over those
// columns (P = V^T X, then X -= V (Tw^T P)) with 256-bit accesses, several
// 16-row chunks in flight per warp. Finally the panel's T factor (32 x 32,
// upper triangular) is built from the Gram matrix V^T V, streamed the same
// way (the loaded fragment of an 8-column group is both the A and the B
// operand of its tiles), and the dlarft recurrence runs on one warp with the
// rows of T in registers.
//
// Reflector convention (dlarfg): beta = -sign(alpha) hypot(alpha, ||x||),
// tau = (beta - alpha) / beta, v = [1; x / (alpha - beta)], R_ii = beta.
#include <stdio.h>

#include "wy.cuh"

namespace {

constexpr int NB = 32;
// measured on cfg4 (round-1 kernel): 512 threads 2.11 ms per launch, 384
// threads (160 registers) 2.34 ms
constexpr int NT = 512;
constexpr int NW = NT / 32;
// (measured on cfg4: 184 KB 2.09 ms per launch, 164 KB 2.14, 132 KB (W = 4) 2.50)
constexpr int SMEM_S = 184 * 1024;  // bytes for the inner-panel columns (+ ~31 KB static)
// (measured: 256 threads at two CTAs per SM, 84 KB panels, was slower: 2.80 vs 2.25 ms per launch)

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
__device__ void factor_inner(double* S, int Mq, int64_t sq, double* red, double* sc, double* Tw, double* tau_j,
                             int col0) {
  // S: W columns of Mq rows (column-major, stride sq: shared memory, or the
  // block itself in place for blocks too tall to stage), rows relative to col0.
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
    const double x = S[s1 * sq + r];
    acc[0] += x * x;
#pragma unroll
    for (int k = 0; k < W; ++k) {
      if (k > s1) acc[k] += x * S[k * sq + r];
      if (k < s1) acc[W + k] += x * S[k * sq + r];  // reflector k (r > s1 > k: stored)
    }
  };
  auto stash = [&](int s1) {  // row s1 of every column, by its owner
#pragma unroll
    for (int k = 0; k < W; ++k) rowb[s1 & 1][k] = S[k * sq + s1];
  };
#pragma unroll
  for (int k = 0; k < 2 * W; ++k) acc[k] = 0.0;
  for (int r = threadIdx.x; r < Mq; r += NT) {
    if (r > 0) accumulate(0, r);
    else stash(0);
  }
#pragma unroll
  for (int s = 0; s < W; ++s) {  // unrolled: the row registers below are indexed statically
    block_sums<2 * W>(acc, red, sc);
    const double* rb = rowb[s & 1];
    const double alpha = rb[s];
    const double ss = sc[0];
    double beta, t, scal;
    if (ss == 0.0) {
      t = 0.0;
      beta = alpha;
      scal = 1.0;
    } else {
      // ||(alpha, x)|| from the sum of squares directly (one sqrt on the
      // step's critical path); hypot only where the squares leave the safe range
      const double n2 = fma(alpha, alpha, ss);
      const double nrm = (n2 > 1e-280 && n2 < 1e280 && ss > 1e-280) ? sqrt(n2) : hypot(alpha, sqrt(ss));
      beta = -copysign(nrm, alpha);
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
    // the row's values are read once into registers, updated, stored, and
    // the next column's sums are formed from the registers
#pragma unroll 2
    for (int r = threadIdx.x; r < Mq; r += NT) {
      if (r < s) continue;
      double x[W];  // row r: reflector entries (k < s), then columns s..W-1
#pragma unroll
      for (int k = 0; k < W; ++k) x[k] = S[k * sq + r];
      double v = 1.0;
      if (r == s) {
        S[s * sq + s] = beta;
      } else {
        v = x[s] * scal;
        S[s * sq + r] = v;
      }
#pragma unroll
      for (int k = 0; k < W; ++k) {
        if (k > s) {
          if (t != 0.0) x[k] = fma(-pk[k], v, x[k]);
          S[k * sq + r] = x[k];
        } else if (k == s) {
          x[k] = v;
        }
      }
      if (s + 1 < W) {
        if (r > s + 1) {
          double xx = 0.0;
#pragma unroll
          for (int k = 0; k < W; ++k)
            if (k == s + 1) xx = x[k];
          acc[0] += xx * xx;
#pragma unroll
          for (int k = 0; k < W; ++k) {
            if (k > s + 1) acc[k] += xx * x[k];
            if (k < s + 1) acc[W + k] += xx * x[k];  // reflector k (r > s + 1 > k)
          }
        } else if (r == s + 1) {  // row s + 1 of every column, by its owner
#pragma unroll
          for (int k = 0; k < W; ++k) rowb[(s + 1) & 1][k] = x[k];
        }
      }
    }
  }
  __syncthreads();
}

// entry (r, k) of the resident inner panel's V: unit lower trapezoidal, W
// columns of Mq rows in S (stride sq); zero outside
template <int W>
__device__ __forceinline__ double vval(const double* S, int64_t sq, int Mq, int r, int k) {
  return (k >= W || r >= Mq || r < k) ? 0.0 : (r == k ? 1.0 : S[k * sq + r]);
}

// X -= V (Tw^T (V^T X)) for the nrest (<= 8 NT8) panel columns X right of the
// resident inner panel (columns c + W.. of Xj, rows c..c+Mq-1; written to
// Aj), as two streaming passes with mma.sync m8n8k4 over 16-row chunks. A
// lane's 256-bit access is rows r0 + 4 t4 .. + 3 of its column (a warp
// access covers one full line per column):
//   pass 1  P(k, u) += V(r, k) X(r, u)   m = k, n = u, reduction over rows:
//           the four MMA k-steps take the four loaded rows in turn
//   pass 2  X(r, u) -= V(r, k) Z(k, u)   m = u, n = r: two MMA tiles whose
//           accumulator pairs are the loaded rows (0, 1) and (2, 3), i.e.
//           tile h holds rows r0 + 4 (n / 2) + 2 h + n % 2
// Each warp owns UN consecutive chunks per trip with all their loads in
// flight; the W x nrest partial sums of the warps are added in warp order.
#ifdef PANEL_PHASES
__shared__ long long g_dbg[4];
#define APH(n, t0) do { if (threadIdx.x == 0) { const long long t_ = clock64(); g_dbg[n] += t_ - t0; t0 = t_; } } while (0)
#else
#define APH(n, t0)
#endif

// 256-bit loads in flight per lane and trip (measured on cfg4, 16-byte loads:
// 8 / 12 / 16 / 18 in flight 1.25 / 1.26 / 1.29 / 1.31 ms per launch)
constexpr int PANEL_LD = 6;

template <int W, int NT8>
__device__ void apply_rest(const double* S, int64_t sq, int Mq, const double* Tw, const double* Xj, double* Aj, int64_t ld, int c,
                           int nrest, double* Pw, double* Zs) {
  constexpr int UN = PANEL_LD / NT8 > 0 ? PANEL_LD / NT8 : 1;  // ~PANEL_LD 256-bit loads in flight per lane
  constexpr int PC = 8 * NT8;                                  // padded column count
  constexpr int KS = (W + 3) / 4;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, g = lane >> 2, t4 = lane & 3;
  // chunks start at the 4-row boundary at or above row c (W = 2: c may be
  // 2 mod 4); rows above c (r < 0) meet V = 0 and are stored back unchanged
  const int rsh = W >= 4 ? 0 : (c & 3);
  const int nch = (Mq + rsh + 15) / 16;
  const int x0 = c + W;
  const double* xcol[NT8];
  bool cok[NT8];
#pragma unroll
  for (int t = 0; t < NT8; ++t) {
    cok[t] = 8 * t + g < nrest;
    xcol[t] = Xj + (int64_t)(x0 + (cok[t] ? 8 * t + g : 0)) * ld + (c - rsh) + 4 * t4;
  }
  auto load_chunks = [&](int ch0, fl::d4 (&x)[UN][NT8]) {
#pragma unroll
    for (int u = 0; u < UN; ++u) {
      const int r = (ch0 + u) * 16 + 4 * t4 - rsh;
#pragma unroll
      for (int t = 0; t < NT8; ++t) {
        fl::d4 v{0.0, 0.0, 0.0, 0.0};
        if (r < Mq && cok[t]) v = fl::ldg256(xcol[t] + (ch0 + u) * 16);
        if (r + 1 >= Mq) v.b = 0.0;
        if (r + 2 >= Mq) v.c = 0.0;
        if (r + 3 >= Mq) v.d = 0.0;
        x[u][t] = v;
      }
    }
  };
#ifdef PANEL_PHASES
  long long tph = clock64();
#endif
  // ---- pass 1 ----
  {
    double acc[NT8][2];
#pragma unroll
    for (int t = 0; t < NT8; ++t) acc[t][0] = acc[t][1] = 0.0;
    for (int ch0 = wid * UN; ch0 < nch; ch0 += NW * UN) {
      fl::d4 x[UN][NT8];
      load_chunks(ch0, x);
#pragma unroll
      for (int u = 0; u < UN; ++u) {
        const int r = (ch0 + u) * 16 + 4 * t4 - rsh;
        const double v0 = vval<W>(S, sq, Mq, r, g), v1 = vval<W>(S, sq, Mq, r + 1, g);
        const double v2 = vval<W>(S, sq, Mq, r + 2, g), v3 = vval<W>(S, sq, Mq, r + 3, g);
#pragma unroll
        for (int t = 0; t < NT8; ++t) {
          fl::dmma(acc[t][0], acc[t][1], v0, x[u][t].a);
          fl::dmma(acc[t][0], acc[t][1], v1, x[u][t].b);
          fl::dmma(acc[t][0], acc[t][1], v2, x[u][t].c);
          fl::dmma(acc[t][0], acc[t][1], v3, x[u][t].d);
        }
      }
    }
    if (g < W) {
#pragma unroll
      for (int t = 0; t < NT8; ++t) {
        Pw[(wid * W + g) * PC + 8 * t + 2 * t4] = acc[t][0];
        Pw[(wid * W + g) * PC + 8 * t + 2 * t4 + 1] = acc[t][1];
      }
    }
  }
  __syncthreads();
  APH(0, tph);
  // P = sum over warps (fixed order); Z = Tw^T P (Tw^T[k][b] = Tw[k * W + b], b <= k)
  for (int o = threadIdx.x; o < W * PC; o += NT) {
    double p = 0.0;
    for (int w = 0; w < NW; ++w) p += Pw[w * W * PC + o];
    Zs[o] = p;
  }
  __syncthreads();
  double az[NT8][KS];  // -Z(k = t4 + 4 s, u = 8 t + g)
#pragma unroll
  for (int t = 0; t < NT8; ++t)
#pragma unroll
    for (int s2 = 0; s2 < KS; ++s2) {
      const int k = t4 + 4 * s2;
      double z = 0.0;
      if (k < W)
        for (int b = 0; b <= k; ++b) z += Tw[k * W + b] * Zs[b * PC + 8 * t + g];
      az[t][s2] = -z;
    }
  APH(1, tph);
  // ---- pass 2 ----
  for (int ch0 = wid * UN; ch0 < nch; ch0 += NW * UN) {
    fl::d4 x[UN][NT8];
    load_chunks(ch0, x);
#pragma unroll
    for (int u = 0; u < UN; ++u) {
      const int rb = (ch0 + u) * 16 + 4 * (g >> 1) + (g & 1) - rsh;
      double vb[2][KS];
#pragma unroll
      for (int h = 0; h < 2; ++h)
#pragma unroll
        for (int s2 = 0; s2 < KS; ++s2) vb[h][s2] = vval<W>(S, sq, Mq, rb + 2 * h, t4 + 4 * s2);
      const int r = (ch0 + u) * 16 + 4 * t4 - rsh;
#pragma unroll
      for (int t = 0; t < NT8; ++t) {
#pragma unroll
        for (int s2 = 0; s2 < KS; ++s2) {
          fl::dmma(x[u][t].a, x[u][t].b, az[t][s2], vb[0][s2]);
          fl::dmma(x[u][t].c, x[u][t].d, az[t][s2], vb[1][s2]);
        }
        if (cok[t] && r < Mq) fl::stg256(Aj + (int64_t)(x0 + 8 * t + g) * ld + c + r, x[u][t]);
      }
    }
  }
  APH(2, tph);
  __syncthreads();
  APH(3, tph);
}

#ifdef PANEL_PHASES  // diagnostic build: cycles per phase (thread 0's clock)
#define PPH(n)                                 \
  do {                                         \
    if (threadIdx.x == 0) {                    \
      const long long t_ = clock64();          \
      ph_acc[n] += t_ - ph_last;               \
      ph_last = t_;                            \
    }                                          \
  } while (0)
#else
#define PPH(n)
#endif

// INPLACE: the inner panels are factored where they lie in the block (blocks
// too tall for even two staged columns): same passes, global instead of
// shared accesses, each thread re-reading only rows it wrote itself.
template <int W, bool INPLACE>
__device__ void panel_body(const PanelArgs& a, int j, double* S, double* red, double* sc, double* Tw,
                           double* Gs, double* Pw, double* Zs) {
  const int m = a.m[j];
  const int64_t ld = a.ld[j];
  double* Aj = a.A + a.off[j];
  double* tau_j = a.tau + (int64_t)j * a.K;
  const int P0 = a.P0;
#ifdef PANEL_PHASES
  long long ph_acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  long long ph_last = clock64();
  if (threadIdx.x == 0) g_dbg[0] = g_dbg[1] = g_dbg[2] = g_dbg[3] = 0;
#endif
  for (int q = 0; q < NB / W; ++q) {
    const int c = P0 + q * W;
    const int Mq = m - c;
    // columns right of the first inner panel are first read from src, later from A
    const double* Xj = (q == 0 && a.src) ? a.src + a.off[j] : Aj;
    double* Sp = INPLACE ? Aj + (int64_t)c * ld + c : S;  // the inner panel's columns, rows from c
    const int64_t sq = INPLACE ? ld : Mq;
    if (INPLACE) {
      if (Xj != Aj)
        for (int k = 0; k < W; ++k)
          for (int r = threadIdx.x; r < Mq; r += NT) Sp[k * sq + r] = Xj[(int64_t)(c + k) * ld + c + r];
    } else {
      // load inner panel rows c..m-1 (8-byte cp.async: every load in flight at once)
      for (int k = 0; k < W; ++k)
#pragma unroll 2
        for (int r = threadIdx.x; r < Mq; r += NT) {
          const unsigned dst = (unsigned)__cvta_generic_to_shared(S + k * Mq + r);
          asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(dst), "l"(Xj + (int64_t)(c + k) * ld + c + r)
                       : "memory");
        }
      asm volatile("cp.async.wait_all;\n" ::: "memory");
    }
    __syncthreads();
    PPH(0);
    factor_inner<W>(Sp, Mq, sq, red, sc, Tw, tau_j, c);
    PPH(1);
    if (!INPLACE)
      for (int k = 0; k < W; ++k)
        for (int r = threadIdx.x; r < Mq; r += NT) Aj[(int64_t)(c + k) * ld + c + r] = S[k * Mq + r];
    PPH(2);
    // apply (I - V Tw V^T)^T to the panel columns right of this inner panel
    {
      const int nrest = P0 + NB - (c + W);
      const int nt8 = (nrest + 7) / 8;
      if (nt8 == 4) apply_rest<W, 4>(Sp, sq, Mq, Tw, Xj, Aj, ld, c, nrest, Pw, Zs);
      else if (nt8 == 3) apply_rest<W, 3>(Sp, sq, Mq, Tw, Xj, Aj, ld, c, nrest, Pw, Zs);
      else if (nt8 == 2) apply_rest<W, 2>(Sp, sq, Mq, Tw, Xj, Aj, ld, c, nrest, Pw, Zs);
      else if (nt8 == 1) apply_rest<W, 1>(Sp, sq, Mq, Tw, Xj, Aj, ld, c, nrest, Pw, Zs);
      PPH(4);
    }
  }
  // ---- T for the 32-column panel from G = V^T V, streamed with DMMA ----
  __syncthreads();  // every inner panel written back; S is reused for the warps' partial tiles
  const int M = m - P0;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, g = lane >> 2, t4 = lane & 3;
  {
    // a lane loads rows r0 + 4 t4 .. + 3 of columns 8 c4 + g (c4 = 0..3):
    // that fragment is the A operand of the tiles (c4, *) and the B operand
    // of the tiles (*, c4); the 10 upper tiles (ta <= tb) are accumulated
    const int nch = (M + 15) / 16;
    double acc[10][2];
#pragma unroll
    for (int t = 0; t < 10; ++t) acc[t][0] = acc[t][1] = 0.0;
    const double* vcol = Aj + (int64_t)(P0 + g) * ld + P0 + 4 * t4;
    for (int ch = w; ch < nch; ch += NW) {
      const int r = ch * 16 + 4 * t4;
      fl::d4 x[4];
#pragma unroll
      for (int c4 = 0; c4 < 4; ++c4)
        x[c4] = (r < M) ? fl::ldg256(vcol + (int64_t)(8 * c4) * ld + ch * 16) : fl::d4{0.0, 0.0, 0.0, 0.0};
      if (ch * 16 < NB || ch * 16 + 16 > M) {  // unit diagonal, zeros above it and past row M
        auto fix = [&](double& v, int row, int col) {
          if (row >= M || row < col) v = 0.0;
          else if (row == col) v = 1.0;
        };
#pragma unroll
        for (int c4 = 0; c4 < 4; ++c4) {
          const int col = 8 * c4 + g;
          fix(x[c4].a, r, col);
          fix(x[c4].b, r + 1, col);
          fix(x[c4].c, r + 2, col);
          fix(x[c4].d, r + 3, col);
        }
      }
      int t = 0;
#pragma unroll
      for (int ta = 0; ta < 4; ++ta)
#pragma unroll
        for (int tb = ta; tb < 4; ++tb) {
          fl::dmma(acc[t][0], acc[t][1], x[ta].a, x[tb].a);
          fl::dmma(acc[t][0], acc[t][1], x[ta].b, x[tb].b);
          fl::dmma(acc[t][0], acc[t][1], x[ta].c, x[tb].c);
          fl::dmma(acc[t][0], acc[t][1], x[ta].d, x[tb].d);
          ++t;
        }
    }
    double* Pg = S;  // (NW, 10, 64)
#pragma unroll
    for (int t = 0; t < 10; ++t) {
      Pg[(w * 10 + t) * 64 + g * 8 + 2 * t4] = acc[t][0];
      Pg[(w * 10 + t) * 64 + g * 8 + 2 * t4 + 1] = acc[t][1];
    }
    __syncthreads();
    for (int o = threadIdx.x; o < 640; o += NT) {
      const int t = o / 64, i = (o % 64) / 8, jj = o % 8;
      int ta = 0, tb = 0, cnt = 0;
      for (int x2 = 0; x2 < 4; ++x2)
        for (int y2 = x2; y2 < 4; ++y2) {
          if (cnt == t) {
            ta = x2;
            tb = y2;
          }
          ++cnt;
        }
      double sum = 0.0;
      for (int ww = 0; ww < NW; ++ww) sum += Pg[(ww * 10 + t) * 64 + i * 8 + jj];
      Gs[(ta * 8 + i) * NB + tb * 8 + jj] = sum;
    }
  }
  __syncthreads();
  PPH(5);
  if (w == 0) {
    // dlarft (forward, columnwise): T[i][i] = tau_i; T[0:i, i] = -tau_i T[0:i, 0:i] G[0:i, i].
    // Lane a keeps row a of T in registers (zero left of the diagonal).
    double* Tp = a.T + ((int64_t)j * (a.K / NB) + P0 / NB) * NB * NB;
    const double tl = tau_j[P0 + lane];
    double Tr[NB];
#pragma unroll
    for (int i = 0; i < NB; ++i) {
      const double ti = __shfl_sync(0xffffffffu, tl, i);
      double z0 = 0.0, z1 = 0.0;
#pragma unroll
      for (int b = 0; b < i; ++b) {
        if (b & 1) z1 = fma(Tr[b], Gs[b * NB + i], z1);
        else z0 = fma(Tr[b], Gs[b * NB + i], z0);
      }
      Tr[i] = (lane < i) ? -ti * (z0 + z1) : (lane == i ? ti : 0.0);
      Tp[i * NB + lane] = Tr[i];
    }
  }
#ifdef PANEL_PHASES
  PPH(6);
  if (threadIdx.x == 0 && (j % 256) == 5)
    printf("PANELPH j=%d P0=%d W=%d M=%d load=%lld factor=%lld wb=%lld groups=%lld (pass1=%lld reduce=%lld pass2=%lld tail=%lld) gram=%lld tbuild=%lld\n", j, P0,
           W, m - P0, ph_acc[0], ph_acc[1], ph_acc[2], ph_acc[4], g_dbg[0], g_dbg[1], g_dbg[2], g_dbg[3], ph_acc[5], ph_acc[6]);
#endif
}

__global__ void __launch_bounds__(NT, 1) panel_kernel(PanelArgs a) {
  extern __shared__ double sm[];
  double* S = sm;                                   // SMEM_S bytes
  __shared__ double red[NW * 32];
  __shared__ double sc[64];
  __shared__ double Tw[64];
  __shared__ double Pw[NW * 8 * 24];  // apply_rest's per-warp partial sums; G of the finished panel
  __shared__ double Zs[256];
  double* Gs = Pw;
  const int j = blockIdx.x;
  const int M = a.m[j] - a.P0;
  if (M <= 0) return;
  const int cap = SMEM_S / 8;
  // blocks whose 8-column inner panels do not fit in shared memory (more than
  // FL_RRQR_BLOCKED_MAX_ROWS rows from this panel on) are factored in place;
  // measured at cfg5 (4096 to 5832 rows): in place 1.30 ms per launch,
  // 4-column staged inner panels 1.35
  if (8 * M <= cap) panel_body<8, false>(a, j, S, red, sc, Tw, Gs, Pw, Zs);
  else panel_body<8, true>(a, j, S, red, sc, Tw, Gs, Pw, Zs);
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
