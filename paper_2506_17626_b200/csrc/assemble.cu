// K1 — fused block assembly (reference: featlsq assembly.py:124-238).
//
// One CTA per (block j, tile of FL_ASM_TILE = 512 rows), two adjacent rows
// per thread; see assemble_kernel below for the two phases. Padding rows [m_j, ld_j)
// are written as exact zeros.
//
// Roofline: HBM write of 8 B per entry; the FP64 work per entry is one
// reciprocal plus ~15 FMA-class instructions on the tabulated path
// (DESIGN.md §3 K1).
#include "common.cuh"

namespace {

constexpr int NT = 256;
constexpr int MAXD = 3;

struct Jet {
  double v, f, s;
};

__device__ __forceinline__ Jet jmul(Jet a, Jet b) {
  // jets.py:55-63, same association as numpy's left-to-right evaluation
  Jet r;
  r.v = a.v * b.v;
  r.f = a.f * b.v + a.v * b.f;
  r.s = a.s * b.v + 2.0 * a.f * b.f + a.v * b.s;
  return r;
}

__device__ __forceinline__ Jet jrecip(Jet a) {
  // jets.py:76-80
  double iv = 1.0 / a.v;
  Jet r;
  r.v = iv;
  r.f = -a.f * iv * iv;
  r.s = (2.0 * a.f * a.f * iv - a.s) * iv * iv;
  return r;
}

__device__ __forceinline__ Jet raw_factor(double t, double mu, double half) {
  // domains.py:109-123; exactly zero (all three) outside |t - mu| < half
  Jet r{0.0, 0.0, 0.0};
  if (fabs(t - mu) < half) {
    double theta = 3.141592653589793 * (t - mu) / half;
    double s, c;
    sincos(theta, &s, &c);
    double scale = 3.141592653589793 / half;
    double opc = 1.0 + c;
    r.v = opc * opc;
    r.f = -2.0 * opc * s * scale;
    r.s = -2.0 * (c + c * c - s * s) * scale * scale;
  }
  return r;
}

// 1 / d for d in [1, 1e300]: MUFU approximation + two Newton steps (the
// relative error squares per step: full precision, <= 1 ulp; no special-case
// branches, which __drcp_rn carries)
__device__ __forceinline__ double rcp_newton(double d) {
  double y;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(d));
  double e = fma(-d, y, 1.0);
  y = fma(y, e, y);
  e = fma(-d, y, 1.0);
  return fma(y, e, y);
}
// the tabulated path's form: y0 (1 + e + e^2), e = 1 - d y0 ~ 2^-23, error e^3:
// one FMA less on the entry's dependent chain
__device__ __forceinline__ double rcp_newton3(double d) {
  double y;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(d));
  const double e = fma(-d, y, 1.0);
  return fma(y, fma(e, e, e), y);
}
// tanh(x) = em / (em + 2) with em = expm1(2x) in [-1, 1e300]: relative
// accuracy for small |x| too (1 - 2 / (exp(2x) + 1) loses it to cancellation)
__device__ __forceinline__ double tanh_from_expm1(double em) { return em * rcp_newton(em + 2.0); }
__device__ __forceinline__ double tanh_from_expm1_tab(double em) { return em * rcp_newton3(em + 2.0); }
// expm1(x) for the table build, |x| <= EXP_SAFE: no special cases and no
// branches (libm's expm1 diverges within a warp, and every warp of the CTA
// waits for the slowest at the chunk barrier). x = n ln2 + r, |r| <= ln2 / 2;
// expm1(x) = 2^n expm1(r) + (2^n - 1), expm1(r) as its degree-13 Taylor
// polynomial (remainder < 1e-17 relative); relative accuracy near 0 is kept
// (n = 0: the polynomial itself). A few ulp.
__device__ __forceinline__ double expm1_table(double x) {
  const double n = rint(x * 1.4426950408889634);
  double r = fma(-n, 6.93147180369123816490e-01, x);  // ln2 high part (trailing zeros: n * hi exact)
  r = fma(-n, 1.90821492927058770002e-10, r);         // ln2 low part
  double q = 1.6059043836821613e-10;                   // 1/13!
  q = fma(q, r, 2.08767569878681e-09);                 // 1/12!
  q = fma(q, r, 2.505210838544172e-08);                // 1/11!
  q = fma(q, r, 2.755731922398589e-07);                // 1/10!
  q = fma(q, r, 2.7557319223985893e-06);               // 1/9!
  q = fma(q, r, 2.48015873015873e-05);                 // 1/8!
  q = fma(q, r, 1.984126984126984e-04);                // 1/7!
  q = fma(q, r, 1.388888888888889e-03);                // 1/6!
  q = fma(q, r, 8.333333333333333e-03);                // 1/5!
  q = fma(q, r, 4.1666666666666664e-02);               // 1/4!
  q = fma(q, r, 1.6666666666666666e-01);               // 1/3!
  q = fma(q, r, 0.5);
  q = fma(q * r, r, r);                                // expm1(r) = r + r^2 (1/2 + r (1/6 + ...))
  const double s = __longlong_as_double(((long long)n + 1023LL) << 52);  // 2^n, |n| <= 332
  return fma(s, q, s - 1.0);
}
// general argument: expm1(2x) clamped below overflow (tanh is 1.0 in fp64 far before)
__device__ __forceinline__ double tanh_fast(double x) { return tanh_from_expm1(fmin(expm1(2.0 * x), 1e300)); }

// activation value and its first two derivatives at pre (basis.py:119-126)
__device__ __forceinline__ void activation(int act, double pre, double& tv, double& g1, double& g2) {
  if (act == FL_ACT_SIN) {
    double sn, cs;
    sincos(pre, &sn, &cs);
    tv = sn;
    g1 = cs;
    g2 = -sn;
  } else if (act == FL_ACT_SIGMOID) {
    const double sg = 0.5 * (1.0 + tanh_fast(0.5 * pre));
    tv = sg;
    g1 = sg * (1.0 - sg);
    g2 = sg * (1.0 - sg) * (1.0 - 2.0 * sg);
  } else {
    tv = tanh_fast(pre);
    g1 = 1.0 - tv * tv;
    g2 = -2.0 * tv * g1;
  }
}

constexpr int ASM_MINB = 3;   // CTAs per SM (D = 3: one less)
constexpr int CK = 64;        // columns per chunk
constexpr int TLMAX = 96;     // lattice coordinates per chunk table (sum over axes)
constexpr int RPT = 2;        // adjacent rows per thread (16-byte stores)
static_assert(RPT % 2 == 0, "rows are stored in pairs");
constexpr int TILE = NT * RPT;
// |2 (x~ W + b)| bound of one table factor: a product of D <= 3 factors
// stays below exp(690) < DBL_MAX, so E + 1 needs no clamp on the table path
constexpr double EXP_SAFE = 230.0;

// Per-row coefficients of entry(r, k) = t A + g1 sum_a fp_ka B_a + g2 sum_a fp_ka^2 C_a.
struct RowCoef {
  double A, B[MAXD], C[MAXD], xt[MAXD];
  int tix[MAXD];
  bool valid, on_box;
};

// Phase 1 for one row: the point, the normalised partition-of-unity window
// jets along every axis (domains.py:109-173: raw (1+cos)^2 factors,
// normaliser over the covering centers in index order, jet quotient
// jets.py:76-80, products jets.py:55-63, mask jets assembly.py:111-112),
// folded with the operator coefficients (problems.py:39-47) and the row
// weight (assembly.py:180-190).
template <int D>
__device__ __forceinline__ void row_coef(const fl_assembly_desc& d, int j, int r, int m, int boxcount,
                                         const int32_t* box, const int (&sidx)[MAXD], const double (*scoef)[2 + 2 * MAXD],
                                         RowCoef& rc) {
  const int S = d.count_per_dim;
  rc.A = 0.0;
  rc.valid = r < m;
  rc.on_box = false;
#pragma unroll
  for (int a = 0; a < MAXD; ++a) {
    rc.B[a] = rc.C[a] = rc.xt[a] = 0.0;
    rc.tix[a] = 0;
  }
  if (!rc.valid) return;
  double x[MAXD];
  const double* mk = nullptr;  // mask jets of this point, (D, 3)
  int coef = 0;
  if (r < boxcount) {
    int rem = r;
    int64_t gid = 0;
    for (int i = D - 1; i >= 0; --i) {
      const int n = box[2 * i + 1];
      const int digit = rem % n;
      rem /= n;
      x[i] = d.axes[d.axis_off[i] + box[2 * i] + digit];
      gid += (int64_t)(box[2 * i] + digit) * d.lattice_stride[i];
      rc.tix[i] = digit;
    }
    rc.on_box = true;
    if (d.mask_int) mk = d.mask_int + gid * D * 3;
  } else {
    const int64_t e = d.con_ptr[j] + (r - boxcount);
    const int pi = d.con_idx[e];
    for (int i = 0; i < D; ++i) x[i] = d.con_pts[(int64_t)pi * D + i];
    coef = 1 + d.con_grp[e];
    if (d.mask_con) mk = d.mask_con + (int64_t)pi * D * 3;
  }
  double fval[MAXD];
  Jet ffull[MAXD];
  for (int i = 0; i < D; ++i) {
    const double* cen = d.centers + (int64_t)i * S;
    const double half = d.half[i];
    const double t = x[i];
    Jet num = raw_factor(t, cen[sidx[i]], half);
    Jet den{0.0, 0.0, 0.0};
    int l = sidx[i] - d.reach, h = sidx[i] + d.reach;
    if (l < 0) l = 0;
    if (h > S - 1) h = S - 1;
    for (int s2 = l; s2 <= h; ++s2) {  // non-covering centers add exact zeros
      Jet f = raw_factor(t, cen[s2], half);
      den.v += f.v;
      den.f += f.f;
      den.s += f.s;
    }
    ffull[i] = jmul(num, jrecip(den));
    Jet numv{num.v, 0.0, 0.0}, denv{den.v, 0.0, 0.0};
    fval[i] = jmul(numv, jrecip(denv)).v;
    rc.xt[i] = (t - cen[sidx[i]]) / half;
  }
  const double* co = scoef[coef];
  const double weight = co[1];
  double wv = 0.0, acc = 0.0;
  for (int a = 0; a < D; ++a) {
    Jet w{0.0, 0.0, 0.0};
    for (int i = 0; i < D; ++i) {
      Jet fi = (i == a) ? ffull[i] : Jet{fval[i], 0.0, 0.0};
      w = (i == 0) ? fi : jmul(w, fi);
    }
    if (mk) w = jmul(w, Jet{mk[3 * a], mk[3 * a + 1], mk[3 * a + 2]});
    if (a == 0) {
      wv = w.v;
      acc = co[0] * wv;
    }
    const double c1 = co[2 + a], c2 = co[2 + D + a];
    acc += c1 * w.f + c2 * w.s;
    rc.B[a] = weight * (c1 * wv + 2.0 * c2 * w.f);
    rc.C[a] = weight * (c2 * wv);
  }
  rc.A = weight * acc;
}

// One CTA per (block j, tile of NT * RPT rows); thread t owns rows RPT t ..
// RPT t + RPT - 1 of the tile and writes them with 16-byte stores.
//
// Phase 1 (row_coef above) folds everything that depends only on the row
// into entry(r, k) = t A_r + g1 sum_a fp_ka B_ra + g2 sum_a fp_ka^2 C_ra,
// with t, g1, g2 the activation jet of feature k at row r and fp_ka =
// W_ka / h_a (basis.py:119-126; the product rule of assembly.py:107-114
// regrouped by activation derivative).
//
// Phase 2 (per 64-column chunk): tanh features on an interior lattice box
// use exp(2 (x~ . W_k + b_k)) = prod_a exp(2 (x~_a W_ka [+ b_k])), kept as
// expm1 values (expm1(a + b) = e_a + e_b + e_a e_b) so tanh = em / (em + 2)
// stays relatively accurate near 0: the per-axis factors of the lattice
// coordinates the tile touches are tabulated once per chunk (~60 expm1 for
// 16384 entries), so an entry costs 2 (D - 1) FMAs, one reciprocal (MUFU +
// 2 Newton steps) and ~10 FMAs,
// with the column terms fp, fp^2 shared by the thread's two rows; rows off
// the lattice (constraint points), other activations and blocks whose
// factors could overflow evaluate exp / sincos per entry.
template <int D>
__global__ void __launch_bounds__(NT, D == 3 ? ASM_MINB - 1 : ASM_MINB) assemble_kernel(fl_assembly_desc d, double* __restrict__ vals,
                                                         const int64_t* __restrict__ boff,
                                                         const int32_t* __restrict__ bld,
                                                         const int32_t* __restrict__ bm) {
  extern __shared__ double smem[];
  const int K = d.nfeat;
  double* tab = smem;             // (CK, TLMAX) exp table of one column chunk
  double* sW = tab + CK * TLMAX;  // (K, D)
  double* sB = sW + K * D;        // (K)
  __shared__ double scoef[8][2 + 2 * MAXD];

  const int j = d.tiles[2 * blockIdx.x];
  const int r0 = d.tiles[2 * blockIdx.x + 1];
  const int m = bm[j];
  const int ld = bld[j];
  const int S = d.count_per_dim;

  bool unsafe = false;
  for (int i = threadIdx.x; i < K * D; i += NT) {
    const int a = i % D;
    const double w = d.weights[(int64_t)j * K * D + i];
    sW[i] = w;
    double e = fabs(2.0 * w);
    if (a == 0) e += fabs(2.0 * d.biases[(int64_t)j * K + i / D]);
    unsafe |= !(e <= EXP_SAFE);
  }
  for (int i = threadIdx.x; i < K; i += NT) sB[i] = d.biases[(int64_t)j * K + i];
  if (threadIdx.x < 8 * (2 + 2 * D)) {
    int g = threadIdx.x / (2 + 2 * D), c = threadIdx.x % (2 + 2 * D);
    if (g <= d.ngroups) scoef[g][c] = d.op_coef[g * (2 + 2 * D) + c];
  }
  __syncthreads();

  // subdomain multi-index (C order, domains.py:73-77)
  int sidx[MAXD];
  {
    int rem = j;
    for (int i = D - 1; i >= 0; --i) {
      sidx[i] = rem % S;
      rem /= S;
    }
  }
  const int32_t* box = d.box + (int64_t)j * D * 2;
  int boxcount = 1;
  for (int i = 0; i < D; ++i) boxcount *= box[2 * i + 1];

  // lattice-coordinate ranges of this tile's box rows, per axis
  int lo[MAXD] = {0, 0, 0}, base[MAXD] = {0, 0, 0};
  int tl = 0;
  const int rb1 = min(r0 + TILE, min(boxcount, m));
  bool use_tab = (d.activation == FL_ACT_TANH) && D >= 2 && rb1 > r0;
  if (use_tab) {
    int st = 1, cnt[MAXD];
    for (int a = D - 1; a >= 0; --a) {
      const int n = box[2 * a + 1];
      const int q0 = r0 / st, q1 = (rb1 - 1) / st;
      int l = 0, c = n;
      if (q1 - q0 < n) {
        const int d0 = q0 % n, d1 = q1 % n;
        if (d1 >= d0) {
          l = d0;
          c = d1 - d0 + 1;
        }
      }
      lo[a] = l;
      cnt[a] = c;
      st *= n;
    }
    for (int a = 0; a < D; ++a) {
      base[a] = tl;
      tl += cnt[a];
    }
    use_tab = tl <= TLMAX;
  }

  // ---- phase 1: this thread's two rows ----
  const int rA = r0 + RPT * threadIdx.x;
  RowCoef rc[RPT];
#pragma unroll
  for (int u = 0; u < RPT; ++u) row_coef<D>(d, j, rA + u, m, boxcount, box, sidx, scoef, rc[u]);
  unsafe = __syncthreads_or(unsafe);
  use_tab = use_tab && !unsafe;
  // ld is a multiple of 16: all RPT rows are stored or none
  const bool store = rA < ld;
  double* out = vals + boff[j] + rA;
  bool row_tab = use_tab;
#pragma unroll
  for (int u = 0; u < RPT; ++u) row_tab = row_tab && (rc[u].on_box || (u > 0 && !rc[u].valid));
  int toff[RPT][MAXD];
#pragma unroll
  for (int u = 0; u < RPT; ++u)
#pragma unroll
    for (int a = 0; a < MAXD; ++a)  // rows off the box (padding) read slot 0, never used
      toff[u][a] = (a < D && rc[u].on_box) ? base[a] + rc[u].tix[a] - lo[a] : 0;
  double invh[MAXD];
#pragma unroll
  for (int a = 0; a < MAXD; ++a) invh[a] = a < D ? 1.0 / d.half[a] : 0.0;

  // column terms fp_a, fp_a^2 of feature k (shared by the two rows)
  auto col_terms = [&](int k, double (&f1)[MAXD], double (&f2)[MAXD]) {
#pragma unroll
    for (int a = 0; a < D; ++a) {
      f1[a] = sW[k * D + a] * invh[a];
      f2[a] = f1[a] * f1[a];
    }
  };
  auto entry = [&](const RowCoef& c, const double (&f1)[MAXD], const double (&f2)[MAXD], double tv, double g1,
                   double g2) {
    double p1 = f1[0] * c.B[0], p2 = f2[0] * c.C[0];
#pragma unroll
    for (int a = 1; a < D; ++a) {
      p1 += f1[a] * c.B[a];
      p2 += f2[a] * c.C[a];
    }
    return tv * c.A + g1 * p1 + g2 * p2;
  };
  // tanh: g2 = -2 t g1, so entry = t A + g1 (p1 + t p2') with p2' = sum_a fp_a^2 (-2 C_a)
  auto entry_tanh = [&](const RowCoef& c, const double (&f1)[MAXD], const double (&f2)[MAXD], double tv) {
    double p1 = f1[0] * c.B[0], p2 = f2[0] * c.C[0];
#pragma unroll
    for (int a = 1; a < D; ++a) {
      p1 += f1[a] * c.B[a];
      p2 += f2[a] * c.C[a];
    }
    const double g1 = fma(-tv, tv, 1.0);
    return fma(g1, fma(tv, p2, p1), tv * c.A);  // c.C holds -2 C on this path (below)
  };

  // this thread's table coordinate: q = tid mod tl (axis ta, normalised
  // coordinate txa), columns tc, tc + tcs, ... of every chunk
  const int tcs = use_tab ? NT / tl : 1;
  const int tq = use_tab ? threadIdx.x % tl : 0, tc = use_tab ? threadIdx.x / tl : 0;
  int ta = 0;
  double txa = 0.0;
  if (use_tab && tc < tcs) {
    while (ta + 1 < D && tq >= base[ta + 1]) ++ta;
    const int digit = lo[ta] + (tq - base[ta]);
    txa = (d.axes[d.axis_off[ta] + box[2 * ta] + digit] - d.centers[(int64_t)ta * S + sidx[ta]]) * invh[ta];
  }

  // threads on the tabulated path only use entry_tanh: fold its factor -2
  // into the rows' C coefficients once (an exact scaling)
  if (row_tab) {
#pragma unroll
    for (int u = 0; u < RPT; ++u)
#pragma unroll
      for (int a = 0; a < MAXD; ++a) rc[u].C[a] *= -2.0;
  }

  // ---- phase 2: 64-column chunks ----
  for (int k0 = 0; k0 < K; k0 += CK) {
    const int nk = min(CK, K - k0);
    if (use_tab) {
      __syncthreads();
      // tab[c * TLMAX + q] = expm1(2 (x~ W_{k0+c, a} [+ b_{k0+c}])), thread -> fixed q
      if (tc < tcs)
        for (int c = tc; c < nk; c += tcs) {
          double e = txa * sW[(k0 + c) * D + ta];
          if (ta == 0) e += sB[k0 + c];
          tab[c * TLMAX + tq] = expm1_table(2.0 * e);
        }
      __syncthreads();
    }
    if (!store) continue;
    if (row_tab) {
      // running pointers to the rows' table slots and to the output column
      // (no index arithmetic per entry)
      const double* tp[RPT][MAXD];
#pragma unroll
      for (int u = 0; u < RPT; ++u)
#pragma unroll
        for (int a = 0; a < MAXD; ++a) tp[u][a] = tab + toff[u][a];
      double* op = out + (int64_t)k0 * ld;
      // four columns x two rows = eight independent entry chains per thread
      // (measured at cfg4, 3 CTAs/SM: unroll 1 / 2 / 4 / 6 / 8 -> 3.48 / 3.39 /
      // 3.10 / 3.17 / 3.14 ms; 2 CTAs/SM without spills 3.36 / 3.28 at 2 / 4)
#pragma unroll 4
      for (int c = 0; c < nk; ++c, op += ld) {
        const int k = k0 + c;
        double f1[MAXD], f2[MAXD];
        col_terms(k, f1, f2);
#pragma unroll
        for (int a = 0; a < D; ++a) asm volatile("" : "+d"(f2[a]));  // shared by the rows, not recomputed per row
        double v[RPT];
#pragma unroll
        for (int u = 0; u < RPT; ++u) {
          // expm1 of a sum from the factors' expm1: prod (1 + e_a) - 1
          double em = tp[u][0][c * TLMAX];
          if (D > 1) {
            const double e1 = tp[u][1][c * TLMAX];
            em = fma(em, e1, em + e1);
          }
          if (D > 2) {
            const double e2 = tp[u][2][c * TLMAX];
            em = fma(em, e2, em + e2);
          }
          // rows past m have all-zero coefficients (row_coef) and read table
          // slot 0, so their entry is a zero without a per-entry branch
          v[u] = entry_tanh(rc[u], f1, f2, tanh_from_expm1_tab(em));
        }
#pragma unroll
        for (int u = 0; u < RPT; u += 2) *reinterpret_cast<double2*>(op + u) = make_double2(v[u], v[u + 1]);
      }
    } else {
      for (int c = 0; c < nk; ++c) {
        const int k = k0 + c;
        double f1[MAXD], f2[MAXD];
        col_terms(k, f1, f2);
        double v[RPT];
#pragma unroll
        for (int u = 0; u < RPT; ++u) {
          double pre = rc[u].xt[0] * sW[k * D + 0];
#pragma unroll
          for (int i = 1; i < D; ++i) pre += rc[u].xt[i] * sW[k * D + i];
          pre += sB[k];
          double tv, g1, g2;
          activation(d.activation, pre, tv, g1, g2);
          v[u] = rc[u].valid ? entry(rc[u], f1, f2, tv, g1, g2) : 0.0;
        }
#pragma unroll
        for (int u = 0; u < RPT; u += 2)
          *reinterpret_cast<double2*>(out + (int64_t)k * ld + u) = make_double2(v[u], v[u + 1]);
      }
    }
  }
}

}  // namespace

extern "C" int32_t fl_assemble_tile_rows(void) { return TILE; }

extern "C" int fl_assemble(const fl_assembly_desc* desc, const fl_blockop* out, void* stream) {
  if (desc->dim < 1 || desc->dim > MAXD || desc->ngroups > 7) return FL_ERR_INVALID;
  if (desc->n_tiles == 0) return FL_OK;
  cudaStream_t s = (cudaStream_t)stream;
  size_t smem = ((size_t)desc->nfeat * (desc->dim + 1) + CK * TLMAX) * sizeof(double);
  if (smem > 220 * 1024) return FL_ERR_INVALID;
  switch (desc->dim) {
    case 1:
      cudaFuncSetAttribute(assemble_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      assemble_kernel<1><<<desc->n_tiles, NT, smem, s>>>(*desc, (double*)out->vals, out->off, out->ld, out->m);
      break;
    case 2:
      cudaFuncSetAttribute(assemble_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      assemble_kernel<2><<<desc->n_tiles, NT, smem, s>>>(*desc, (double*)out->vals, out->off, out->ld, out->m);
      break;
    default:
      cudaFuncSetAttribute(assemble_kernel<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      assemble_kernel<3><<<desc->n_tiles, NT, smem, s>>>(*desc, (double*)out->vals, out->off, out->ld, out->m);
      break;
  }
  FL_CHECK_LAUNCH();
  return FL_OK;
}
