// K1 — fused block assembly (reference: featlsq assembly.py:124-238).
//
// One CTA per (block j, tile of FL_ASM_TILE rows). Phase 1: one thread per
// row evaluates the point, the normalised partition-of-unity window jets
// along every axis (domains.py:109-173: raw (1+cos)^2 factors, per-dim
// normaliser summed over the covering centers in index order, jet quotient
// jets.py:76-80, product over dims jets.py:55-63) and the normalised input
// (basis.py:99-103) into shared memory. Phase 2: every thread produces
// entries (row, k) for k = cg, cg+4, ...: tanh jet of the feature
// (basis.py:119-126, jets.py:89-93), product rule with the window
// (assembly.py:107-114), operator combination (problems.py:39-47) and row
// weight (assembly.py:180-190), stored column-major so a warp writes 32
// consecutive rows of one column (256 B, coalesced). Padding rows
// [m_j, ld_j) are written as exact zeros.
//
// Roofline: HBM write of 8 B per entry (plus a fp64 tanh per entry; see
// DESIGN.md for the FP64 side).
#include "common.cuh"

namespace {

constexpr int TILE = FL_ASM_TILE;
constexpr int NT = 256;
constexpr int CG = NT / TILE;  // column groups
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

struct RowInfo {
  double wv;              // window value
  double wd1[MAXD];       // window d/dx_a
  double wd2[MAXD];       // window d2/dx_a2
  double xt[MAXD];        // normalised input
  int coef;               // op_coef row (0 interior, 1+g constraint group)
  int valid;
};

template <int D>
__global__ void __launch_bounds__(NT) assemble_kernel(fl_assembly_desc d, double* __restrict__ vals,
                                                      const int64_t* __restrict__ boff,
                                                      const int32_t* __restrict__ bld,
                                                      const int32_t* __restrict__ bm) {
  extern __shared__ double smem[];
  const int K = d.nfeat;
  double* sW = smem;              // (K, D)
  double* sB = sW + K * D;        // (K)
  __shared__ RowInfo rinfo[TILE];
  __shared__ double scoef[8][2 + 2 * MAXD];

  const int j = d.tiles[2 * blockIdx.x];
  const int r0 = d.tiles[2 * blockIdx.x + 1];
  const int m = bm[j];
  const int ld = bld[j];
  const int S = d.count_per_dim;

  for (int i = threadIdx.x; i < K * D; i += NT) sW[i] = d.weights[(int64_t)j * K * D + i];
  for (int i = threadIdx.x; i < K; i += NT) sB[i] = d.biases[(int64_t)j * K + i];
  if (threadIdx.x < 8 * (2 + 2 * D)) {
    int g = threadIdx.x / (2 + 2 * D), c = threadIdx.x % (2 + 2 * D);
    if (g <= d.ngroups) scoef[g][c] = d.op_coef[g * (2 + 2 * D) + c];
  }

  // subdomain multi-index (C order, domains.py:73-77)
  int sidx[MAXD];
  {
    int rem = j;
    for (int i = D - 1; i >= 0; --i) {
      sidx[i] = rem % S;
      rem /= S;
    }
  }

  if (threadIdx.x < TILE) {
    const int r = r0 + threadIdx.x;
    RowInfo ri;
    ri.valid = 0;
    ri.coef = 0;
    if (r < m) {
      ri.valid = 1;
      double x[MAXD];
      const int32_t* box = d.box + (int64_t)j * D * 2;
      int boxcount = 1;
      for (int i = 0; i < D; ++i) boxcount *= box[2 * i + 1];
      const double* mk = nullptr;  // mask jets of this point, (D, 3)
      if (r < boxcount) {
        int rem = r;
        int64_t gid = 0;
        for (int i = D - 1; i >= 0; --i) {
          int cnt = box[2 * i + 1];
          int digit = rem % cnt;
          rem /= cnt;
          x[i] = d.axes[d.axis_off[i] + box[2 * i] + digit];
          gid += (int64_t)(box[2 * i] + digit) * d.lattice_stride[i];
        }
        ri.coef = 0;
        if (d.mask_int) mk = d.mask_int + gid * D * 3;
      } else {
        int64_t e = d.con_ptr[j] + (r - boxcount);
        int pi = d.con_idx[e];
        for (int i = 0; i < D; ++i) x[i] = d.con_pts[(int64_t)pi * D + i];
        ri.coef = 1 + d.con_grp[e];
        if (d.mask_con) mk = d.mask_con + (int64_t)pi * D * 3;
      }
      // per-dim normalised factors: value-only and full jets
      double fval[MAXD];
      Jet ffull[MAXD];
      for (int i = 0; i < D; ++i) {
        const double* cen = d.centers + (int64_t)i * S;
        const double half = d.half[i];
        const double t = x[i];
        Jet num = raw_factor(t, cen[sidx[i]], half);
        Jet den{0.0, 0.0, 0.0};
        int lo = sidx[i] - d.reach, hi = sidx[i] + d.reach;
        if (lo < 0) lo = 0;
        if (hi > S - 1) hi = S - 1;
        for (int s = lo; s <= hi; ++s) {  // non-covering centers add exact zeros
          Jet f = raw_factor(t, cen[s], half);
          den.v += f.v;
          den.f += f.f;
          den.s += f.s;
        }
        Jet q = jmul(num, jrecip(den));
        ffull[i] = q;
        Jet numv{num.v, 0.0, 0.0}, denv{den.v, 0.0, 0.0};
        fval[i] = jmul(numv, jrecip(denv)).v;
        ri.xt[i] = (t - cen[sidx[i]]) / half;
      }
      for (int a = 0; a < D; ++a) {
        Jet w{0.0, 0.0, 0.0};
        for (int i = 0; i < D; ++i) {
          Jet fi = (i == a) ? ffull[i] : Jet{fval[i], 0.0, 0.0};
          w = (i == 0) ? fi : jmul(w, fi);
        }
        if (mk) w = jmul(w, Jet{mk[3 * a], mk[3 * a + 1], mk[3 * a + 2]});  // window * mask (assembly.py:111-112)
        if (a == 0) ri.wv = w.v;
        ri.wd1[a] = w.f;
        ri.wd2[a] = w.s;
      }
    }
    rinfo[threadIdx.x] = ri;
  }
  __syncthreads();

  const int tr = threadIdx.x % TILE;
  const int cg = threadIdx.x / TILE;
  const int r = r0 + tr;
  if (r >= ld) return;
  double* out = vals + boff[j] + r;
  const RowInfo& ri = rinfo[tr];
  if (!ri.valid) {
    for (int k = cg; k < K; k += CG) out[(int64_t)k * ld] = 0.0;
    return;
  }
  double invh[MAXD];
  for (int a = 0; a < D; ++a) invh[a] = 1.0 / d.half[a];
  const double* co = scoef[ri.coef];
  const double vcoef = co[0], weight = co[1];
  for (int k = cg; k < K; k += CG) {
    double pre = ri.xt[0] * sW[k * D + 0];
    for (int i = 1; i < D; ++i) pre += ri.xt[i] * sW[k * D + i];
    pre += sB[k];
    double tv, g1, g2;  // activation value, first and second derivative
    if (d.activation == FL_ACT_TANH) {
      tv = tanh(pre);
      g1 = 1.0 - tv * tv;
      g2 = -2.0 * tv * g1;
    } else if (d.activation == FL_ACT_SIN) {
      double sn, cs;
      sincos(pre, &sn, &cs);
      tv = sn;
      g1 = cs;
      g2 = -sn;
    } else {
      double sg = 0.5 * (1.0 + tanh(0.5 * pre));
      tv = sg;
      g1 = sg * (1.0 - sg);
      g2 = sg * (1.0 - sg) * (1.0 - 2.0 * sg);
    }
    double acc = 0.0;
    for (int a = 0; a < D; ++a) {
      double fp = sW[k * D + a] * invh[a];
      double f1 = g1 * fp;
      double f2 = g2 * fp * fp;
      double v = ri.wv * tv;
      double d1 = ri.wd1[a] * tv + ri.wv * f1;
      double d2 = ri.wd2[a] * tv + 2.0 * ri.wd1[a] * f1 + ri.wv * f2;
      if (a == 0) acc = vcoef * v;
      acc = acc + co[2 + a] * d1 + co[2 + D + a] * d2;
    }
    out[(int64_t)k * ld] = acc * weight;
  }
}

}  // namespace

extern "C" int fl_assemble(const fl_assembly_desc* desc, const fl_blockop* out, void* stream) {
  if (desc->dim < 1 || desc->dim > MAXD || desc->ngroups > 7) return FL_ERR_INVALID;
  if (desc->n_tiles == 0) return FL_OK;
  cudaStream_t s = (cudaStream_t)stream;
  size_t smem = (size_t)desc->nfeat * (desc->dim + 1) * sizeof(double);
  if (smem > 200 * 1024) return FL_ERR_INVALID;
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
