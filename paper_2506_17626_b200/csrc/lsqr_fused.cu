// K4 fused — one HBM pass over Q per LSQR iteration (solvers.py:119-144).
//
// The loop is rotated so that one kernel does the second half of iteration k
// and the first product of iteration k+1 for every block j:
//
//   x      += (phi_k / rho_k) w_k                          (x update, monitor, divergence)
//   v'_j    = Q_j^T (u'[I_j] / beta_{k+1}) - beta_{k+1} v_j (first use of a column tile of Q_j)
//   p_j    += Q_j[:, tile] v'_j[tile]                       (second use of the same tile)
//
// A column tile (W columns, all m_j rows) is staged once in shared memory
// (TMA bulk copies into an ST-deep mbarrier ring) and used by both products,
// because p_j = Q_j v'_j = sum over tiles of Q_j[:, tile] v'_j[tile] needs
// each tile's own entries only. The normalisation v_{k+1} = v'/alpha_{k+1}
// (alpha is a grid-wide norm) is applied afterwards by linearity in the row
// kernel:
//
//   u''    = (sum over covering blocks of p) / alpha_{k+1} - alpha_{k+1} u'/beta_{k+1}
//   v      = v' / alpha_{k+1};  w = v - (theta_{k+1} / rho_k) w
//
// so Q is read from HBM once per iteration instead of twice (Q v and
// Q^T u by separate passes). Scalars: the last CTA of each kernel (fixed-order
// sums) runs the reference's recurrences; every kernel is a no-op once `done`.
//
// One CTA streams one column range of one block: block j's column tiles are
// split over S CTAs (S <= FL_LSQR_SPLIT_MAX), each writing its own copy of
// p_j, which the row kernel sums in a fixed order — finer work units shorten
// the tail of the last wave. The CTA shape (NT threads, RPT rows per thread,
// W columns per tile, ST ring stages) is picked per layout from the
// instantiated table at the bottom: NT = 256 runs two CTAs per SM so one
// block's prologue/epilogue overlaps another block's stream.
#include <float.h>
#include <stdio.h>
#include <stdlib.h>

#include "common.cuh"

namespace {

// shared memory per CTA with MB CTAs resident per SM: 227 KB for one, else
// (228 KB - MB x 1 KB reserved) / MB
constexpr int smem_per_cta(int mb) { return mb <= 1 ? 232448 : (233472 - mb * 1024) / mb; }

__device__ __forceinline__ bool is_done(const fl_lsqr_state* st) { return *(volatile const int32_t*)&st->done; }

// mode 0: initialisation (v = 0, no x update); mode 1: iteration `it`.
// RPT * NT >= ld of every block.
template <int NT, int RPT, int W, int ST, int MB>
__global__ void __launch_bounds__(NT, MB)
    fused_kernel(fl_blockop op, fl_lsqr_vecs vec, fl_lsqr_state* st, int64_t it, int mode, int ldmax, int S) {
  constexpr int NW = NT / 32;
  constexpr int GL = NW;        // lanes per column in the cross-warp shuffle tree
  constexpr int CPP = 32 / GL;  // columns per shuffle pass
  if (is_done(st)) return;
  extern __shared__ __align__(128) double sm[];
  double* tile = sm;  // [ST][W][ldmax] column tiles of Q_j
  __shared__ double red[2 * NW * W];
  __shared__ double red2[NW];
  __shared__ __align__(8) uint64_t bars[ST];
  __shared__ int s_bad;
  __shared__ bool is_last;

  const int ub = blockIdx.x / S, h = blockIdx.x % S;
  const int j = op.order ? op.order[ub] : ub;  // largest blocks first (shorter tail)
  const int m = op.m[j];
  const int ld = op.ld[j];
  const int nc = op.ncols[j];
  const int64_t co = op.col_off[j];
  const double* Q = op.vals + op.off[j];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const double beta = st->beta;
  const bool work = beta > 0.0;
  const int nt_all = (nc + W - 1) / W;
  const int t0 = (int)((int64_t)nt_all * h / S);  // this CTA's column tiles [t0, t1)
  const int t1 = (int)((int64_t)nt_all * (h + 1) / S);
  const int ntiles = work ? t1 - t0 : 0;
  const int cbeg = min(t0 * W, nc), cend = min(t1 * W, nc);  // x update runs even when beta = 0
  const int64_t cob = co + cbeg;  // first y-space entry of the range
  const int ncr = cend - cbeg;
  if (threadIdx.x == 0) {
    s_bad = 0;
    for (int s = 0; s < ST; ++s)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"((unsigned)__cvta_generic_to_shared(&bars[s]))
                   : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();

  // TMA bulk copies: thread 0 moves whole columns (ld * 8 bytes each) into
  // the stage and arms the stage's mbarrier with the byte count
  auto issue = [&](int tidx) {
    if (threadIdx.x != 0 || tidx >= ntiles) return;
    const int s = tidx % ST;
    const int c0 = (t0 + tidx) * W;
    const int ncl = min(W, nc - c0);
    const unsigned bar = (unsigned)__cvta_generic_to_shared(&bars[s]);
    const unsigned bytes = (unsigned)ld * 8u;
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(bar), "r"(bytes * ncl) : "memory");
    for (int c = 0; c < ncl; ++c) {
      const unsigned dst = (unsigned)__cvta_generic_to_shared(tile + (s * W + c) * ldmax);
      asm volatile(
          "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(dst),
          "l"(Q + (int64_t)(c0 + c) * ld), "r"(bytes), "r"(bar)
          : "memory");
    }
  };
  auto wait_tile = [&](int tidx) {
    const unsigned bar = (unsigned)__cvta_generic_to_shared(&bars[tidx % ST]);
    const unsigned parity = (unsigned)((tidx / ST) & 1);
    unsigned ok = 0;
    while (!ok)
      asm volatile(
          "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }\n"
          : "=r"(ok)
          : "r"(bar), "r"(parity)
          : "memory");
  };
  // the ring fills while the x update and the u gather run
#pragma unroll
  for (int s = 0; s < ST - 1; ++s) issue(s);

  // ---- x update for this block's columns (iteration `it`) ----
  double wss = 0.0;
  bool improve = false;
  const double phibar = st->phibar;
  if (mode == 0) {
    for (int c = threadIdx.x; c < ncr; c += NT)
      vec.x[cob + c] = vec.w[cob + c] = vec.xbest[cob + c] = vec.v[cob + c] = 0.0;
  } else {
    const double step = st->phi / st->rho;
    const bool record = (st->stride <= 1 || it % st->stride == 0);
    // best iterate: by residual here, or (test-error monitor, monitor.cu) the
    // previous recorded x when its error was the new best
    const bool mon = st->monitor;
    improve = mon ? (*(volatile const int32_t*)&st->improved != 0) : (record && (phibar < st->best));
    int bad = 0;
    for (int c = threadIdx.x; c < ncr; c += NT) {
      const double wc = vec.w[cob + c];
      const double xo = vec.x[cob + c];
      const double xn = xo + step * wc;
      vec.x[cob + c] = xn;
      bad |= !isfinite(xn);
      if (improve) vec.xbest[cob + c] = mon ? xo : xn;
      wss += wc * wc;
    }
    if (bad) atomicOr(&s_bad, 1);
  }
  double ass = 0.0;  // sum of v'^2 over this CTA's columns (thread 0)
  if (work) {
    // ---- u'/beta and the partial product live in registers: thread t owns
    //      rows t, t + NT, ... ----
    const int32_t* rows = op.rows + op.row_off[j];
    double uh_r[RPT], pp_r[RPT];
#pragma unroll
    for (int i = 0; i < RPT; ++i) {
      const int r = threadIdx.x + i * NT;
      uh_r[i] = (r < m) ? vec.u[rows[r]] / beta : 0.0;
      pp_r[i] = 0.0;
    }
    // v_j[tile] is read one tile ahead (broadcast loads, off the critical path)
    double vnext[W];
    auto load_v = [&](int tdx) {
#pragma unroll
      for (int c = 0; c < W; ++c) {
        const int col = (t0 + tdx) * W + c;
        vnext[c] = (mode == 1 && col < nc) ? vec.v[co + col] : 0.0;
      }
    };
    load_v(0);
    for (int tdx = 0; tdx < ntiles; ++tdx) {
      double vcur[W];
#pragma unroll
      for (int c = 0; c < W; ++c) vcur[c] = vnext[c];
      if (tdx + 1 < ntiles) load_v(tdx + 1);
      wait_tile(tdx);
      const int ncl = min(W, nc - (t0 + tdx) * W);  // valid columns in this tile
      const double* tl = tile + (tdx % ST) * W * ldmax;
      double acc[W];
#pragma unroll
      for (int c = 0; c < W; ++c) acc[c] = 0.0;
#pragma unroll
      for (int i = 0; i < RPT; ++i) {
        const int r = threadIdx.x + i * NT;
        if (r < ld) {
#pragma unroll
          for (int c = 0; c < W; ++c)
            if (c < ncl) acc[c] += tl[c * ldmax + r] * uh_r[i];
        }
      }
#pragma unroll
      for (int c = 0; c < W; ++c) {
        const double s = fl::warp_sum(acc[c]);
        if (lane == 0) red[(tdx & 1) * NW * W + wid * W + c] = s;
      }
      __syncthreads();         // partials visible; every thread is done with tile tdx-1
      issue(tdx + ST - 1);     // refills the stage tile tdx-1 used
      // v'[tile] = Q[:, tile]^T u - beta v[tile] (solvers.py:136): every warp
      // sums the NW warp partials itself with the same GL-lane shuffle tree
      // (CPP columns per pass), so no second barrier is needed; `red`
      // alternates buffers by tile parity
      double tc[W];
      const double* rb = red + (tdx & 1) * NW * W;
#pragma unroll
      for (int c0 = 0; c0 < W; c0 += CPP) {
        const int c = c0 + lane / GL;
        double s = (c < W) ? rb[(lane % GL) * W + c] : 0.0;
#pragma unroll
        for (int o = GL / 2; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
#pragma unroll
        for (int q = 0; q < CPP; ++q) {
          const double sq = __shfl_sync(0xffffffffu, s, q * GL);
          if (c0 + q < W) tc[c0 + q] = sq;
        }
      }
#pragma unroll
      for (int c = 0; c < W; ++c) {
        const int col = (t0 + tdx) * W + c;
        double vn = 0.0;
        if (c < ncl) vn = tc[c] - ((mode == 1) ? beta * vcur[c] : 0.0);
        tc[c] = vn;
        if (threadIdx.x == 0) {
          if (c < ncl) vec.vp[co + col] = vn;
          ass += vn * vn;
        }
      }
#pragma unroll
      for (int i = 0; i < RPT; ++i) {
        const int r = threadIdx.x + i * NT;
        if (r < ld) {
#pragma unroll
          for (int c = 0; c < W; ++c)
            if (c < ncl) pp_r[i] += tl[c * ldmax + r] * tc[c];
        }
      }
    }
#pragma unroll
    for (int i = 0; i < RPT; ++i) {
      const int r = threadIdx.x + i * NT;
      if (r < m) op.partial[h * op.partial_len + op.row_off[j] + r] = pp_r[i];
    }
  }
  // ---- grid reductions: alpha^2, w^2, non-finite ----
  __syncthreads();
  double wsum = fl::block_sum(wss, red2);
  const int G = gridDim.x;
  double* slots = op.red_scratch;
  if (threadIdx.x == 0) {
    slots[blockIdx.x] = ass;
    slots[G + blockIdx.x] = wsum;
    if (s_bad) atomicOr(&st->nonfinite, 1);
    __threadfence();
    const unsigned prev = atomicAdd(op.counter, 1u);
    is_last = (prev == (unsigned)G - 1);
  }
  __syncthreads();
  if (!is_last) return;
  __threadfence();
  double a = 0.0, b = 0.0;
  for (int i = threadIdx.x; i < G; i += NT) {
    a += ((volatile double*)slots)[i];
    b += ((volatile double*)slots)[G + i];
  }
  a = fl::block_sum(a, red2);
  b = fl::block_sum(b, red2);
  if (threadIdx.x != 0) return;
  *op.counter = 0u;
  const double alpha = sqrt(a);
  if (mode == 0) {  // solvers.py:108-117
    st->alpha = alpha;
    st->rhobar = alpha;
    st->theta = 0.0;
    st->rho = 1.0;
    st->anorm = 0.0;  // scipy-rule accumulators (scipy.sparse.linalg.lsqr init)
    st->ddnorm = 0.0;
    st->xxnorm = 0.0;
    st->z = 0.0;
    st->cs2 = -1.0;
    st->sn2 = 0.0;
    if (alpha == 0.0) {
      st->breakdown = 1;
      st->done = 1;
    }
    return;
  }
  st->it = it;
  if (st->monitor) st->improved = 0;  // every CTA has read it
  if (*(volatile int32_t*)&st->nonfinite) {  // DivergenceError at iteration it
    st->diverged_at = it;
    st->done = 1;
    return;
  }
  if (improve && !st->monitor) {
    st->best = phibar;
    st->best_it = it;
  }
  if (beta == 0.0) {  // solvers.py:133-135
    st->breakdown = 1;
    st->done = 1;
    return;
  }
  st->alpha = alpha;
  if (alpha == 0.0) {  // solvers.py:138-140
    st->breakdown = 1;
    st->done = 1;
    return;
  }
  const double theta = st->s * alpha;  // solvers.py:142-143
  st->theta = theta;
  st->rhobar = -st->c * alpha;
  if (st->use_rule) {
    const double rho = st->rho, phi = st->phi;
    const double tau = st->s * phi;
    st->ddnorm += b / (rho * rho);
    const double delta = st->sn2 * rho;
    const double gambar = -st->cs2 * rho;
    const double rhs = phi - delta * st->z;
    const double zbar = rhs / gambar;
    const double xnorm = sqrt(st->xxnorm + zbar * zbar);
    const double gamma = sqrt(gambar * gambar + theta * theta);
    st->cs2 = gambar / gamma;
    st->sn2 = theta / gamma;
    st->z = rhs / gamma;
    st->xxnorm += st->z * st->z;
    const double acond = st->anorm * sqrt(st->ddnorm);
    const double rnorm = st->phibar;
    const double arnorm = alpha * fabs(tau);
    const double eps = DBL_EPSILON;
    const double test1 = rnorm / st->bnorm;
    const double test2 = arnorm / (st->anorm * rnorm + eps);
    const double test3 = 1.0 / (acond + eps);
    const double t1 = test1 / (1.0 + st->anorm * xnorm / st->bnorm);
    const double rtol = st->btol + st->atol * st->anorm * xnorm / st->bnorm;
    int istop = 0;
    if (1.0 + test3 <= 1.0) istop = 6;
    if (1.0 + test2 <= 1.0) istop = 5;
    if (1.0 + t1 <= 1.0) istop = 4;
    if (test3 <= st->ctol) istop = 3;
    if (test2 <= st->atol) istop = 2;
    if (test1 <= rtol) istop = 1;
    if (istop) {
      st->istop = istop;
      st->done = 1;
    }
  }
}

// Row pass of iteration `it`: u'' = gather(p)/alpha - alpha u'/beta, ||u''||,
// v = v'/alpha, w = v - (theta/rho_prev) w, then the scalar step (S1) of
// iteration `it` in the last CTA (solvers.py:120-127).
__global__ void __launch_bounds__(256) row_kernel(fl_blockop op, fl_lsqr_vecs vec, fl_lsqr_state* st, int64_t it,
                                                 int S) {
  if (is_done(st)) return;
  __shared__ double sh[8];
  const double alpha = st->alpha, bprev = st->beta_prev;
  const double tr = st->theta / st->rho;  // rho here is rho_{it-1}
  const int gtid = blockIdx.x * blockDim.x + threadIdx.x, gsz = gridDim.x * blockDim.x;
  double ss = 0.0;
  for (int g = gtid; g < op.nrows; g += gsz) {
    double acc = 0.0;
    for (int e = op.gptr[g]; e < op.gptr[g + 1]; ++e) {
      const int64_t src = op.gsrc[e];
      for (int h = 0; h < S; ++h) acc += op.partial[h * op.partial_len + src];
    }
    const double un = acc / alpha - alpha * (vec.u[g] / bprev);
    vec.u[g] = un;
    ss += un * un;
  }
  for (int64_t c = gtid; c < op.ncols_total; c += gsz) {
    const double vv = vec.vp[c] / alpha;  // v = v'/alpha (:141)
    vec.v[c] = vv;
    vec.w[c] = vv - tr * vec.w[c];       // w = v - (theta/rho) w (:144)
  }
  ss = fl::block_sum(ss, sh);
  double tot;
  if (fl::grid_sum_last(ss, op.red_scratch, op.counter, &tot, sh) && threadIdx.x == 0) {
    const double beta = sqrt(tot);
    const double rho = hypot(st->rhobar, beta);
    const double c = st->rhobar / rho, s = beta / rho;
    const double phi = c * st->phibar;
    if (st->use_rule) st->anorm = sqrt(st->anorm * st->anorm + alpha * alpha + beta * beta);
    st->beta = beta;
    if (beta > 0.0) st->beta_prev = beta;
    st->rho = rho;
    st->c = c;
    st->s = s;
    st->phi = phi;
    st->phibar = s * st->phibar;
    vec.trace[it] = st->phibar;
  }
}

// ---- CTA-shape table -----------------------------------------------------
// A shape fits a layout when RPT * NT >= ldmax and its ring (ST * W * ldmax
// doubles) plus static shared memory fits the per-CTA budget. Entries are in
// preference order; FEATLSQ_FUSED="NT,W,ST,MB" restricts the choice (tuning).

enum { SKIP = 1 };

template <int NT, int RPT, int W, int ST, int MB>
int try_fused(const fl_blockop* op, fl_lsqr_vecs* vecs, fl_lsqr_state* st, int64_t it, int mode, int ldmax,
              int S, cudaStream_t s, bool dry) {
  if ((int64_t)RPT * NT < ldmax) return SKIP;
  static int stat = -1;
  static size_t attr = 0;
  if (stat < 0) {
    cudaFuncAttributes a;
    FL_CUDA(cudaFuncGetAttributes(&a, fused_kernel<NT, RPT, W, ST, MB>));
    stat = (int)a.sharedSizeBytes;
  }
  const size_t dyn = (size_t)ST * W * ldmax * sizeof(double);
  if (dyn + stat > (size_t)smem_per_cta(MB)) return SKIP;
  if (dry) return FL_OK;
  if (dyn > attr) {
    FL_CUDA(cudaFuncSetAttribute(fused_kernel<NT, RPT, W, ST, MB>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)dyn));
    attr = dyn;
  }
  fused_kernel<NT, RPT, W, ST, MB><<<op->nblocks * S, NT, dyn, s>>>(*op, *vecs, st, it, mode, ldmax, S);
  FL_CHECK_LAUNCH();
  return FL_OK;
}

struct Shape {
  int nt, rpt, w, st, mb;
  int (*fn)(const fl_blockop*, fl_lsqr_vecs*, fl_lsqr_state*, int64_t, int, int, int, cudaStream_t, bool);
};

#define FL_SHAPE(NT, R, W, S, MB) {NT, R, W, S, MB, try_fused<NT, R, W, S, MB>}
const Shape kShapes[] = {
    FL_SHAPE(512, 1, 8, 3, 1), FL_SHAPE(512, 2, 8, 3, 1), FL_SHAPE(512, 3, 4, 3, 1), FL_SHAPE(512, 3, 3, 3, 1),
    FL_SHAPE(512, 4, 4, 3, 1), FL_SHAPE(512, 4, 3, 3, 1), FL_SHAPE(512, 4, 2, 4, 1),
    FL_SHAPE(256, 12, 1, 3, 3), FL_SHAPE(256, 12, 1, 5, 2), FL_SHAPE(256, 12, 1, 4, 2),
    FL_SHAPE(128, 24, 1, 3, 3), FL_SHAPE(128, 24, 1, 2, 4), FL_SHAPE(256, 12, 1, 2, 4),
    FL_SHAPE(512, 6, 3, 3, 1), FL_SHAPE(512, 6, 1, 9, 1),
    FL_SHAPE(512, 8, 2, 3, 1), FL_SHAPE(512, 8, 1, 6, 1), FL_SHAPE(512, 8, 1, 4, 1),
    FL_SHAPE(512, 12, 1, 4, 1), FL_SHAPE(512, 12, 1, 3, 1),
};
#undef FL_SHAPE

struct EnvShape {
  int nt = 0, w = 0, st = 0, mb = 0;
  EnvShape() {
    const char* e = getenv("FEATLSQ_FUSED");
    if (e) sscanf(e, "%d,%d,%d,%d", &nt, &w, &st, &mb);
  }
};

int ldmax_of(const fl_blockop* op) { return (int)fl::round_up(op->max_rows > 0 ? op->max_rows : 1, 16); }

// Column split S: the fewest CTAs per block that give at least 4 work units
// per resident CTA slot (FEATLSQ_SPLIT overrides, tuning).
int split_of(const fl_blockop* op, const Shape& sh) {
  static const int env = [] {
    const char* e = getenv("FEATLSQ_SPLIT");
    return e ? atoi(e) : 0;
  }();
  if (env > 0) return env < FL_LSQR_SPLIT_MAX ? env : FL_LSQR_SPLIT_MAX;
  static int nsm = 0;
  if (!nsm) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    if (nsm <= 0) nsm = 148;
  }
  int S = 1;
  while (S < FL_LSQR_SPLIT_MAX && (int64_t)op->nblocks * S < 4LL * nsm * sh.mb) ++S;
  return S;
}

// the shape picked for this layout (first fit in table order), or nullptr
const Shape* shape_of(const fl_blockop* op) {
  static const EnvShape env;
  const int ldmax = ldmax_of(op);
  for (const Shape& sh : kShapes) {
    if (env.nt && (sh.nt != env.nt || sh.w != env.w || sh.st != env.st || sh.mb != env.mb)) continue;
    if (sh.fn(op, nullptr, nullptr, 0, 0, ldmax, 1, nullptr, true) == FL_OK) return &sh;
  }
  return nullptr;
}

int fused(const fl_blockop* op, fl_lsqr_vecs* vecs, fl_lsqr_state* st, int64_t it, int mode, int S,
          cudaStream_t s) {
  const Shape* sh = shape_of(op);
  if (!sh) return FL_ERR_INVALID;
  return sh->fn(op, vecs, st, it, mode, ldmax_of(op), S, s, false);
}

int row_grid(const fl_blockop* op) {
  const int64_t n = op->nrows > op->ncols_total ? op->nrows : op->ncols_total;
  int64_t g = (n + 255) / 256;
  if (g > 148 * 8) g = 148 * 8;
  return (int)(g < 1 ? 1 : g);
}

}  // namespace

namespace fl {
bool fused_ok(const fl_blockop* op) { return shape_of(op) != nullptr; }
// init: caller has run lsqr_init_a (u = rhs, beta); this runs v' = Q^T u/beta, p = Q v'
int lsqr_fused_init(const fl_blockop* op, fl_lsqr_vecs* vecs, fl_lsqr_state* st, cudaStream_t s) {
  const Shape* sh = shape_of(op);
  if (!sh) return FL_ERR_INVALID;
  return fused(op, vecs, st, 0, 0, split_of(op, *sh), s);
}
int monitor_step(const fl_test_monitor* mon, const double* x, fl_lsqr_state* st, int64_t it, cudaStream_t s);
int lsqr_fused_iterate(const fl_blockop* op, fl_lsqr_vecs* vecs, fl_lsqr_state* st, int64_t first_it,
                       int64_t count, const fl_test_monitor* mon, cudaStream_t s) {
  const Shape* sh = shape_of(op);
  if (!sh) return FL_ERR_INVALID;
  const int S = split_of(op, *sh);
  const int rg = row_grid(op);
  for (int64_t k = 0; k < count; ++k) {
    const int64_t it = first_it + k;
    row_kernel<<<rg, 256, 0, s>>>(*op, *vecs, st, it, S);
    FL_CHECK_LAUNCH();
    int e = fused(op, vecs, st, it, 1, S, s);
    if (e) return e;
    if (mon && (e = monitor_step(mon, vecs->x, st, it, s))) return e;
  }
  return FL_OK;
}
}  // namespace fl
