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
// (cp.async, double buffered) and used by both products, because p_j =
// Q_j v'_j = sum over tiles of Q_j[:, tile] v'_j[tile] needs each tile's own
// entries only. The normalisation v_{k+1} = v'/alpha_{k+1} (alpha is a grid-
// wide norm) is applied afterwards by linearity in the row kernel:
//
//   u''    = (sum over covering blocks of p) / alpha_{k+1} - alpha_{k+1} u'/beta_{k+1}
//   v      = v' / alpha_{k+1};  w = v - (theta_{k+1} / rho_k) w
//
// so Q is read from HBM once per iteration instead of twice (Q v and
// Q^T u by separate passes). Scalars: the last CTA of each kernel (fixed-order
// sums) runs the reference's recurrences; every kernel is a no-op once `done`.
#include <float.h>

#include "common.cuh"

namespace {

constexpr int NT = 512;
constexpr int NW = NT / 32;
constexpr int SMEM_BUDGET = 210 * 1024;
constexpr int STAGES = 3;    // column-tile ring
constexpr int RPT_MAX = 12;  // rows per thread held in registers (ld <= 6144)
constexpr int VMAX = 1024;   // columns per block staged in shared memory

__device__ __forceinline__ bool is_done(const fl_lsqr_state* st) { return *(volatile const int32_t*)&st->done; }

__device__ __forceinline__ void cp16(void* s, const void* g) {
  unsigned a = (unsigned)__cvta_generic_to_shared(s);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(a), "l"(g));
}
__device__ __forceinline__ void commit() { asm volatile("cp.async.commit_group;\n" ::); }
__device__ __forceinline__ void waitN() { asm volatile("cp.async.wait_group %0;\n" ::"n"(STAGES - 2)); }

// mode 0: initialisation (v = 0, no x update); mode 1: iteration `it`.
// RPT = rows per thread (RPT * NT >= ld of every block), W = columns per tile.
template <int RPT, int W>
__global__ void __launch_bounds__(NT, 1) fused_kernel(fl_blockop op, fl_lsqr_vecs vec, fl_lsqr_state* st,
                                                      int64_t it, int mode, int ldmax) {
  if (is_done(st)) return;
  extern __shared__ double sm[];
  double* tile = sm;               // [STAGES][W][ldmax] column tiles of Q_j
  __shared__ double red[2 * NW * W];
  __shared__ double red2[NW];
  __shared__ __align__(8) uint64_t bars[STAGES];
  __shared__ double vsh[VMAX];  // v_j, staged once (off the reduction's critical path)
  __shared__ int s_bad;
  __shared__ bool is_last;
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"((unsigned)__cvta_generic_to_shared(&bars[s]))
                   : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();

  const int j = op.order ? op.order[blockIdx.x] : blockIdx.x;  // largest blocks first (shorter tail)
  const int m = op.m[j];
  const int ld = op.ld[j];
  const int nc = op.ncols[j];
  const int64_t co = op.col_off[j];
  const double* Q = op.vals + op.off[j];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const double beta = st->beta;
  if (threadIdx.x == 0) s_bad = 0;

  // ---- x update for this block's columns (iteration `it`) ----
  double wss = 0.0;
  bool improve = false;
  const double phibar = st->phibar;
  if (mode == 0) {
    for (int c = threadIdx.x; c < nc; c += NT) vec.x[co + c] = vec.w[co + c] = vec.xbest[co + c] = vec.v[co + c] = 0.0;
  } else {
    const double step = st->phi / st->rho;
    const bool record = (st->stride <= 1 || it % st->stride == 0);
    improve = record && (phibar < st->best);
    int bad = 0;
    for (int c = threadIdx.x; c < nc; c += NT) {
      const double wc = vec.w[co + c];
      const double xn = vec.x[co + c] + step * wc;
      vec.x[co + c] = xn;
      bad |= !isfinite(xn);
      if (improve) vec.xbest[co + c] = xn;
      wss += wc * wc;
    }
    __syncthreads();
    if (bad) atomicOr(&s_bad, 1);
  }
  double ass = 0.0;  // sum of v'^2 over this block's columns (thread 0)
  const bool work = (beta > 0.0) && nc > 0;
  if (work) {
    // ---- u'/beta and the partial product live in registers: thread t owns
    //      rows t, t + NT, ... (RPT * NT >= ldmax) ----
    const int32_t* rows = op.rows + op.row_off[j];
    if (mode == 1)
      for (int c = threadIdx.x; c < nc; c += NT) vsh[c] = vec.v[co + c];
    double uh_r[RPT], pp_r[RPT];
#pragma unroll
    for (int i = 0; i < RPT; ++i) {
      const int r = threadIdx.x + i * NT;
      uh_r[i] = (r < m) ? vec.u[rows[r]] / beta : 0.0;
      pp_r[i] = 0.0;
    }
    const int ntiles = (nc + W - 1) / W;
    // TMA bulk copies: thread 0 moves whole columns (ld * 8 bytes each) into
    // the stage and arms the stage's mbarrier with the byte count
    auto issue = [&](int tidx) {
      if (threadIdx.x != 0 || tidx >= ntiles) return;
      const int s = tidx % STAGES;
      const int c0 = tidx * W;
      const int ncl = min(W, nc - c0);
      const unsigned bar = (unsigned)__cvta_generic_to_shared(&bars[s]);
      const unsigned bytes = (unsigned)ld * 8u;
      asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(bar), "r"(bytes * ncl)
                   : "memory");
      for (int c = 0; c < ncl; ++c) {
        const unsigned dst = (unsigned)__cvta_generic_to_shared(tile + (s * W + c) * ldmax);
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(dst),
            "l"(Q + (int64_t)(c0 + c) * ld), "r"(bytes), "r"(bar)
            : "memory");
      }
    };
    auto wait_tile = [&](int tidx) {
      const unsigned bar = (unsigned)__cvta_generic_to_shared(&bars[tidx % STAGES]);
      const unsigned parity = (unsigned)((tidx / STAGES) & 1);
      unsigned ok = 0;
      while (!ok)
        asm volatile(
            "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }\n"
            : "=r"(ok)
            : "r"(bar), "r"(parity)
            : "memory");
    };
#pragma unroll
    for (int s = 0; s < STAGES - 1; ++s) issue(s);
    for (int tdx = 0; tdx < ntiles; ++tdx) {
      wait_tile(tdx);
      const int ncl = min(W, nc - tdx * W);  // valid columns in this tile
      const double* tl = tile + (tdx % STAGES) * W * ldmax;
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
      __syncthreads();  // partials visible; every thread is done with tile tdx-1
      issue(tdx + STAGES - 1);  // refills the stage tile tdx-1 used
      // v'[tile] = Q[:, tile]^T u - beta v[tile] (solvers.py:136): every warp
      // sums the NW warp partials itself with the same 16-lane shuffle tree
      // (two columns per pass: lanes 0-15 column c, lanes 16-31 column c+1),
      // so no second barrier is needed; `red` alternates buffers by tile parity
      double tc[W];
      const double* rb = red + (tdx & 1) * NW * W;
#pragma unroll
      for (int c0 = 0; c0 < W; c0 += 2) {
        const int c = c0 + (lane >> 4);
        double s = (c < W) ? rb[(lane & 15) * W + c] : 0.0;
#pragma unroll
        for (int o = 8; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        const double s0 = __shfl_sync(0xffffffffu, s, 0), s1 = __shfl_sync(0xffffffffu, s, 16);
        tc[c0] = s0;
        if (c0 + 1 < W) tc[c0 + 1] = s1;
      }
#pragma unroll
      for (int c = 0; c < W; ++c) {
        const int col = tdx * W + c;
        double vn = 0.0;
        if (c < ncl) vn = tc[c] - ((mode == 1) ? beta * vsh[col] : 0.0);
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
      if (r < m) op.partial[op.row_off[j] + r] = pp_r[i];
    }
  }
  // ---- grid reductions: alpha^2, w^2, non-finite ----
  __syncthreads();
  double wsum = fl::block_sum(wss, red2);
  const int G = gridDim.x;
  double* slots = op.red_scratch;
  if (threadIdx.x == 0) {
    slots[j] = ass;
    slots[G + j] = wsum;
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
  if (*(volatile int32_t*)&st->nonfinite) {  // DivergenceError at iteration it
    st->diverged_at = it;
    st->done = 1;
    return;
  }
  if (improve) {
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
__global__ void __launch_bounds__(256) row_kernel(fl_blockop op, fl_lsqr_vecs vec, fl_lsqr_state* st, int64_t it) {
  if (is_done(st)) return;
  __shared__ double sh[8];
  const double alpha = st->alpha, bprev = st->beta_prev;
  const double tr = st->theta / st->rho;  // rho here is rho_{it-1}
  const int gtid = blockIdx.x * blockDim.x + threadIdx.x, gsz = gridDim.x * blockDim.x;
  double ss = 0.0;
  for (int g = gtid; g < op.nrows; g += gsz) {
    double acc = 0.0;
    for (int e = op.gptr[g]; e < op.gptr[g + 1]; ++e) acc += op.partial[op.gsrc[e]];
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

int pick_w(int ldmax) {
  if (ldmax > RPT_MAX * NT) return 0;
  const long w = SMEM_BUDGET / ((long)STAGES * ldmax * 8);
  if (w >= 8) return 8;
  if (w >= 4) return 4;
  if (w >= 3) return 3;
  if (w >= 2) return 2;
  return w >= 1 ? 1 : 0;
}

template <int RPT, int W>
int launch_fused(const fl_blockop* op, fl_lsqr_vecs* vecs, fl_lsqr_state* st, int64_t it, int mode, int ldmax,
                 cudaStream_t s) {
  const size_t smem = (size_t)STAGES * W * ldmax * sizeof(double);
  static bool attr = false;
  if (!attr) {
    FL_CUDA(cudaFuncSetAttribute(fused_kernel<RPT, W>, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_BUDGET));
    attr = true;
  }
  fused_kernel<RPT, W><<<op->nblocks, NT, smem, s>>>(*op, *vecs, st, it, mode, ldmax);
  FL_CHECK_LAUNCH();
  return FL_OK;
}

// (rows per thread, tile width) pairs: RPT = ceil(ldmax / NT) rounded up to an
// instantiated value, W = the widest tile whose 3-stage ring fits the budget
int fused(const fl_blockop* op, fl_lsqr_vecs* vecs, fl_lsqr_state* st, int64_t it, int mode, cudaStream_t s) {
  const int ldmax = (int)fl::round_up(op->max_rows > 0 ? op->max_rows : 1, 16);
  const int w = pick_w(ldmax);
  const int rpt = (ldmax + NT - 1) / NT;
#define FL_FUSED(R, WW) return launch_fused<R, WW>(op, vecs, st, it, mode, ldmax, s)
  if (w == 0) return FL_ERR_INVALID;
  if (rpt <= 1) FL_FUSED(1, 8);
  if (rpt <= 2) FL_FUSED(2, 8);
  if (rpt <= 3) { if (w >= 4) FL_FUSED(3, 4); FL_FUSED(3, 3); }
  if (rpt <= 4) { if (w >= 4) FL_FUSED(4, 4); if (w >= 3) FL_FUSED(4, 3); FL_FUSED(4, 2); }
  if (rpt <= 6) { if (w >= 3) FL_FUSED(6, 3); if (w >= 2) FL_FUSED(6, 2); FL_FUSED(6, 1); }
  if (rpt <= 8) { if (w >= 2) FL_FUSED(8, 2); FL_FUSED(8, 1); }
  FL_FUSED(12, 1);
#undef FL_FUSED
}

int row_grid(const fl_blockop* op) {
  const int64_t n = op->nrows > op->ncols_total ? op->nrows : op->ncols_total;
  int64_t g = (n + 255) / 256;
  if (g > 148 * 8) g = 148 * 8;
  return (int)(g < 1 ? 1 : g);
}

}  // namespace

namespace fl {
bool fused_ok(const fl_blockop* op) {
  return op->max_ncols <= VMAX && pick_w((int)round_up(op->max_rows > 0 ? op->max_rows : 1, 16)) > 0;
}
// init: caller has run lsqr_init_a (u = rhs, beta); this runs v' = Q^T u/beta, p = Q v'
int lsqr_fused_init(const fl_blockop* op, fl_lsqr_vecs* vecs, fl_lsqr_state* st, cudaStream_t s) {
  return fused(op, vecs, st, 0, 0, s);
}
int lsqr_fused_iterate(const fl_blockop* op, fl_lsqr_vecs* vecs, fl_lsqr_state* st, int64_t first_it,
                       int64_t count, cudaStream_t s) {
  const int rg = row_grid(op);
  for (int64_t k = 0; k < count; ++k) {
    const int64_t it = first_it + k;
    row_kernel<<<rg, 256, 0, s>>>(*op, *vecs, st, it);
    FL_CHECK_LAUNCH();
    int e = fused(op, vecs, st, it, 1, s);
    if (e) return e;
  }
  return FL_OK;
}
}  // namespace fl
