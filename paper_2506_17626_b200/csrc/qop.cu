// K3/K4/K5 — block operator products, device-resident LSQR, recovery.
//
// K3 (reference filtering.py:146-157 CSR SpMV of PreconditionedOperator,
// assembly.py:91-104 for the raw system): the operator is stored as J dense
// column-major blocks (Q_j for the preconditioned operator, A_j for the raw
// one). Forward products write one partial value per (block, local row)
// and a fixed-order gather sums the covering blocks of every global row, so
// overlap rows are reduced deterministically (no fp64 atomics). Transposed
// products gather r[I_j] once per CTA into shared memory and reduce each
// column with a warp (disjoint outputs).
//
// K4 (solvers.py:87-145): the Golub-Kahan recurrences run on the device.
// Per iteration three kernels: qv (p = Q v, with v = v'/alpha and the w
// update of the previous iteration folded in), ured (u' = gather(p) -
// alpha u, ||u'||, then the scalar step rho/c/s/phi/phibar in the last CTA)
// and qtu (x += (phi/rho) w with the monitor's best-iterate copy, then
// v' = Q^T (u'/beta) - beta v, ||v'||, theta/rhobar in the last CTA). Every
// grid reduction is deposit-per-CTA + last-CTA fixed-order sum, so the whole
// loop is run-to-run bit-reproducible. Only scalars ever leave the device.
//
// K5 (filtering.py:169-183 -> linalg.py:100-112 dtrtrs): per-block
// column-oriented back substitution against R_j, scatter to kept columns.
#include <float.h>
#include <stdio.h>
#include <stdlib.h>

#include "common.cuh"

namespace fl {
bool fused_ok(const fl_blockop* op);
int lsqr_fused_init(const fl_blockop* op, fl_lsqr_vecs* vecs, fl_lsqr_state* st, cudaStream_t s);
int monitor_step(const fl_test_monitor* mon, const double* x, fl_lsqr_state* st, int64_t it, cudaStream_t s);
int lsqr_fused_iterate(const fl_blockop* op, fl_lsqr_vecs* vecs, fl_lsqr_state* st, int64_t first_it,
                       int64_t count, const fl_test_monitor* mon, cudaStream_t s);
}  // namespace fl

namespace {

constexpr int NT = 256;
constexpr int NW = NT / 32;
constexpr int RT = FL_ROW_TILE;   // rows per forward tile (one per thread)
constexpr int CT = FL_COL_TILE;   // columns per transposed tile

// ---------------------------------------------------------------- forward
// p[row_off_j + r] = sum_c B_j[r, c] * xs[c]; xs staged in shared memory.
__device__ __forceinline__ double row_dot(const double* __restrict__ Bj, int64_t ld, int r, int nc,
                                          const double* __restrict__ xs) {
  const double* p = Bj + r;
  double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
  int c = 0;
  for (; c + 4 <= nc; c += 4) {
    a0 += __ldg(p + (c + 0) * ld) * xs[c + 0];
    a1 += __ldg(p + (c + 1) * ld) * xs[c + 1];
    a2 += __ldg(p + (c + 2) * ld) * xs[c + 2];
    a3 += __ldg(p + (c + 3) * ld) * xs[c + 3];
  }
  for (; c < nc; ++c) a0 += __ldg(p + c * ld) * xs[c];
  return (a0 + a1) + (a2 + a3);
}

__global__ void __launch_bounds__(NT) fwd_kernel(fl_blockop op, const double* __restrict__ x) {
  extern __shared__ double xs[];
  const int j = op.row_tiles[2 * blockIdx.x];
  const int r0 = op.row_tiles[2 * blockIdx.x + 1];
  const int nc = op.ncols[j];
  const int64_t co = op.col_off[j];
  for (int c = threadIdx.x; c < nc; c += NT) xs[c] = x[co + c];
  __syncthreads();
  const int r = r0 + threadIdx.x;
  if (r < op.m[j]) op.partial[op.row_off[j] + r] = row_dot(op.vals + op.off[j], op.ld[j], r, nc, xs);
}

__global__ void __launch_bounds__(NT) gather_kernel(fl_blockop op, double* __restrict__ out) {
  const int g = blockIdx.x * NT + threadIdx.x;
  if (g >= op.nrows) return;
  double acc = 0.0;
  for (int e = op.gptr[g]; e < op.gptr[g + 1]; ++e) acc += op.partial[op.gsrc[e]];
  out[g] = acc;
}

// -------------------------------------------------------------- transposed
// out[col_off_j + c] = B_j[:, c] . rs, rs = r[rows_j] (optionally scaled).
// The first ns rows of rs are staged in shared memory (all m of them unless
// the block is taller than the staging buffer); rows past ns are gathered
// from src[rows[i]] / div as they are used.
__device__ __forceinline__ double col_dot(const double* __restrict__ col, int m, const double* __restrict__ rs,
                                          int lane, int ns, const double* __restrict__ src,
                                          const int32_t* __restrict__ rows, double div) {
  const int ms = m < ns ? m : ns;
  double a0 = 0.0, a1 = 0.0;
  int i = lane;
  for (; i + 32 < ms; i += 64) {
    a0 += __ldg(col + i) * rs[i];
    a1 += __ldg(col + i + 32) * rs[i + 32];
  }
  if (i < ms) a0 += __ldg(col + i) * rs[i];
  for (i = ms + lane; i < m; i += 32) a0 += __ldg(col + i) * (src[rows[i]] / div);
  return fl::warp_sum(a0 + a1);
}

__global__ void __launch_bounds__(NT) adj_kernel(fl_blockop op, const double* __restrict__ r,
                                                 double* __restrict__ out, int ns) {
  extern __shared__ double rs[];
  const int j = op.col_tiles[2 * blockIdx.x];
  const int c0 = op.col_tiles[2 * blockIdx.x + 1];
  const int m = op.m[j];
  const int32_t* rows = op.rows + op.row_off[j];
  for (int i = threadIdx.x; i < m && i < ns; i += NT) rs[i] = r[rows[i]];
  __syncthreads();
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int nc = op.ncols[j];
  const double* Bj = op.vals + op.off[j];
  const int64_t ld = op.ld[j];
  for (int c = c0 + wid; c < c0 + CT && c < nc; c += NW) {
    double d = col_dot(Bj + c * ld, m, rs, lane, ns, r, rows, 1.0);
    if (lane == 0) out[op.col_off[j] + c] = d;
  }
}

// ------------------------------------------------------------------- LSQR
__device__ __forceinline__ bool state_done(const fl_lsqr_state* st) { return *(volatile const int32_t*)&st->done; }

// it = iteration number being executed (1-based)
__global__ void __launch_bounds__(NT) lsqr_qv_kernel(fl_blockop op, fl_lsqr_vecs vec, fl_lsqr_state* st) {
  if (state_done(st)) return;
  extern __shared__ double xs[];
  const int j = op.row_tiles[2 * blockIdx.x];
  const int r0 = op.row_tiles[2 * blockIdx.x + 1];
  const int nc = op.ncols[j];
  const int64_t co = op.col_off[j];
  const double alpha = st->alpha;
  const double tr = st->theta / st->rho;
  const bool writer = (r0 == 0);
  for (int c = threadIdx.x; c < nc; c += NT) {
    const double vv = vec.vp[co + c] / alpha;  // v = v' / alpha   (solvers.py:141)
    xs[c] = vv;
    if (writer) {
      vec.v[co + c] = vv;
      vec.w[co + c] = vv - tr * vec.w[co + c];  // w = v - (theta/rho) w (solvers.py:144)
    }
  }
  __syncthreads();
  const int r = r0 + threadIdx.x;
  if (r < op.m[j]) op.partial[op.row_off[j] + r] = row_dot(op.vals + op.off[j], op.ld[j], r, nc, xs);
}

__global__ void __launch_bounds__(NT) lsqr_ured_kernel(fl_blockop op, fl_lsqr_vecs vec, fl_lsqr_state* st,
                                                       int64_t it) {
  if (state_done(st)) return;
  __shared__ double sh[NW];
  const int g = blockIdx.x * NT + threadIdx.x;
  const double alpha = st->alpha, bprev = st->beta_prev;
  double ss = 0.0;
  if (g < op.nrows) {
    double acc = 0.0;
    for (int e = op.gptr[g]; e < op.gptr[g + 1]; ++e) acc += op.partial[op.gsrc[e]];
    // u = Q v - alpha u with u = u_stored / beta_prev  (solvers.py:120)
    const double un = acc - alpha * (vec.u[g] / bprev);
    vec.u[g] = un;
    ss = un * un;
  }
  ss = fl::block_sum(ss, sh);
  double tot;
  if (fl::grid_sum_last(ss, op.red_scratch, op.counter, &tot, sh) && threadIdx.x == 0) {
    // solvers.py:121-127
    const double beta = sqrt(tot);
    const double rho = hypot(st->rhobar, beta);
    const double c = st->rhobar / rho, s = beta / rho;
    const double phi = c * st->phibar;
    st->beta = beta;
    if (beta > 0.0) st->beta_prev = beta;  // u is stored unnormalised; u/beta is the true u
    st->rho = rho;
    st->c = c;
    st->s = s;
    st->phi = phi;
    st->phibar = s * st->phibar;
    vec.trace[it] = st->phibar;
    if (st->use_rule) {  // scipy lsqr: anorm uses the previous alpha and the new beta
      st->anorm = sqrt(st->anorm * st->anorm + alpha * alpha + beta * beta);
    }
  }
}

__global__ void __launch_bounds__(NT) lsqr_qtu_kernel(fl_blockop op, fl_lsqr_vecs vec, fl_lsqr_state* st,
                                                      int64_t it, int ns) {
  if (state_done(st)) return;
  extern __shared__ double rs[];
  __shared__ double sh[NW];
  __shared__ int s_bad;
  const int j = op.col_tiles[2 * blockIdx.x];
  const int c0 = op.col_tiles[2 * blockIdx.x + 1];
  const int m = op.m[j];
  const int nc = op.ncols[j];
  const int64_t co = op.col_off[j];
  const double beta = st->beta;
  const double step = st->phi / st->rho;
  const double phibar = st->phibar;
  const bool record = (st->stride <= 1 || it % st->stride == 0);
  const bool mon = st->monitor;  // test-error monitor: copy the previous x when it was the best
  const bool improve = mon ? (*(volatile const int32_t*)&st->improved != 0) : (record && (phibar < st->best));
  if (threadIdx.x == 0) s_bad = 0;
  __syncthreads();
  // x = x + (phi/rho) w; finiteness; monitor best iterate (solvers.py:128-132, 59-69)
  double wss = 0.0;
  {
    int bad = 0;
    for (int c = c0 + threadIdx.x; c < c0 + CT && c < nc; c += NT) {
      const double wc = vec.w[co + c];
      const double xo = vec.x[co + c];
      const double xn = xo + step * wc;
      vec.x[co + c] = xn;
      bad |= !isfinite(xn);
      if (improve) vec.xbest[co + c] = mon ? xo : xn;
      wss += wc * wc;
    }
    if (bad) atomicOr(&s_bad, 1);
  }
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  double ass = 0.0;
  if (beta > 0.0) {
    const int32_t* rows = op.rows + op.row_off[j];
    for (int i = threadIdx.x; i < m && i < ns; i += NT) rs[i] = vec.u[rows[i]] / beta;  // u = u / beta (:123)
    __syncthreads();
    const double* Bj = op.vals + op.off[j];
    const int64_t ld = op.ld[j];
    for (int c = c0 + wid; c < c0 + CT && c < nc; c += NW) {
      const double d = col_dot(Bj + c * ld, m, rs, lane, ns, vec.u, rows, beta);
      if (lane == 0) {
        const double vn = d - beta * vec.v[co + c];  // v' = Q^T u - beta v (:136)
        vec.vp[co + c] = vn;
        ass += vn * vn;
      }
    }
  }
  __syncthreads();
  const int bad = s_bad;
  ass = fl::block_sum(ass, sh);
  wss = fl::block_sum(wss, sh);
  // deposit (ass, wss, bad) per CTA: pack into two slots
  double* slots = op.red_scratch;
  const int G = gridDim.x;
  __shared__ bool is_last;
  if (threadIdx.x == 0) {
    slots[blockIdx.x] = ass;
    slots[G + blockIdx.x] = wss;
    if (bad) atomicOr(&st->nonfinite, 1);
    __threadfence();
    unsigned int prev = atomicAdd(op.counter, 1u);
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
  a = fl::block_sum(a, sh);
  b = fl::block_sum(b, sh);
  if (threadIdx.x != 0) return;
  *op.counter = 0u;
  st->it = it;
  if (st->monitor) st->improved = 0;
  if (*(volatile int32_t*)&st->nonfinite) {  // DivergenceError("non-finite iterate at iteration it")
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
  const double alpha = sqrt(a);
  st->alpha = alpha;
  if (alpha == 0.0) {  // solvers.py:138-140
    st->breakdown = 1;
    st->done = 1;
    return;
  }
  st->theta = st->s * alpha;  // solvers.py:142-143
  st->rhobar = -st->c * alpha;
  if (st->use_rule) {
    // scipy.sparse.linalg.lsqr (damp = 0) stopping tests 1-3 on the same scalars
    const double rho = st->rho, theta = st->theta, phi = st->phi;
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

// init: u = rhs, beta = ||rhs|| (solvers.py:103-107)
__global__ void __launch_bounds__(NT) lsqr_init_a(fl_blockop op, const double* __restrict__ rhs, fl_lsqr_vecs vec,
                                                  fl_lsqr_state* st) {
  __shared__ double sh[NW];
  const int g = blockIdx.x * NT + threadIdx.x;
  double ss = 0.0;
  if (g < op.nrows) {
    const double h = rhs[g];
    vec.u[g] = h;
    if (vec.ub)
      for (int e = op.gptr[g]; e < op.gptr[g + 1]; ++e) vec.ub[op.gsrc[e]] = h;
    ss = h * h;
  }
  ss = fl::block_sum(ss, sh);
  double tot;
  if (fl::grid_sum_last(ss, op.red_scratch, op.counter, &tot, sh) && threadIdx.x == 0) {
    const double beta = sqrt(tot);
    st->beta = beta;
    st->beta_prev = beta;
    st->bnorm = beta;
    st->phibar = beta;
    if (beta == 0.0) st->done = 1;
  }
}

// init: v' = Q^T (rhs/beta), alpha = ||v'|| (solvers.py:108-117); x = w = 0
__global__ void __launch_bounds__(NT) lsqr_init_b(fl_blockop op, fl_lsqr_vecs vec, fl_lsqr_state* st, int ns) {
  if (state_done(st)) return;
  extern __shared__ double rs[];
  __shared__ double sh[NW];
  const int j = op.col_tiles[2 * blockIdx.x];
  const int c0 = op.col_tiles[2 * blockIdx.x + 1];
  const int m = op.m[j];
  const int nc = op.ncols[j];
  const int64_t co = op.col_off[j];
  const double beta = st->beta;
  const int32_t* rows = op.rows + op.row_off[j];
  for (int i = threadIdx.x; i < m && i < ns; i += NT) rs[i] = vec.u[rows[i]] / beta;
  for (int c = c0 + threadIdx.x; c < c0 + CT && c < nc; c += NT) {
    vec.x[co + c] = 0.0;
    vec.w[co + c] = 0.0;
    vec.xbest[co + c] = 0.0;
  }
  __syncthreads();
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  double ass = 0.0;
  const double* Bj = op.vals + op.off[j];
  const int64_t ld = op.ld[j];
  for (int c = c0 + wid; c < c0 + CT && c < nc; c += NW) {
    const double d = col_dot(Bj + c * ld, m, rs, lane, ns, vec.u, rows, beta);
    if (lane == 0) {
      vec.vp[co + c] = d;
      ass += d * d;
    }
  }
  ass = fl::block_sum(ass, sh);
  double tot;
  if (fl::grid_sum_last(ass, op.red_scratch, op.counter, &tot, sh) && threadIdx.x == 0) {
    const double alpha = sqrt(tot);
    st->alpha = alpha;
    st->rhobar = alpha;
    st->theta = 0.0;  // first qv: w = v - 0 * 0 = v (solvers.py:117)
    st->rho = 1.0;
    st->anorm = 0.0;
    st->ddnorm = 0.0;
    st->xxnorm = 0.0;
    st->z = 0.0;
    st->cs2 = -1.0;
    st->sn2 = 0.0;
    if (alpha == 0.0) {
      st->breakdown = 1;
      st->done = 1;
    }
  }
}

// ---------------------------------------------------------------- recovery
__global__ void __launch_bounds__(NT) backsub_kernel(int K, const double* __restrict__ R,
                                                     const int32_t* __restrict__ rank,
                                                     const int32_t* __restrict__ perm,
                                                     const int64_t* __restrict__ y_off,
                                                     const double* __restrict__ y, double* __restrict__ coeffs,
                                                     int32_t* singular) {
  extern __shared__ double sy[];
  const int j = blockIdx.x;
  const int r = rank[j];
  const double* Rj = R + (int64_t)j * K * K;
  // every column of block j starts at exactly 0 (dropped columns stay 0)
  for (int c = threadIdx.x; c < K; c += NT) coeffs[(int64_t)j * K + c] = 0.0;
  for (int t = threadIdx.x; t < r; t += NT) sy[t] = y[y_off[j] + t];
  __shared__ int s_sing;
  if (threadIdx.x == 0) s_sing = 0;
  __syncthreads();
  for (int t = threadIdx.x; t < r; t += NT)
    if (Rj[(int64_t)t * K + t] == 0.0) s_sing = 1;
  __syncthreads();
  if (s_sing) {
    if (threadIdx.x == 0) atomicMin(singular, j);
    return;
  }
  // column-oriented back substitution (dtrtrs/dtrsv upper, no-transpose)
  for (int t = r - 1; t >= 0; --t) {
    const double at = sy[t] / Rj[(int64_t)t * K + t];
    __syncthreads();
    if (threadIdx.x == 0) sy[t] = at;
    for (int i = threadIdx.x; i < t; i += NT) sy[i] -= at * Rj[(int64_t)t * K + i];
    __syncthreads();
  }
  for (int t = threadIdx.x; t < r; t += NT) coeffs[(int64_t)j * K + perm[(int64_t)j * K + t]] = sy[t];
}

}  // namespace

// ---------------------------------------------------------------- C-ABI

namespace {
int set_smem(const void* fn, size_t bytes) {
  if (bytes > 220 * 1024) return FL_ERR_INVALID;
  FL_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
  return FL_OK;
}
size_t col_smem(const fl_blockop* op) { return (size_t)(op->max_ncols > 0 ? op->max_ncols : 1) * sizeof(double); }
// rows of a block's vector staged in shared memory by the transposed kernels:
// all of them up to 200 KB, the rest gathered from global memory (col_dot)
constexpr size_t ROW_STAGE_MAX = 200 * 1024;
size_t row_smem(const fl_blockop* op) {
  const size_t b = (size_t)(op->max_rows > 0 ? op->max_rows : 1) * sizeof(double);
  return b < ROW_STAGE_MAX ? b : ROW_STAGE_MAX;
}
int row_staged(const fl_blockop* op) { return (int)(row_smem(op) / sizeof(double)); }
int grid_rows(const fl_blockop* op) { return (op->nrows + NT - 1) / NT; }
// one HBM pass per iteration (lsqr_fused.cu) unless a column tile does not fit
// on chip or FEATLSQ_LSQR=split asks for the two-pass kernels
bool use_fused(const fl_blockop* op) {
  const char* e = getenv("FEATLSQ_LSQR");
  if (e && e[0] == 's') return false;
  return fl::fused_ok(op);
}
}  // namespace

extern "C" int fl_blockop_apply(const fl_blockop* op, const double* x, double* out, void* stream) {
  cudaStream_t s = (cudaStream_t)stream;
  if (op->nrows == 0) return FL_OK;
  if (op->n_row_tiles > 0) {
    int e = set_smem((const void*)fwd_kernel, col_smem(op));
    if (e) return e;
    fwd_kernel<<<op->n_row_tiles, NT, col_smem(op), s>>>(*op, x);
    FL_CHECK_LAUNCH();
  }
  gather_kernel<<<grid_rows(op), NT, 0, s>>>(*op, out);
  FL_CHECK_LAUNCH();
  return FL_OK;
}

extern "C" int fl_blockop_apply_t(const fl_blockop* op, const double* r, double* out, void* stream) {
  if (op->n_col_tiles == 0) return FL_OK;
  int e = set_smem((const void*)adj_kernel, row_smem(op));
  if (e) return e;
  adj_kernel<<<op->n_col_tiles, NT, row_smem(op), (cudaStream_t)stream>>>(*op, r, out, row_staged(op));
  FL_CHECK_LAUNCH();
  return FL_OK;
}

extern "C" int fl_lsqr_init(const fl_blockop* op, const double* rhs, fl_lsqr_vecs* vecs, fl_lsqr_state* st,
                            void* stream) {
  cudaStream_t s = (cudaStream_t)stream;
  if (op->nrows == 0) return FL_ERR_INVALID;
  lsqr_init_a<<<grid_rows(op), NT, 0, s>>>(*op, rhs, *vecs, st);
  FL_CHECK_LAUNCH();
  if (op->n_col_tiles == 0) return FL_OK;
  if (use_fused(op)) return fl::lsqr_fused_init(op, vecs, st, s);
  int e = set_smem((const void*)lsqr_init_b, row_smem(op));
  if (e) return e;
  lsqr_init_b<<<op->n_col_tiles, NT, row_smem(op), s>>>(*op, *vecs, st, row_staged(op));
  FL_CHECK_LAUNCH();
  return FL_OK;
}

extern "C" int fl_lsqr_iterate_monitored(const fl_blockop* op, fl_lsqr_vecs* vecs, fl_lsqr_state* st,
                                         int64_t first_it, int64_t count, const fl_test_monitor* mon,
                                         void* stream) {
  cudaStream_t s = (cudaStream_t)stream;
  if (op->n_col_tiles == 0 || op->n_row_tiles == 0) return FL_ERR_INVALID;
  if (use_fused(op)) return fl::lsqr_fused_iterate(op, vecs, st, first_it, count, mon, s);
  int e = set_smem((const void*)lsqr_qv_kernel, col_smem(op));
  if (e) return e;
  e = set_smem((const void*)lsqr_qtu_kernel, row_smem(op));
  if (e) return e;
  for (int64_t k = 0; k < count; ++k) {
    const int64_t it = first_it + k;
    lsqr_qv_kernel<<<op->n_row_tiles, NT, col_smem(op), s>>>(*op, *vecs, st);
    lsqr_ured_kernel<<<grid_rows(op), NT, 0, s>>>(*op, *vecs, st, it);
    lsqr_qtu_kernel<<<op->n_col_tiles, NT, row_smem(op), s>>>(*op, *vecs, st, it, row_staged(op));
    if (mon && (e = fl::monitor_step(mon, vecs->x, st, it, s))) return e;
  }
  FL_CHECK_LAUNCH();
  return FL_OK;
}

extern "C" int fl_lsqr_iterate(const fl_blockop* op, fl_lsqr_vecs* vecs, fl_lsqr_state* st, int64_t first_it,
                               int64_t count, void* stream) {
  return fl_lsqr_iterate_monitored(op, vecs, st, first_it, count, nullptr, stream);
}

extern "C" int fl_backsub_scatter(int32_t nblocks, int32_t K, const double* R, const int32_t* rank,
                                  const int32_t* perm, const int64_t* y_off, const double* y, double* coeffs,
                                  int32_t* singular_block, void* stream) {
  if (nblocks == 0) return FL_OK;
  size_t smem = (size_t)K * sizeof(double);
  int e = set_smem((const void*)backsub_kernel, smem);
  if (e) return e;
  backsub_kernel<<<nblocks, NT, smem, (cudaStream_t)stream>>>(K, R, rank, perm, y_off, y, coeffs, singular_block);
  FL_CHECK_LAUNCH();
  return FL_OK;
}

extern "C" const char* fl_version(void) { return "featlsq_b200 0.1 sm_100a"; }

namespace {
thread_local char g_err[512] = "";
}
void fl::set_error(const char* file, int line, cudaError_t e) {
  snprintf(g_err, sizeof(g_err), "%s:%d: %s (%s)", file, line, cudaGetErrorName(e), cudaGetErrorString(e));
}
extern "C" const char* fl_last_error(void) { return g_err; }
