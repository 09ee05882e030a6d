// N4 — conjugate gradients on the normal equations, optionally with the
// additive-Schwarz block preconditioner (reference: solvers.py:150-239,
// the runner's "cg" / "as-cg" baselines, runner.py:296-305).
//
// The products M p and M^T (M p) are the block-operator kernels of qop.cu
// (HBM-bound streams of the raw blocks); the vector algebra, the two dot
// products and the scalar recurrences run in the small kernels below with a
// device-resident state, so the host enqueues the whole budget without
// synchronising. Semantics follow the reference line by line: breakdown when
// p.q <= 0 or non-finite (before the x update), DivergenceError on a
// non-finite x, the monitor's residual ||M x - rhs|| only at recorded
// iterations, breakdown when the old r.z is exactly 0.
//
// CG reuses fl_lsqr_state for loop control (it, done, breakdown, stride,
// best/best_it/improved, diverged_at, nonfinite); its scalars live in
// alpha = r.z, beta = p.q, phi = step, theta = r.z_next / r.z and
// phibar = the last recorded residual.
#include <float.h>

#include "common.cuh"

namespace {

constexpr int NT = 256;
constexpr int GMAX = 148 * 4;

__device__ __forceinline__ bool done_(const fl_lsqr_state* st) { return *(volatile const int32_t*)&st->done; }

int grid_for(int64_t n) {
  int64_t g = (n + NT - 1) / NT;
  if (g > GMAX) g = GMAX;
  return (int)(g < 1 ? 1 : g);
}

enum { DOT_PQ = 0, DOT_RZ_INIT = 1, DOT_RZ = 2 };

// a . b over n entries (fixed-order grid reduction); the last CTA applies
// the recurrence step `mode`
__global__ void __launch_bounds__(NT) dot_kernel(const double* __restrict__ a, const double* __restrict__ b,
                                                 int64_t n, fl_cg_vecs v, fl_lsqr_state* st, int mode) {
  if (mode != DOT_RZ_INIT && done_(st)) return;
  __shared__ double sh[NT / 32];
  double s = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)NT + threadIdx.x; i < n; i += (int64_t)gridDim.x * NT) s += a[i] * b[i];
  s = fl::block_sum(s, sh);
  double tot;
  if (!fl::grid_sum_last(s, v.scratch, v.counter, &tot, sh) || threadIdx.x != 0) return;
  if (mode == DOT_RZ_INIT) {
    st->alpha = tot;
  } else if (mode == DOT_PQ) {  // solvers.py:218-222
    st->beta = tot;
    if (tot <= 0.0 || !isfinite(tot)) {
      st->breakdown = 1;
      st->done = 1;
    } else {
      st->phi = st->alpha / tot;
    }
  } else {  // solvers.py:232-238
    if (st->alpha == 0.0) {
      st->breakdown = 1;
      st->done = 1;
    } else {
      st->theta = tot / st->alpha;
      st->alpha = tot;
    }
  }
}

// x += step p; r -= step q (solvers.py:223-228); the best-iterate copy of
// the previous recorded x is folded in (monitor.cu); the last CTA records
// the iteration and the divergence
__global__ void __launch_bounds__(NT) update_kernel(fl_cg_vecs v, int64_t n, fl_lsqr_state* st, int64_t it) {
  if (done_(st)) return;
  __shared__ int s_bad;
  __shared__ double sh[NT / 32];
  if (threadIdx.x == 0) s_bad = 0;
  __syncthreads();
  const double step = st->phi;
  const bool improve = *(volatile const int32_t*)&st->improved != 0;
  int bad = 0;
  for (int64_t i = blockIdx.x * (int64_t)NT + threadIdx.x; i < n; i += (int64_t)gridDim.x * NT) {
    const double xo = v.x[i];
    const double xn = xo + step * v.p[i];
    v.x[i] = xn;
    v.r[i] = v.r[i] - step * v.q[i];
    bad |= !isfinite(xn);
    if (improve) v.xbest[i] = xo;
  }
  if (bad) atomicOr(&s_bad, 1);
  __syncthreads();
  double tot;
  if (!fl::grid_sum_last(s_bad ? 1.0 : 0.0, v.scratch, v.counter, &tot, sh) || threadIdx.x != 0) return;
  st->it = it;
  st->improved = 0;  // every CTA has read it
  if (tot != 0.0) {
    st->diverged_at = it;
    st->done = 1;
  }
}

// residual ||M x - rhs|| of iteration `it` (tmp = M x); records it and, when
// no test-error monitor ranks the iterates, keeps the best by residual
// (solvers.py:59-69 with error = residual). it < 0: final residual -> out.
__global__ void __launch_bounds__(NT) residual_kernel(fl_cg_vecs v, int64_t nrows, fl_lsqr_state* st, int64_t it,
                                                      int by_residual, double* out) {
  if (it >= 0) {
    if (*(volatile const int64_t*)&st->it != it || *(volatile const int64_t*)&st->diverged_at) return;
    if (st->stride > 1 && it % st->stride != 0) return;
  }
  __shared__ double sh[NT / 32];
  double s = 0.0;
  for (int64_t g = blockIdx.x * (int64_t)NT + threadIdx.x; g < nrows; g += (int64_t)gridDim.x * NT) {
    const double d = v.tmp[g] - v.rhs[g];
    s += d * d;
  }
  s = fl::block_sum(s, sh);
  double tot;
  if (!fl::grid_sum_last(s, v.scratch, v.counter, &tot, sh) || threadIdx.x != 0) return;
  const double res = sqrt(tot);
  if (it < 0) {
    out[0] = res;
    return;
  }
  v.res_trace[it] = res;
  st->phibar = res;
  if (by_residual && res < st->best) {
    st->best = res;
    st->best_it = it;
    st->improved = 1;
  }
}

// z[idx_b] = inv_b r[idx_b] for every preconditioner block (row-major inv_b)
__global__ void __launch_bounds__(NT) precond_kernel(fl_block_precond pre, fl_cg_vecs v, const fl_lsqr_state* st,
                                                     int init) {
  if (!init && done_(st)) return;
  const int b = blockIdx.x;
  const int64_t i0 = pre.idx_off[b];
  const int sz = (int)(pre.idx_off[b + 1] - i0);
  const double* inv = pre.vals + pre.val_off[b];
  extern __shared__ double rs[];
  for (int k = threadIdx.x; k < sz; k += NT) rs[k] = v.r[pre.idx[i0 + k]];
  __syncthreads();
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  for (int row = wid; row < sz; row += NT / 32) {
    const double* ir = inv + (int64_t)row * sz;
    double s = 0.0;
    for (int k = lane; k < sz; k += 32) s += ir[k] * rs[k];
    s = fl::warp_sum(s);
    if (lane == 0) v.z[pre.idx[i0 + row]] = s;
  }
}

// p = z + theta p (solvers.py:237); init: p = z
__global__ void __launch_bounds__(NT) p_kernel(fl_cg_vecs v, int64_t n, const fl_lsqr_state* st, int init) {
  if (!init && done_(st)) return;
  const double beta = init ? 0.0 : st->theta;
  for (int64_t i = blockIdx.x * (int64_t)NT + threadIdx.x; i < n; i += (int64_t)gridDim.x * NT)
    v.p[i] = init ? v.z[i] : v.z[i] + beta * v.p[i];
}

int precond(const fl_block_precond* pre, fl_cg_vecs* v, const fl_lsqr_state* st, int init, cudaStream_t s) {
  if (!pre || pre->nblocks == 0) return FL_OK;
  const size_t smem = (size_t)(pre->max_size > 0 ? pre->max_size : 1) * sizeof(double);
  if (smem > 200 * 1024) return FL_ERR_INVALID;
  FL_CUDA(cudaFuncSetAttribute(precond_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  precond_kernel<<<pre->nblocks, NT, smem, s>>>(*pre, *v, st, init);
  FL_CHECK_LAUNCH();
  return FL_OK;
}

}  // namespace

namespace fl {
int monitor_step(const fl_test_monitor* mon, const double* x, fl_lsqr_state* st, int64_t it, cudaStream_t s);
}

extern "C" int fl_blockop_apply(const fl_blockop* op, const double* x, double* out, void* stream);
extern "C" int fl_blockop_apply_t(const fl_blockop* op, const double* r, double* out, void* stream);

extern "C" int fl_cg_init(const fl_blockop* op, fl_cg_vecs* v, const fl_block_precond* pre, fl_lsqr_state* st,
                          void* stream) {
  cudaStream_t s = (cudaStream_t)stream;
  const int64_t n = op->ncols_total;
  int e = fl_blockop_apply_t(op, v->rhs, v->r, stream);  // r = M^T rhs (solvers.py:209)
  if (e) return e;
  if ((e = precond(pre, v, st, 1, s))) return e;          // z = P r (or z = r: same buffer)
  p_kernel<<<grid_for(n), NT, 0, s>>>(*v, n, st, 1);
  FL_CHECK_LAUNCH();
  dot_kernel<<<grid_for(n), NT, 0, s>>>(v->r, v->z, n, *v, st, DOT_RZ_INIT);
  FL_CHECK_LAUNCH();
  return FL_OK;
}

extern "C" int fl_cg_iterate(const fl_blockop* op, fl_cg_vecs* v, const fl_block_precond* pre, fl_lsqr_state* st,
                             int64_t first_it, int64_t count, const fl_test_monitor* mon, void* stream) {
  cudaStream_t s = (cudaStream_t)stream;
  const int64_t n = op->ncols_total, N = op->nrows;
  const int gn = grid_for(n), gN = grid_for(N);
  int e;
  for (int64_t k = 0; k < count; ++k) {
    const int64_t it = first_it + k;
    if ((e = fl_blockop_apply(op, v->p, v->tmp, stream))) return e;    // q = M^T (M p)
    if ((e = fl_blockop_apply_t(op, v->tmp, v->q, stream))) return e;
    dot_kernel<<<gn, NT, 0, s>>>(v->p, v->q, n, *v, st, DOT_PQ);
    update_kernel<<<gn, NT, 0, s>>>(*v, n, st, it);
    FL_CHECK_LAUNCH();
    // monitor.observe at recorded iterations (the host knows the stride)
    const int32_t stride = v->stride > 1 ? v->stride : 1;  // host copy of st->stride
    if (stride <= 1 || it % stride == 0) {
      if ((e = fl_blockop_apply(op, v->x, v->tmp, stream))) return e;
      residual_kernel<<<gN, NT, 0, s>>>(*v, N, st, it, mon ? 0 : 1, nullptr);
      FL_CHECK_LAUNCH();
      if (mon && (e = fl::monitor_step(mon, v->x, st, it, s))) return e;
    }
    if ((e = precond(pre, v, st, 0, s))) return e;
    dot_kernel<<<gn, NT, 0, s>>>(v->r, v->z, n, *v, st, DOT_RZ);
    p_kernel<<<gn, NT, 0, s>>>(*v, n, st, 0);
    FL_CHECK_LAUNCH();
  }
  return FL_OK;
}

extern "C" int fl_block_precond_apply(const fl_block_precond* pre, const double* r, double* z, void* stream) {
  fl_cg_vecs v{};
  v.r = const_cast<double*>(r);
  v.z = z;
  return precond(pre, &v, nullptr, 1, (cudaStream_t)stream);
}

extern "C" int fl_cg_residual(const fl_blockop* op, fl_cg_vecs* v, double* out, void* stream) {
  int e = fl_blockop_apply(op, v->x, v->tmp, stream);
  if (e) return e;
  residual_kernel<<<grid_for(op->nrows), NT, 0, (cudaStream_t)stream>>>(*v, op->nrows, nullptr, -1, 0, out);
  FL_CHECK_LAUNCH();
  return FL_OK;
}
