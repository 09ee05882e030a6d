// K6 — device test-lattice monitor (reference: runner.py:265-276
// `_error_matrix`, assembly.py:313-318 `l1_error`, solvers.py:59-69
// `ConvergenceMonitor.observe`).
//
// The runner evaluates the test-lattice L1 error of every recorded LSQR
// iterate y through T = P[:, kept] S^{-1} (P = solution blocks at the test
// points, S = blockdiag R_j) and keeps the iterate with the lowest error.
// Here T lives in HBM as per-block dense blocks over the test-point layout
// (built once by tbuild_kernel), and each recorded iteration costs one
// streaming pass over T (mon_fwd_kernel, HBM-bound: 8 B per T entry) plus a
// fixed-order gather/|.|/sum (mon_err_kernel) whose last CTA updates the
// best error. The x -> x_best copy is folded into the next iteration's
// x update (lsqr_fused.cu / qop.cu), so no extra pass over y is needed.
#include "common.cuh"

namespace {

constexpr int NT = 256;
constexpr int TB = FL_TBUILD_ROWS;  // rows per T-build CTA (one 16-lane group per row)

// solvers.py:59-61: the iterate of iteration `it` exists (not diverged, not
// past the end of the loop) and falls on the stride; it < 0 = direct call
__device__ __forceinline__ bool recorded(const fl_lsqr_state* st, int64_t it) {
  if (it < 0) return true;
  if (*(volatile const int64_t*)&st->it != it || *(volatile const int64_t*)&st->diverged_at) return false;
  return st->stride <= 1 || it % st->stride == 0;
}

// T_j[i, c] = (P_j[i, perm_j[c]] - sum_{k<c} T_j[i, k] R_j[k, c]) / R_j[c, c]
__global__ void __launch_bounds__(NT) tbuild_kernel(fl_blockop P, const double* __restrict__ R,
                                                    const int32_t* __restrict__ perm, int K, fl_blockop T,
                                                    const int32_t* __restrict__ tiles) {
  extern __shared__ double tsm[];  // [TB][K]
  const int j = tiles[2 * blockIdx.x], r0 = tiles[2 * blockIdx.x + 1];
  const int m = P.m[j], ld = P.ld[j], r = T.ncols[j];
  const int grp = threadIdx.x >> 4, l = threadIdx.x & 15;
  const int row = r0 + grp;
  const bool ok = row < m;
  const double* Rj = R + (int64_t)j * K * K;
  const int32_t* pj = perm + (int64_t)j * K;
  const double* Pj = P.vals + P.off[j];
  double* tr = tsm + grp * K;
  for (int c = 0; c < r; ++c) {
    const double* Rc = Rj + (int64_t)c * K;
    const double pv = (l == 0 && ok) ? Pj[(int64_t)pj[c] * ld + row] : 0.0;
    double s = 0.0;
    for (int k = l; k < c; k += 16) s += tr[k] * Rc[k];
#pragma unroll
    for (int o = 8; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (l == 0) tr[c] = ok ? (pv - s) / Rc[c] : 0.0;
    __syncwarp();
  }
  if (!ok) return;
  double* Tj = const_cast<double*>(T.vals) + T.off[j];  // T is the output store
  for (int c = l; c < r; c += 16) Tj[(int64_t)c * ld + row] = tr[c];
}

// partial[row_off_j + r] = T_j[r, :] . x_j
__global__ void __launch_bounds__(NT) mon_fwd_kernel(fl_blockop T, const double* __restrict__ x,
                                                     const fl_lsqr_state* st, int64_t it) {
  if (!recorded(st, it)) return;
  extern __shared__ double xs[];
  const int j = T.row_tiles[2 * blockIdx.x], r0 = T.row_tiles[2 * blockIdx.x + 1];
  const int nc = T.ncols[j];
  const int64_t co = T.col_off[j];
  for (int c = threadIdx.x; c < nc; c += NT) xs[c] = x[co + c];
  __syncthreads();
  const int r = r0 + threadIdx.x;
  if (r >= T.m[j]) return;
  const double* p = T.vals + T.off[j] + r;
  const int64_t ld = T.ld[j];
  double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
  int c = 0;
  for (; c + 4 <= nc; c += 4) {
    a0 += __ldg(p + (c + 0) * ld) * xs[c + 0];
    a1 += __ldg(p + (c + 1) * ld) * xs[c + 1];
    a2 += __ldg(p + (c + 2) * ld) * xs[c + 2];
    a3 += __ldg(p + (c + 3) * ld) * xs[c + 3];
  }
  for (; c < nc; ++c) a0 += __ldg(p + c * ld) * xs[c];
  T.partial[T.row_off[j] + r] = (a0 + a1) + (a2 + a3);
}

// e = mean |T y + lift - truth| / spread (assembly.py:313-318); the last CTA
// records it and updates the best (solvers.py:62-69: strict <)
__global__ void __launch_bounds__(NT) mon_err_kernel(fl_test_monitor mon, fl_lsqr_state* st, int64_t it) {
  if (!recorded(st, it)) return;
  __shared__ double sh[NT / 32];
  const fl_blockop& T = mon.T;
  double s = 0.0;
  for (int g = blockIdx.x * NT + threadIdx.x; g < T.nrows; g += gridDim.x * NT) {
    double acc = 0.0;
    for (int e = T.gptr[g]; e < T.gptr[g + 1]; ++e) acc += T.partial[T.gsrc[e]];
    s += fabs((acc + mon.lift[g]) - mon.truth[g]);
  }
  s = fl::block_sum(s, sh);
  double tot;
  if (fl::grid_sum_last(s, T.red_scratch, T.counter, &tot, sh) && threadIdx.x == 0) {
    const double e = (tot / (double)T.nrows) / mon.spread;
    if (it < 0) {
      mon.result[0] = e;
      return;
    }
    mon.err_trace[it] = e;
    if (e < st->best) {
      st->best = e;
      st->best_it = it;
      st->improved = 1;
    }
  }
}

__global__ void __launch_bounds__(NT) flush_kernel(fl_lsqr_vecs vec, const fl_lsqr_state* st, int64_t n) {
  if (!st->monitor || !*(volatile const int32_t*)&st->improved) return;
  for (int64_t c = blockIdx.x * (int64_t)NT + threadIdx.x; c < n; c += (int64_t)gridDim.x * NT)
    vec.xbest[c] = vec.x[c];
}

int err_grid(const fl_blockop& T) {
  int g = (T.nrows + NT - 1) / NT;
  if (g > 148 * 4) g = 148 * 4;
  return g < 1 ? 1 : g;
}

}  // namespace

namespace fl {
// one recorded-iteration evaluation of the monitor (no-op on the device when
// iteration `it` is not recorded)
int monitor_step(const fl_test_monitor* mon, const double* x, fl_lsqr_state* st, int64_t it, cudaStream_t s) {
  const fl_blockop& T = mon->T;
  if (T.nrows == 0) return FL_ERR_INVALID;
  if (T.n_row_tiles > 0) {
    const size_t smem = (size_t)(T.max_ncols > 0 ? T.max_ncols : 1) * sizeof(double);
    mon_fwd_kernel<<<T.n_row_tiles, NT, smem, s>>>(T, x, st, it);
    FL_CHECK_LAUNCH();
  }
  mon_err_kernel<<<err_grid(T), NT, 0, s>>>(*mon, st, it);
  FL_CHECK_LAUNCH();
  return FL_OK;
}
}  // namespace fl

extern "C" int fl_error_blocks(const fl_blockop* P, const double* R, const int32_t* perm, int32_t K,
                               const fl_blockop* T, int32_t n_tiles, const int32_t* tiles, void* stream) {
  if (n_tiles == 0) return FL_OK;
  if (K <= 0) return FL_ERR_INVALID;
  const size_t smem = (size_t)TB * K * sizeof(double);
  if (smem > 200 * 1024) return FL_ERR_INVALID;
  FL_CUDA(cudaFuncSetAttribute(tbuild_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  tbuild_kernel<<<n_tiles, NT, smem, (cudaStream_t)stream>>>(*P, R, perm, K, *T, tiles);
  FL_CHECK_LAUNCH();
  return FL_OK;
}

extern "C" int fl_monitor_error(const fl_test_monitor* mon, const double* y, void* stream) {
  return fl::monitor_step(mon, y, nullptr, -1, (cudaStream_t)stream);
}

extern "C" int fl_lsqr_monitor_flush(const fl_blockop* op, fl_lsqr_vecs* vecs, fl_lsqr_state* st, void* stream) {
  const int64_t n = op->ncols_total;
  if (n <= 0) return FL_OK;
  int64_t g = (n + NT - 1) / NT;
  if (g > 148 * 8) g = 148 * 8;
  flush_kernel<<<(int)g, NT, 0, (cudaStream_t)stream>>>(*vecs, st, n);
  FL_CHECK_LAUNCH();
  return FL_OK;
}
