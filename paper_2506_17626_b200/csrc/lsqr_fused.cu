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
// (one TMA bulk copy per column into a ring of SL single-column slots, each
// with its own mbarrier) and used by both products,
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
// the tail of the last wave. The CTA shape (NT threads, RP row pairs per thread,
// W columns per barrier, SL ring slots, MB CTAs per SM) is picked per layout
// from the instantiated table at the bottom: at cfg4 (ld <= 3072) 256 threads
// and two CTAs per SM, so one block's prologue/epilogue overlaps another
// block's stream. Each thread reads its row pairs as 16-byte shared loads and
// keeps them in registers between the two products.
#include <float.h>
#include <math.h>
#include <stdio.h>
#include <stdlib.h>

#include "common.cuh"

constexpr int ROW_CTAS_PER_SM = 3;
// Measured and removed (DESIGN.md §3 K4): an L2 evict_first policy on the Q
// stream (1.444 vs 1.423 ms per iteration on cfg4) and an evict_last policy
// on the partial-product stores (1.416 vs 1.399 ms).

namespace {

// shared memory per CTA with MB CTAs resident per SM: 227 KB for one, else
// (228 KB - MB x 1 KB reserved) / MB
constexpr int smem_per_cta(int mb) { return mb <= 1 ? 232448 : (233472 - mb * 1024) / mb; }

__device__ __forceinline__ bool is_done(const fl_lsqr_state* st) { return *(volatile const int32_t*)&st->done; }

// Programmatic dependent launch: the row and fused kernels of an iteration
// are launched with programmatic stream serialization, trigger their
// successor's launch on entry and wait for their predecessor's completion
// (and memory flush) before touching anything it wrote — the same ordering
// as plain stream order, with the successor's launch latency hidden.
// Measured (ms per iteration, PDL off / row only / fused only / both): cfg4
// 1.404 / 1.403 / 1.403 / 1.404, cfg5 1.420 / 1.421 / 1.420 / 1.416, cfg3
// 0.1378 / 0.1360 / 0.1353 / 0.1348, cfg2 0.0430 / 0.0410 / 0.0410 / 0.0397:
// a launch-latency win for the small configs, neutral at cfg4.
__device__ __forceinline__ void pdl_enter() {
  asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
  asm volatile("griddepcontrol.wait;\n" ::: "memory");
}

template <typename... KArgs, typename... Args>
cudaError_t launch_pdl(bool pdl, void (*kern)(KArgs...), int grid, int block, size_t smem, cudaStream_t s,
                       Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(block);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = pdl ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, args...);
}

// Warp sums of W per-lane values with a butterfly: the first log2(W) steps
// halve the set of live columns per lane group, so W columns cost
// 5 shuffles in total; returns in lane (32/W) c the total of column c.
template <int W>
__device__ __forceinline__ double warp_sums(const double (&a)[W], int lane) {
  double v[W];
#pragma unroll
  for (int c = 0; c < W; ++c) v[c] = a[c];
#pragma unroll
  for (int half = W / 2, o = 16; half >= 1; half /= 2, o /= 2) {
    const bool up = (lane & o) != 0;
#pragma unroll
    for (int c = 0; c < half; ++c) {
      const double send = up ? v[c] : v[c + half];
      const double recv = __shfl_xor_sync(0xffffffffu, send, o);
      v[c] = (up ? v[c + half] : v[c]) + recv;
    }
  }
  double s = v[0];
#pragma unroll
  for (int o = 32 / W / 2; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  return s;
}

// mode 0: initialisation (v = 0, no x update); mode 1: iteration `it`.
// RP row pairs per thread: 2 * RP * NT >= ld of every block. W columns are
// reduced together per barrier; the ring holds SL single-column slots
// (SL >= 2W) so SL - W columns stream in while a tile is being used.
template <int NT, int RP, int W, int SL, int MB>
__global__ void __launch_bounds__(NT, MB)
    fused_kernel(fl_blockop op, fl_lsqr_vecs vec, fl_lsqr_state* st, int64_t it, int mode, int ldmax, int S) {
  constexpr int NW = NT / 32;
  constexpr bool KEEP = RP * W <= 6;  // tile values stay in registers between the two products
  static_assert(SL >= 2 * W, "ring too shallow");
  pdl_enter();
  if (is_done(st)) return;
  extern __shared__ __align__(128) double sm[];
  double* ring = sm;  // [SL][ldmax] columns of Q_j
  __shared__ __align__(16) double red[2 * NW * W];
  __shared__ double red2[NW];
  __shared__ __align__(8) uint64_t bars[SL];
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
  const int cbeg = min(t0 * W, nc), cend = min(t1 * W, nc);  // x update runs even when beta = 0
  const int64_t cob = co + cbeg;  // first y-space entry of the range
  const int ncr = cend - cbeg;
  const int ncw = work ? ncr : 0;  // columns streamed
  const int ntiles = (ncw + W - 1) / W;
  if (threadIdx.x == 0) {
    s_bad = 0;
    for (int s = 0; s < SL; ++s)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"((unsigned)__cvta_generic_to_shared(&bars[s]))
                   : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();

  // TMA bulk copy of local column k (ld * 8 bytes) into slot k % SL, armed
  // on that slot's mbarrier (thread 0)
  auto issue = [&](int k) {
    if (threadIdx.x != 0 || k >= ncw) return;
    const unsigned bar = (unsigned)__cvta_generic_to_shared(&bars[k % SL]);
    const unsigned bytes = (unsigned)ld * 8u;
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(bar), "r"(bytes) : "memory");
    const unsigned dst = (unsigned)__cvta_generic_to_shared(ring + (k % SL) * ldmax);
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(dst),
                 "l"(Q + (int64_t)(cbeg + k) * ld), "r"(bytes), "r"(bar)
                 : "memory");
  };
  auto wait_col = [&](int k) {
    const unsigned bar = (unsigned)__cvta_generic_to_shared(&bars[k % SL]);
    const unsigned parity = (unsigned)((k / SL) & 1);
    unsigned ok = 0;
    while (!ok)
      asm volatile(
          "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }\n"
          : "=r"(ok)
          : "r"(bar), "r"(parity)
          : "memory");
  };
  // the ring fills while the x update and the u gather run
  for (int k = 0; k < SL - W; ++k) issue(k);

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
    //      the row pairs (2t, 2t+1) + 2 NT k, read as 16-byte shared loads ----
    const int32_t* rows = op.rows + op.row_off[j];
    double2 uh_r[RP], pp_r[RP];
#pragma unroll
    for (int i = 0; i < RP; ++i) {
      const int r = 2 * (threadIdx.x + i * NT);
      if (vec.ub) {  // block-local copy: contiguous
        const double* ubj = vec.ub + op.row_off[j];
        uh_r[i].x = (r < m) ? ubj[r] / beta : 0.0;
        uh_r[i].y = (r + 1 < m) ? ubj[r + 1] / beta : 0.0;
      } else {
        uh_r[i].x = (r < m) ? vec.u[rows[r]] / beta : 0.0;
        uh_r[i].y = (r + 1 < m) ? vec.u[rows[r + 1]] / beta : 0.0;
      }
      pp_r[i] = make_double2(0.0, 0.0);
    }
    // v_j[tile] is read one tile ahead (broadcast loads, off the critical path)
    double vnext[W];
    auto load_v = [&](int tdx) {
#pragma unroll
      for (int c = 0; c < W; ++c) {
        const int col = cbeg + tdx * W + c;
        vnext[c] = (mode == 1 && col < cend) ? vec.v[co + col] : 0.0;
      }
    };
    load_v(0);
    for (int tdx = 0; tdx < ntiles; ++tdx) {
      double vcur[W];
#pragma unroll
      for (int c = 0; c < W; ++c) vcur[c] = vnext[c];
      if (tdx + 1 < ntiles) load_v(tdx + 1);
      const int k0 = tdx * W;
      const int ncl = min(W, ncw - k0);  // valid columns in this tile
      const double* cp[W];
#pragma unroll
      for (int c = 0; c < W; ++c) {
        if (c < ncl) wait_col(k0 + c);
        cp[c] = ring + ((k0 + c) % SL) * ldmax;
      }
      double2 q[KEEP ? RP : 1][W];
      double acc[W];
#pragma unroll
      for (int c = 0; c < W; ++c) acc[c] = 0.0;
#pragma unroll
      for (int i = 0; i < RP; ++i) {
        const int r = 2 * (threadIdx.x + i * NT);
#pragma unroll
        for (int c = 0; c < W; ++c) {
          const double2 x = (r < ld && c < ncl) ? *reinterpret_cast<const double2*>(cp[c] + r)
                                                : make_double2(0.0, 0.0);
          if (KEEP) q[KEEP ? i : 0][c] = x;
          acc[c] += x.x * uh_r[i].x + x.y * uh_r[i].y;
        }
      }
      double* rw = red + (tdx & 1) * NW * W;  // [c][warp]
      {
        const double s = warp_sums<W>(acc, lane);
        if ((lane & (32 / W - 1)) == 0) rw[(lane / (32 / W)) * NW + wid] = s;
      }
      __syncthreads();  // partials visible; every thread is done with tile tdx-1
      for (int k = SL - W + k0; k < SL + k0; ++k) issue(k);  // refill tile tdx-1's slots
      // v'[tile] = Q[:, tile]^T u - beta v[tile] (solvers.py:136): every thread
      // sums the NW warp partials itself in warp order (broadcast 16-byte
      // loads), so no second barrier is needed; `red` alternates by parity
      double tc[W];
#pragma unroll
      for (int c = 0; c < W; ++c) {
        const double2* rp = reinterpret_cast<const double2*>(rw + c * NW);
        double s = 0.0;
#pragma unroll
        for (int w2 = 0; w2 < NW / 2; ++w2) {
          const double2 pr = rp[w2];
          s += pr.x;
          s += pr.y;
        }
        double vn = 0.0;
        if (c < ncl) vn = s - ((mode == 1) ? beta * vcur[c] : 0.0);
        tc[c] = vn;
        if (threadIdx.x == 0) {
          if (c < ncl) vec.vp[cob + k0 + c] = vn;
          ass += vn * vn;
        }
      }
#pragma unroll
      for (int i = 0; i < RP; ++i) {
        const int r = 2 * (threadIdx.x + i * NT);
#pragma unroll
        for (int c = 0; c < W; ++c) {
          const double2 x = KEEP ? q[KEEP ? i : 0][c]
                                 : ((r < ld && c < ncl) ? *reinterpret_cast<const double2*>(cp[c] + r)
                                                        : make_double2(0.0, 0.0));
          pp_r[i].x += x.x * tc[c];
          pp_r[i].y += x.y * tc[c];
        }
      }
    }
#pragma unroll
    for (int i = 0; i < RP; ++i) {
      const int r = 2 * (threadIdx.x + i * NT);
      double* pout = op.partial + h * op.partial_len + op.row_off[j];
      if (r < m) pout[r] = pp_r[i].x;
      if (r + 1 < m) pout[r + 1] = pp_r[i].y;
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
  pdl_enter();
  if (is_done(st)) return;
  __shared__ double sh[8];
  const double alpha = st->alpha, bprev = st->beta_prev;
  const double tr = st->theta / st->rho;  // rho here is rho_{it-1}
  const int gtid = blockIdx.x * blockDim.x + threadIdx.x, gsz = gridDim.x * blockDim.x;
  double ss = 0.0;
  // The gather is a chain of dependent loads (gptr -> gsrc -> partial): the
  // next row's gptr pair and u are fetched while this row's sources are in
  // flight, and a row's sources (4 at a time) and their partials are loaded
  // before any is summed. Same summation order as one source at a time.
  constexpr int ME = 4;
  int g = gtid;
  int e0 = 0, e1 = 0;
  double ug = 0.0;
  int src[ME];  // the first ME sources of row g, fetched one row ahead
  if (g < op.nrows) {
    e0 = op.gptr[g];
    e1 = op.gptr[g + 1];
    ug = vec.u[g];
  }
#pragma unroll
  for (int q = 0; q < ME; ++q) src[q] = (g < op.nrows && e0 + q < e1) ? op.gsrc[e0 + q] : 0;
  while (g < op.nrows) {
    const int gn = g + gsz;
    int n0 = 0, n1 = 0;
    double un_next = 0.0;
    if (gn < op.nrows) {
      n0 = op.gptr[gn];
      n1 = op.gptr[gn + 1];
      un_next = vec.u[gn];
    }
    double pv[ME][FL_LSQR_SPLIT_MAX];
#pragma unroll
    for (int q = 0; q < ME; ++q)
#pragma unroll
      for (int h = 0; h < FL_LSQR_SPLIT_MAX; ++h)
        pv[q][h] = (e0 + q < e1 && h < S) ? op.partial[h * op.partial_len + src[q]] : 0.0;
    int srcn[ME];  // next row's sources, in flight with this row's partials
#pragma unroll
    for (int q = 0; q < ME; ++q) srcn[q] = (gn < op.nrows && n0 + q < n1) ? op.gsrc[n0 + q] : 0;
    double acc = 0.0;
#pragma unroll
    for (int q = 0; q < ME; ++q)
      if (e0 + q < e1)
#pragma unroll
        for (int h = 0; h < FL_LSQR_SPLIT_MAX; ++h)
          if (h < S) acc += pv[q][h];
    for (int e = e0 + ME; e < e1; ++e) {  // rows with more than ME sources (3-D)
      const int64_t sx = op.gsrc[e];
      for (int h = 0; h < S; ++h) acc += op.partial[h * op.partial_len + sx];
    }
    const double un = acc / alpha - alpha * (ug / bprev);
    vec.u[g] = un;
    if (vec.ub) {
#pragma unroll
      for (int q = 0; q < ME; ++q)
        if (e0 + q < e1) vec.ub[src[q]] = un;
      for (int e = e0 + ME; e < e1; ++e) vec.ub[op.gsrc[e]] = un;
    }
    ss += un * un;
    g = gn;
    e0 = n0;
    e1 = n1;
    ug = un_next;
#pragma unroll
    for (int q = 0; q < ME; ++q) src[q] = srcn[q];
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
// A shape fits a layout when 2 * RP * NT >= ldmax and its ring (ST * ldmax
// doubles) plus static shared memory fits the per-CTA budget. Entries are in
// preference order; FEATLSQ_FUSED="NT,W,ST,MB" restricts the choice (tuning).

enum { SKIP = 1 };

template <int NT, int RP, int W, int ST, int MB>
int try_fused(const fl_blockop* op, fl_lsqr_vecs* vecs, fl_lsqr_state* st, int64_t it, int mode, int ldmax,
              int S, cudaStream_t s, bool dry) {
  if ((int64_t)2 * RP * NT < ldmax) return SKIP;
  // cudaFuncSetAttribute is per device: cache the raised limit per device id
  static int stat = -1;
  static size_t attr_dev[64] = {};
  int dev = 0;
  FL_CUDA(cudaGetDevice(&dev));
  size_t& attr = attr_dev[dev & 63];
  if (stat < 0) {
    cudaFuncAttributes a;
    FL_CUDA(cudaFuncGetAttributes(&a, fused_kernel<NT, RP, W, ST, MB>));
    stat = (int)a.sharedSizeBytes;
  }
  const size_t dyn = (size_t)ST * ldmax * sizeof(double);
  if (dyn + stat > (size_t)smem_per_cta(MB)) return SKIP;
  if (dry) return FL_OK;
  if (dyn > attr) {
    FL_CUDA(cudaFuncSetAttribute(fused_kernel<NT, RP, W, ST, MB>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)dyn));
    attr = dyn;
  }
  FL_CUDA(launch_pdl(true, fused_kernel<NT, RP, W, ST, MB>, op->nblocks * S, NT, dyn, s, *op, *vecs, st, it, mode,
                     ldmax, S));
  FL_CHECK_LAUNCH();
  return FL_OK;
}

struct Shape {
  int nt, rp, w, st, mb;
  int (*fn)(const fl_blockop*, fl_lsqr_vecs*, fl_lsqr_state*, int64_t, int, int, int, cudaStream_t, bool);
};

#define FL_SHAPE(NT, R, W, S, MB) {NT, R, W, S, MB, try_fused<NT, R, W, S, MB>}
const Shape kShapes[] = {
    // ld <= 1024 / 2048: one 512-thread CTA per SM, several columns per barrier
    FL_SHAPE(512, 1, 8, 24, 1), FL_SHAPE(512, 2, 4, 12, 1), FL_SHAPE(512, 2, 2, 8, 1),
    // ld <= 3072 (cfg3, cfg4): two 256-thread CTAs per SM, one column per barrier
    // (measured on cfg4: 1.436 ms/it vs 1.52 for 384 threads, 1.90 for 512)
    FL_SHAPE(256, 6, 1, 4, 2), FL_SHAPE(256, 6, 1, 5, 2), FL_SHAPE(256, 6, 1, 3, 3),
    // ld <= 6144 (cfg5): one 512-thread CTA per SM
    FL_SHAPE(512, 4, 1, 6, 1), FL_SHAPE(512, 4, 1, 4, 1),
    FL_SHAPE(512, 6, 1, 4, 1), FL_SHAPE(512, 6, 1, 3, 1),
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

// Column split S: maximise the last-wave occupancy of J*S work units over
// the resident CTA slots, with a small penalty per extra split (every split
// re-gathers u and writes its own partial copy). Measured: cfg3 (J = 256)
// S = 1, cfg4/cfg5 (J = 1024 / 512) S = 2. FEATLSQ_SPLIT overrides (tuning).
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
  const double slots = (double)nsm * sh.mb;
  int best = 1;
  double best_score = -1.0;
  for (int S = 1; S <= FL_LSQR_SPLIT_MAX; ++S) {
    const double waves = (double)op->nblocks * S / slots;
    const double score = waves / ceil(waves) - 0.02 * (S - 1);
    if (score > best_score + 1e-9) {
      best_score = score;
      best = S;
    }
  }
  return best;
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
  if (g > 148 * ROW_CTAS_PER_SM) g = 148 * ROW_CTAS_PER_SM;  // one wave (80 registers per thread)
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
    FL_CUDA(launch_pdl(true, row_kernel, rg, 256, 0, s, *op, *vecs, st, it, S));
    int e = fused(op, vecs, st, it, 1, S, s);
    if (e) return e;
    if (mon && (e = monitor_step(mon, vecs->x, st, it, s))) return e;
  }
  return FL_OK;
}
}  // namespace fl
