/*
 * featlsq_b200.h — C-ABI of the B200-native RRQR-filtered ELM-FBPINN
 * least-squares hot path (arXiv 2506.17626, reference package `featlsq`).
 *
 * Plain C: device pointers, int32/int64 sizes, an opaque CUDA stream handle
 * (`void*`, a cudaStream_t; NULL = legacy default stream). No allocation of
 * caller-visible memory happens inside the library; every call is stream
 * ordered and reentrant (no global mutable state). Return value 0 = OK,
 * negative = one of FL_ERR_* below, mapped 1:1 by the host layer onto the
 * reference exceptions (`featlsq/errors.py:4-41`).
 *
 * Entry point -> reference interface it replaces (reference tree
 * pkg/src/featlsq/):
 *   fl_assemble            assembly.py:124-238 `assemble` per-block loop
 *                          (+ domains.py:109-173 window jets, basis.py:106-133
 *                          feature jets, assembly.py:107-114, problems.py:39-47)
 *   fl_rrqr                filtering.py:92-115 `filter_system` ->
 *                          linalg.py:58-97 `qr_column_pivot` (dgeqp3+dorgqr)
 *   fl_blockop_apply       filtering.py:146-150 PreconditionedOperator.apply,
 *                          assembly.py:91-96 `apply`
 *   fl_blockop_apply_t     filtering.py:152-157 apply_transpose,
 *                          assembly.py:99-104 `apply_transpose`
 *   fl_lsqr_*              solvers.py:87-145 `lsqr` (device-resident loop)
 *   fl_backsub_scatter     filtering.py:169-183 `recover_solution` ->
 *                          linalg.py:100-112 `back_substitute` (dtrtrs)
 */
#ifndef FEATLSQ_B200_H
#define FEATLSQ_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* error codes */
#define FL_OK                    0
#define FL_ERR_INVALID         (-1)  /* InvalidInputError */
#define FL_ERR_DEGENERATE      (-2)  /* DegenerateSubdomainError (see fl_rrqr out-param) */
#define FL_ERR_DIVERGENCE      (-3)  /* DivergenceError (see fl_lsqr_state.diverged_at) */
#define FL_ERR_SINGULAR        (-4)  /* SingularFactorError */
#define FL_ERR_CUDA            (-5)  /* launch / runtime failure */

/* activations (basis.py:36-40) */
#define FL_ACT_TANH    0
#define FL_ACT_SIN     1
#define FL_ACT_SIGMOID 2

/* ------------------------------------------------------------------------
 * Block store: J per-subdomain dense blocks, each column-major with leading
 * dimension ld[j] (multiple of 16 doubles, zero padded), concatenated at
 * element offsets off[j]. Block j has m[j] rows (global ids rows[row_off[j]
 * .. row_off[j]+m[j])) and ncols[j] columns mapped to the y-space entries
 * col_off[j] .. col_off[j]+ncols[j]. The same layout carries the raw blocks
 * A_j (ncols = K, col_off = j*K) and the orthonormal blocks Q_j (ncols = r_j,
 * col_off = prefix sums of r_j). `gptr/gsrc` is the row-gather map: for
 * global row g, gsrc[gptr[g]..gptr[g+1]) are the partial-buffer positions
 * (row_off[j] + local row) of the blocks covering g, in increasing j.
 * ---------------------------------------------------------------------- */
typedef struct fl_blockop {
  int32_t nblocks;          /* J */
  int32_t nrows;            /* global row count N */
  int64_t ncols_total;      /* y-space length */
  int64_t partial_len;      /* sum_j m[j] */
  int32_t max_rows;         /* max_j m[j]     (shared-memory sizing) */
  int32_t max_ncols;        /* max_j ncols[j] (shared-memory sizing) */
  const double* vals;       /* block values */
  const int64_t* off;       /* (J,) element offsets */
  const int32_t* ld;        /* (J,) */
  const int32_t* m;         /* (J,) */
  const int32_t* ncols;     /* (J,) */
  const int64_t* col_off;   /* (J,) */
  const int64_t* row_off;   /* (J,) */
  const int32_t* rows;      /* (partial_len,) global row of each block row */
  const int32_t* gptr;      /* (N+1,) */
  const int32_t* gsrc;      /* (partial_len,) */
  /* launch tables (host-built, device-resident) */
  int32_t n_row_tiles;      /* tiles of FL_ROW_TILE rows */
  const int32_t* row_tiles; /* (n_row_tiles, 2): block, first row */
  int32_t n_col_tiles;      /* tiles of FL_COL_TILE columns */
  const int32_t* col_tiles; /* (n_col_tiles, 2): block, first column */
  double* partial;          /* (FL_LSQR_SPLIT_MAX * partial_len,) scratch */
  double* red_scratch;      /* (>= 2 * max(n_row_tiles, n_col_tiles, FL_LSQR_SPLIT_MAX * J) + 64) scratch */
  unsigned int* counter;    /* (4,) zero-initialised scratch */
  const int32_t* order;     /* (J,) block processing order (largest first), NULL = 0..J-1 */
} fl_blockop;

#define FL_ROW_TILE 256
#define FL_COL_TILE 32
/* The fused LSQR iteration may split each block's columns over up to this
 * many CTAs (each writes its own copy of the block's partial product). */
#define FL_LSQR_SPLIT_MAX 4

/* ------------------------------------------------------------------------
 * Assembly (assembly.py:124-238). Row r of block j: r < prod(box_cnt) is the
 * interior lattice point with per-dim index box_lo[i] + (C-order digit i of
 * r); otherwise constraint entry con_idx[con_ptr[j] + r - box] (a point index
 * into con_pts) of group con_grp[...]. All pointers are device pointers.
 * ---------------------------------------------------------------------- */
typedef struct fl_assembly_desc {
  int32_t dim;              /* d <= 3 */
  int32_t nsub;             /* J */
  int32_t count_per_dim;    /* S */
  int32_t nfeat;            /* K */
  int32_t activation;       /* FL_ACT_* */
  int32_t ngroups;          /* constraint groups (<= 7) */
  int32_t reach;            /* ceil(overlap_ratio): centers within +-reach of
                               the own center can cover a point of block j */
  const double* centers;    /* (d, S) decomposition centers */
  const double* half;       /* (d,) half widths */
  const double* weights;    /* (J, K, d) first-layer weights */
  const double* biases;     /* (J, K) first-layer biases */
  const double* axes;       /* concatenated lattice axes */
  const int64_t* axis_off;  /* (d,) start of axis i in `axes` */
  const double* op_coef;    /* (1+G, 2+2d): value, weight, first[d], second[d]
                               row 0 = interior operator, 1+g = group g */
  const double* con_pts;    /* (Ncp, d) constraint points */
  const int32_t* box;       /* (J, d, 2): lo, count */
  const int64_t* con_ptr;   /* (J+1,) */
  const int32_t* con_idx;   /* constraint point index */
  const int32_t* con_grp;   /* constraint group */
  int32_t n_tiles;          /* row tiles of fl_assemble_tile_rows() rows */
  const int32_t* tiles;     /* (n_tiles, 2): block, first row */
  /* hard-constraint mask (assembly.py:107-114): the window jet along axis a
     is multiplied by the mask's jet along a, given per point as (value,
     d/dx_a, d2/dx_a^2); NULL = no mask */
  const double* mask_int;   /* (n_interior, d, 3) interior lattice points, C order */
  const double* mask_con;   /* (Ncp, d, 3) constraint points */
  int64_t lattice_stride[3];/* C-order strides of the interior lattice (row id of a
                               lattice point = sum_i index_i * stride_i) */
} fl_assembly_desc;

/* rows per K1 tile: the `tiles` table lists (block, first row) in steps of
   fl_assemble_tile_rows() rows (FL_ASM_TILE in this build) */
#define FL_ASM_TILE 512
int32_t fl_assemble_tile_rows(void);

int fl_assemble(const fl_assembly_desc* desc, const fl_blockop* out, void* stream);

/* ------------------------------------------------------------------------
 * Truncated column-pivoted Householder QR of every block, in place
 * (linalg.py:58-97 rule: LAPACK dgeqp3 pivot choice, stop at the first
 * |R_tt| < sigma |R_00|, sigma = 0 keeps min(m, K)). On return block j's
 * first rank[j] columns hold Q_j (thin, sign-normalised so diag R > 0),
 * R[j*K*K ..] holds R_j column-major with leading dimension K, perm[j*K ..]
 * the pivot order (perm[j*K + t] = original local column of pivot t),
 * diag[j*K + t] = |R_tt| / |R_00|. rank[j] = -1 flags a non-finite block.
 * max_rows bounds m[j] over all blocks.
 * ---------------------------------------------------------------------- */
int fl_rrqr(const fl_blockop* blocks, int32_t K, int32_t max_rows, double sigma, double* R,
            int32_t* perm, int32_t* rank, double* diag, void* stream);

/* Same contract as fl_rrqr, BLAS-3 route for K >= 32, K % 32 == 0 and every
 * m[j] >= K: unpivoted blocked Householder QR A_j = Q0 R0
 * (DMMA trailing updates), truncated QRCP of R0 with LAPACK's dlaqps rule,
 * Q_j = Q0 [Q1; 0]. `A` is left unchanged; Q_j is written to the store `Q`
 * (same layout as A). `workspace` needs fl_rrqr_blocked_workspace() bytes;
 * store_elems = total doubles of the A store. No host synchronisation.
 * Shared-memory bound: K <= FL_RRQR_BLOCKED_MAX_K (else FL_ERR_INVALID); any
 * number of rows (blocks of up to FL_RRQR_BLOCKED_MAX_ROWS rows have the
 * 8-column inner panels of K2a staged in shared memory, taller ones are
 * factored in place). fl_rrqr stages one
 * max_rows-long reflector on chip: 8 * (4 K + max_rows) + 4 K bytes <= 220 KB
 * (about 25.8k rows at K = 512), else FL_ERR_INVALID; the host maps blocks
 * that neither route takes to CapExceededError. */
#define FL_RRQR_BLOCKED_MAX_K 640
#define FL_RRQR_BLOCKED_MAX_ROWS 2944
#define FL_RRQR_DIRECT_SMEM_MAX (220 * 1024)
int64_t fl_rrqr_blocked_workspace(int32_t nblocks, int32_t K, int64_t store_elems);
int fl_rrqr_blocked(const fl_blockop* A, const fl_blockop* Q, int32_t K, int64_t store_elems,
                    double sigma, double* R, int32_t* perm, int32_t* rank, double* diag,
                    void* workspace, void* stream);

/* y-space -> rows: out[g] = sum over covering blocks of (B_j x_j)[g] */
int fl_blockop_apply(const fl_blockop* op, const double* x, double* out, void* stream);
/* rows -> y-space: out_j = B_j^T r[I_j] */
int fl_blockop_apply_t(const fl_blockop* op, const double* r, double* out, void* stream);

/* ------------------------------------------------------------------------
 * Device LSQR (solvers.py:87-145). State lives in device memory; the host
 * reads only fl_lsqr_state after the loop.
 * ---------------------------------------------------------------------- */
typedef struct fl_lsqr_state {
  double alpha, beta, rhobar, phibar, rho, c, s, phi, theta;
  double beta_prev;         /* scale of the stored (unnormalised) u */
  double best;              /* monitor best residual */
  /* scipy stopping-rule accumulators (scipy.sparse.linalg.lsqr) */
  double anorm, ddnorm, xxnorm, z, cs2, sn2, bnorm, atol, btol, ctol;
  int64_t it;               /* iterations completed */
  int64_t best_it;          /* monitor best iteration (-1 none) */
  int64_t diverged_at;      /* first non-finite iteration, 0 = none */
  int32_t done;             /* 1 = loop finished (breakdown / rule / divergence) */
  int32_t breakdown;
  int32_t istop;            /* scipy rule code when a tolerance stopped it */
  int32_t use_rule;
  int32_t stride;           /* monitor stride */
  int32_t nonfinite;        /* scratch flag set by any CTA seeing a non-finite x */
  int32_t monitor;          /* 1 = best iterate by test error (fl_test_monitor), 0 = by residual */
  int32_t improved;         /* test-error monitor: x of the last recorded iteration is the new best */
} fl_lsqr_state;

typedef struct fl_lsqr_vecs {
  double* u;                /* (N,) unnormalised u; true u = u / beta_prev */
  double* v;                /* (n,) */
  double* vp;               /* (n,) unnormalised v' */
  double* w;                /* (n,) */
  double* x;                /* (n,) */
  double* xbest;            /* (n,) monitor best iterate */
  double* trace;            /* (max_iters+1,) phibar per iteration */
  double* ub;               /* (partial_len,) or null: u at every block row (block-local
                               order), kept by the row kernel so the fused kernel reads
                               its rows contiguously instead of gathering through rows */
} fl_lsqr_vecs;

/* rhs -> u, beta, v = Q^T u / alpha, w = v (solvers.py:98-117) */
int fl_lsqr_init(const fl_blockop* op, const double* rhs, fl_lsqr_vecs* vecs,
                 fl_lsqr_state* st, void* stream);
/* iterations first_it .. first_it+count-1 (solvers.py:119-144); every
 * kernel is a no-op once st->done is set, so a caller may enqueue the whole
 * budget (or capture it in a CUDA graph) without host synchronisation. */
int fl_lsqr_iterate(const fl_blockop* op, fl_lsqr_vecs* vecs, fl_lsqr_state* st,
                    int64_t first_it, int64_t count, void* stream);

/* ------------------------------------------------------------------------
 * K6 — device test-lattice monitor (runner.py:265-276 `_error_matrix`,
 * assembly.py:313-318 `l1_error`, solvers.py:59-69 `observe`). The error
 * of the iterate y is e = mean_g |(T y)[g] + lift[g] - truth[g]| / spread
 * with T_j = P_j[:, kept_j] R_j^{-1} (P = solution blocks at the test points).
 * ---------------------------------------------------------------------- */
typedef struct fl_test_monitor {
  fl_blockop T;             /* rows = test points, ncols = r_j, col_off = y offsets */
  const double* lift;       /* (n_test,) lift values at the test points */
  const double* truth;      /* (n_test,) true values */
  double spread;            /* std of the true values */
  double* err_trace;        /* (max_iters + 1,) e per recorded iteration */
  double* result;           /* (1,) output of fl_monitor_error */
} fl_test_monitor;

/* T_j = P_j[:, perm_j[0:r_j]] R_j^{-1} row by row (forward substitution with
 * R_j^T); r_j = T->ncols[j]. `tiles` = (n_tiles, 2) (block, first row) in
 * steps of FL_TBUILD_ROWS rows. P and T share one layout. */
int fl_error_blocks(const fl_blockop* P, const double* R, const int32_t* perm, int32_t K,
                    const fl_blockop* T, int32_t n_tiles, const int32_t* tiles, void* stream);
#define FL_TBUILD_ROWS 16
/* e(y) -> mon->result[0] */
int fl_monitor_error(const fl_test_monitor* mon, const double* y, void* stream);
/* fl_lsqr_iterate plus, after each recorded iteration (stride), e(x_it) ->
 * err_trace[it] and the best iterate by e (st->monitor must be 1); call
 * fl_lsqr_monitor_flush after the last iteration. */
int fl_lsqr_iterate_monitored(const fl_blockop* op, fl_lsqr_vecs* vecs, fl_lsqr_state* st,
                              int64_t first_it, int64_t count, const fl_test_monitor* mon,
                              void* stream);
/* copies x into xbest if the last recorded iterate improved the best */
int fl_lsqr_monitor_flush(const fl_blockop* op, fl_lsqr_vecs* vecs, fl_lsqr_state* st, void* stream);

/* ------------------------------------------------------------------------
 * N4 — CG on the normal equations with an optional block (additive-Schwarz)
 * preconditioner (solvers.py:150-239). Loop control reuses fl_lsqr_state
 * (it, done, breakdown, stride, best / best_it / improved, diverged_at;
 * monitor must be 1); scalars: alpha = r.z, beta = p.q, phi = step,
 * theta = r.z_next / r.z, phibar = last recorded residual ||M x - rhs||.
 * ---------------------------------------------------------------------- */
typedef struct fl_cg_vecs {
  double* tmp;              /* (N,) M p / M x */
  double* p;                /* (n,) */
  double* q;                /* (n,) M^T M p */
  double* r;                /* (n,) normal-equation residual */
  double* z;                /* (n,) P r (may equal r: no preconditioner) */
  double* x;                /* (n,) */
  double* xbest;            /* (n,) best recorded iterate */
  double* res_trace;        /* (max_iters + 1,) residual per recorded iteration */
  const double* rhs;        /* (N,) */
  double* scratch;          /* (>= 2 * 592) reduction slots */
  unsigned int* counter;    /* (1,) zero-initialised */
  int32_t stride;           /* recorded iterations: it % stride == 0 */
} fl_cg_vecs;

/* z[idx_b] = inv_b r[idx_b], inv_b row-major size_b x size_b with
 * size_b = idx_off[b+1] - idx_off[b] */
typedef struct fl_block_precond {
  int32_t nblocks;
  int32_t max_size;
  const int64_t* idx_off;   /* (nblocks + 1,) */
  const int32_t* idx;       /* concatenated column indices */
  const int64_t* val_off;   /* (nblocks,) start of inv_b in vals */
  const double* vals;
} fl_block_precond;

/* Additive-Schwarz setup (solvers.py:178-192): per block j of A (ncols_j <=
 * FL_AS_MAX_K) the Gramian A_j^T A_j, its Jacobi eigendecomposition and the
 * pseudo-inverse over eigenvalues > cutoff * the largest, written row-major
 * to inv + j * ncols_j^2 (a dense K x K per block: blocks of equal width);
 * degenerate[j] = 1 when the cutoff dropped an eigenvalue. */
#define FL_AS_MAX_K 96
int fl_as_setup(const fl_blockop* A, double cutoff, double* inv, int32_t* degenerate, void* stream);

/* z = P r on its own (AdditiveSchwarz.apply) */
int fl_block_precond_apply(const fl_block_precond* pre, const double* r, double* z, void* stream);
/* r = M^T rhs, z = P r, p = z, r.z (pre may be NULL) */
int fl_cg_init(const fl_blockop* op, fl_cg_vecs* v, const fl_block_precond* pre,
               fl_lsqr_state* st, void* stream);
/* iterations first_it .. first_it+count-1; mon (may be NULL) ranks the
 * recorded iterates by test error instead of residual */
int fl_cg_iterate(const fl_blockop* op, fl_cg_vecs* v, const fl_block_precond* pre,
                  fl_lsqr_state* st, int64_t first_it, int64_t count,
                  const fl_test_monitor* mon, void* stream);
/* ||M x - rhs|| -> out[0] */
int fl_cg_residual(const fl_blockop* op, fl_cg_vecs* v, double* out, void* stream);

/* ------------------------------------------------------------------------
 * Recovery (filtering.py:169-183): coeffs[kept global column] = R_j^{-1} y_j,
 * every other entry of coeffs (length J*K) exactly 0.
 * ---------------------------------------------------------------------- */
int fl_backsub_scatter(int32_t nblocks, int32_t K, const double* R, const int32_t* rank,
                       const int32_t* perm, const int64_t* y_off, const double* y,
                       double* coeffs, int32_t* singular_block, void* stream);

/* diagnostics: FP64 throughput probe (mode 0 DFMA, 1 DMMA m8n8k4); flops
 * per call = grid*256*iters*16 (mode 0) or grid*8*iters*2048 (mode 1) */
int fl_probe_fp64(int32_t mode, int32_t grid, int32_t iters, double* out, void* stream);
/* diagnostics: streaming read of n doubles (16-byte loads); bytes = 8 n */
int fl_probe_read(const double* buf, int64_t n, double* out, void* stream);

/* diagnostics: one batched compact-WY block-reflector launch (DMMA):
 * C_j[row0:m_j, tile] -= V_j op(T_j) V_j^T C_j[row0:m_j, tile] with V_j the
 * nb-wide (32 or 64) unit-lower panel whose diagonal starts at row0. */
int fl_dev_wy_apply(const double* V, const int64_t* voff, const int32_t* vld, double* C,
                    const int64_t* coff, const int32_t* cld, const int32_t* m, const double* T,
                    int64_t tstride, int32_t nb, int32_t row0, int32_t transT, const int32_t* ncols,
                    const int32_t* tiles, int32_t ntiles, void* stream);

/* Diagnostic (kernel-level tests): fused K2c over caller tables. Every block
 * j: C_j (m_j x rank_j, holding [Q1_j; 0]) <- H_0 .. H_{K-1} C_j with the
 * reflectors in V_j's K columns (unit diagonal implicit, entries on and above
 * it ignored) applied as 64-wide compact-WY blocks whose T factors are
 * T64[j][b] (64 x 64 column-major upper triangular); K % 64 == 0. Replaces
 * dorgqr's Q formation (linalg.py:74) on route R. */
int fl_dev_qform(const double* V, const int64_t* voff, const int32_t* vld, const int32_t* m, double* C,
                 const int64_t* coff, const int32_t* cld, const int32_t* rank, const double* T64, int32_t K,
                 int32_t nblocks, void* stream);

/* build metadata */
const char* fl_version(void);
/* description of the calling thread's last FL_ERR_CUDA ("file:line: name (text)") */
const char* fl_last_error(void);

#ifdef __cplusplus
}
#endif
#endif /* FEATLSQ_B200_H */
