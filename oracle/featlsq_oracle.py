"""CPU ORACLE — TEST INFRASTRUCTURE ONLY.

A numpy/scipy restatement of the reference hot path (`featlsq`, arXiv
2506.17626; reference tree `pkg/src/featlsq/`). Only `tests/`,
`__graft_entry__.smoke()` and `bench.py`'s `cpu_baseline` / `--impl
reference` leg may import this module, and only as the checker or as the timed
CPU baseline — never as part of the product path.

Pinning: `tests/test_oracle_golden.py` checks every function here against
golden vectors produced by importing the reference itself in the build
container (`tests/golden/make_golden.py`) and against the reference's
committed demo artifacts (`pkg/demos/out/oscillator/oscillator-baseline/`),
which this oracle reproduces.

Third-party arithmetic: the reference's QR is LAPACK `dgeqp3` + `dorgqr`
through `scipy.linalg.qr(pivoting=True)` (`linalg.py:74`) and its triangular
solve is `dtrtrs` (`linalg.py:112`); scipy 1.18.1 / scipy-openblas 0.3.30 in
this image. `qr_column_pivot` calls the same LAPACK routines (the algorithm
is LAPACK's); `qrcp_dlaqp2` restates LAPACK's unblocked pivot rule (`dlaqp2`:
IDAMAX first-max pivot over the current swapped positions, norm downdate
`temp = max(0, 1 - (|r_kj|/vn1_j)^2)`, recompute when
`temp*(vn1/vn2)^2 <= sqrt(eps)`) in numpy so the rule the CUDA kernel follows
is written out and checked independently of LAPACK.

Inputs are duck-typed: anything with the attributes of the reference's
`ProblemSpec`, `Decomposition` and `FeatureBasis` works (the product's value
types or the reference's own).
"""

from __future__ import annotations

import numpy as np
import scipy.linalg
import scipy.sparse
import scipy.sparse.linalg

EPS = np.finfo(float).eps * 0.5          # LAPACK dlamch('E') = 2^-53
TOL3Z = np.sqrt(EPS)                     # dlaqp2 recompute threshold


# ---------------------------------------------------------------------------
# jets: (value, first, second) triples, domains.py / jets.py semantics

def _mul(a, b):
    """Jet product rule, `jets.py:55-63`."""
    return (a[0] * b[0], a[1] * b[0] + a[0] * b[1],
            a[2] * b[0] + 2.0 * a[1] * b[1] + a[0] * b[2])


def _recip(a):
    """Jet reciprocal, `jets.py:76-80`."""
    iv = 1.0 / a[0]
    return (iv, -a[1] * iv * iv, (2.0 * a[1] * a[1] * iv - a[2]) * iv * iv)


def factor_arrays(t, mu, half):
    """Raw (1 + cos theta)^2 factor with two derivatives, exactly zero outside
    the strict support (`domains.py:109-123`)."""
    t = np.asarray(t, dtype=float)
    inside = np.abs(t - mu) < half
    theta = np.where(inside, np.pi * (t - mu) / half, 0.0)
    c, s = np.cos(theta), np.sin(theta)
    scale = np.pi / half
    w = (1.0 + c) ** 2
    w1 = -2.0 * (1.0 + c) * s * scale
    w2 = -2.0 * (c + c * c - s * s) * scale * scale
    for arr in (w, w1, w2):
        arr[~inside] = 0.0
    return w, w1, w2


def normalized_factor(dec, i, s, t, deriv):
    """w_s / sum_r w_r along dimension i (`domains.py:126-154`)."""
    mu, half = float(dec.centers[i, s]), float(dec.half_widths[i])
    w = factor_arrays(t, mu, half)
    num = w if deriv else (w[0], np.zeros_like(w[0]), np.zeros_like(w[0]))
    den = (np.zeros_like(t), np.zeros_like(t), np.zeros_like(t))
    for r in range(dec.count_per_dim):
        f = factor_arrays(t, float(dec.centers[i, r]), half)
        if not deriv:
            f = (f[0], np.zeros_like(f[0]), np.zeros_like(f[0]))
        den = (den[0] + f[0], den[1] + f[1], den[2] + f[2])
    if np.any(den[0] <= 0.0):
        raise ValueError("window normalizer vanishes at an evaluation point")
    return _mul(num, _recip(den))


def window_jet(dec, j, x, axis):
    """Product of per-dim normalized factors, derivatives along `axis` only
    (`domains.py:157-173`)."""
    idx = np.unravel_index(j, (dec.count_per_dim,) * dec.dim)
    jet = None
    for i in range(dec.dim):
        fac = normalized_factor(dec, i, int(idx[i]), x[:, i], i == axis)
        jet = fac if jet is None else _mul(jet, fac)
    return jet


def support(dec, j, x):
    """Strict support test (`domains.py:176-184`)."""
    idx = np.unravel_index(j, (dec.count_per_dim,) * dec.dim)
    m = np.ones(x.shape[0], dtype=bool)
    for i in range(dec.dim):
        m &= np.abs(x[:, i] - dec.centers[i, idx[i]]) < dec.half_widths[i]
    return m


def feature_jet(basis, j, x, axis):
    """Depth-1 feature jets of subdomain j (`basis.py:99-133`, activations
    `basis.py:24-40`, tanh jet `jets.py:89-93`)."""
    dec = basis.decomposition
    idx = np.unravel_index(j, (dec.count_per_dim,) * dec.dim)
    mu = np.array([dec.centers[i, idx[i]] for i in range(dec.dim)])
    xt = (x - mu) / dec.half_widths
    w0 = basis.weights[0][j]
    pre = xt @ w0.T
    if basis.biases[0] is not None:
        pre = pre + basis.biases[0][j]
    first = np.broadcast_to(w0[:, axis] * (1.0 / dec.half_widths[axis]), pre.shape)
    if basis.activation == "tanh":
        t = np.tanh(pre)
        sech2 = 1.0 - t * t
        return t, sech2 * first, -2.0 * t * sech2 * first * first
    if basis.activation == "sin":
        s, c = np.sin(pre), np.cos(pre)
        return s, c * first, -s * first * first
    sg = 0.5 * (1.0 + np.tanh(0.5 * pre))
    d1 = sg * (1.0 - sg)
    d2 = sg * (1.0 - sg) * (1.0 - 2.0 * sg)
    return sg, d1 * first, d2 * first * first


def operator_rows(op, problem, dec, basis, j, pts):
    """L[window_j * feature_j](pts) (`assembly.py:107-114`,
    `problems.py:39-47`)."""
    jets = []
    for a in range(dec.dim):
        w = window_jet(dec, j, pts, a)
        if problem.mask_jets is not None:  # window * mask (assembly.py:111-112)
            mk = problem.mask_jets(pts, a)
            w = _mul(w, (np.broadcast_to(mk.value, w[0].shape), np.broadcast_to(mk.first, w[0].shape),
                         np.broadcast_to(mk.second, w[0].shape)))
        wj = (w[0][:, None], w[1][:, None], w[2][:, None])
        jets.append(_mul(wj, feature_jet(basis, j, pts, a)))
    out = op.value_coef * jets[0][0]
    for a, jet in enumerate(jets):
        out = out + op.first_coefs[a] * jet[1] + op.second_coefs[a] * jet[2]
    return out


# ---------------------------------------------------------------------------
# assembly (assembly.py:124-238), including hard-constraint mask/lift problems

def default_counts(problem, dec, basis):
    """assembly.py:32-40 + :141-146 (one extra point per subdomain when masked)."""
    k, d = basis.feature_count, dec.dim
    root = int(np.ceil(k ** (1.0 / d)))
    while root > 1 and (root - 1) ** d >= k:
        root -= 1
    while root ** d < k:
        root += 1
    extra = 0 if problem.mask_jets is None else 1
    return dec.count_per_dim * (root + extra)


def lattice_axes(problem, dec, basis, interior_per_dim):
    d = dec.dim
    if interior_per_dim is None:
        interior_per_dim = default_counts(problem, dec, basis)
    counts = ((int(interior_per_dim),) * d if not isinstance(interior_per_dim, (tuple, list))
              else tuple(int(c) for c in interior_per_dim))
    if problem.mask_jets is None:
        axes = tuple(np.linspace(dec.domain.bounds[i, 0], dec.domain.bounds[i, 1], counts[i])
                     for i in range(d))
    else:  # cell centres (assembly.py:159-166)
        steps = dec.domain.widths / np.asarray(counts)
        axes = tuple(dec.domain.bounds[i, 0] + steps[i] * (np.arange(counts[i]) + 0.5)
                     for i in range(d))
    return counts, axes


def lift_operator_values(problem, op, pts):
    """assembly.py:117-121."""
    if problem.lift_jets is None:
        return np.zeros(np.atleast_2d(pts).shape[0])
    jets = [problem.lift_jets(pts, a) for a in range(problem.domain.dim)]
    out = op.value_coef * jets[0].value
    for a, jet in enumerate(jets):
        out = out + op.first_coefs[a] * jet.first + op.second_coefs[a] * jet.second
    return out


def assemble(problem, dec, basis, interior_per_dim, only=None):
    """Returns dict(blocks=[(rows int64, matrix (m, K))], rhs, row_count,
    column_count, interior_count, axes). `only` restricts the per-block loop
    to the listed subdomains (bounded CPU-baseline samples)."""
    d = dec.dim
    counts, axes = lattice_axes(problem, dec, basis, interior_per_dim)
    mesh = np.meshgrid(*axes, indexing="ij")
    interior = np.stack([m.ravel() for m in mesh], axis=1)
    n_int = interior.shape[0]
    iw = 1.0 / np.sqrt(n_int)
    rhs = [(problem.forcing(interior) - lift_operator_values(problem, problem.operator, interior)) * iw]
    con_off, off = [], n_int
    for con in problem.constraints:
        n_con = con.points.shape[0]
        w = np.sqrt(con.weight / n_con)
        rhs.append((np.asarray(con.targets, float)
                    - lift_operator_values(problem, con.operator, con.points)) * w)
        con_off.append((off, w))
        off += n_con
    k = basis.feature_count
    blocks = []
    for j in (range(dec.subdomain_count) if only is None else only):
        idx = np.unravel_index(j, (dec.count_per_dim,) * d)
        dim_idx =[np.nonzero(np.abs(axes[i] - dec.centers[i, idx[i]]) < dec.half_widths[i])[0]
                   for i in range(d)]
        row_sets, parts = [], []
        if all(ix.size for ix in dim_idx):
            grids = np.meshgrid(*dim_idx, indexing="ij")
            row_sets.append(np.ravel_multi_index([g.ravel() for g in grids], counts))
            pts = np.stack([axes[i][g.ravel()] for i, g in enumerate(grids)], axis=1)
            parts.append(operator_rows(problem.operator, problem, dec, basis, j, pts) * iw)
        else:
            row_sets.append(np.empty(0, dtype=np.int64))
            parts.append(np.empty((0, k)))
        for con, (co, w) in zip(problem.constraints, con_off):
            cp = np.atleast_2d(con.points)
            inside = support(dec, j, cp)
            row_sets.append(co + np.nonzero(inside)[0])
            parts.append(operator_rows(con.operator, problem, dec, basis, j, cp[inside]) * w
                         if inside.any() else np.empty((0, k)))
        blocks.append((np.concatenate(row_sets).astype(np.int64),
                       np.concatenate(parts, axis=0)))
    return dict(blocks=blocks, rhs=np.concatenate(rhs), row_count=off,
                column_count=basis.column_count, interior_count=n_int, axes=axes)


# ---------------------------------------------------------------------------
# truncated column-pivoted QR (linalg.py:58-97)

def _truncate(diag, rows, cols, sigma):
    limit = min(rows, cols)
    lead = diag[0] if diag.size else 0.0
    if lead == 0.0:
        return limit if sigma == 0.0 else 0
    if sigma == 0.0:
        return limit
    below = np.nonzero(diag < sigma * lead)[0]
    return int(below[0]) if below.size else limit


def qr_column_pivot(a, sigma):
    """The reference rule on LAPACK dgeqp3+dorgqr: returns (q, r, kept,
    dropped, diag_ratios) with diag(r) > 0."""
    a = np.asarray(a, dtype=float)
    rows, cols = a.shape
    if cols == 0:
        e = np.empty(0, dtype=np.int64)
        return np.empty((rows, 0)), np.empty((0, 0)), e, e, np.empty(0)
    q, r, perm = scipy.linalg.qr(a, mode="economic", pivoting=True)
    diag = np.abs(np.diag(r))
    rank = _truncate(diag, rows, cols, sigma)
    lead = diag[0] if diag.size else 0.0
    ratios = diag / lead if lead > 0.0 else np.zeros_like(diag)
    q, r = q[:, :rank].copy(), r[:rank, :rank].copy()
    signs = np.sign(np.diag(r))
    signs[signs == 0.0] = 1.0
    return q * signs, r * signs[:, None], perm[:rank].copy(), np.sort(perm[rank:]), ratios[:rank]


def qrcp_dlaqp2(a, sigma, record_gaps=False):
    """Independent numpy restatement of LAPACK's unblocked pivoted QR rule
    (dlaqp2 + dlarfg + dlarf), stopped at the reference's truncation point,
    with the thin Q formed from the kept reflectors (dorg2r). Returns the same
    tuple as `qr_column_pivot` (+ the per-step pivot margin when asked)."""
    a = np.array(a, dtype=float, order="F")
    m, n = a.shape
    kmax = min(m, n)
    perm = np.arange(n)
    vn1 = np.linalg.norm(a, axis=0)
    vn2 = vn1.copy()
    taus, diag, gaps = [], [], []
    lead = None
    rank = kmax
    for i in range(kmax):
        cand = vn1[i:]
        p = i + int(np.argmax(cand))            # first max = IDAMAX
        if record_gaps and cand.size > 1:
            top = cand[p - i]
            rest = np.delete(cand, p - i)
            gaps.append((top - rest.max()) / top if top > 0 else 0.0)
        if p != i:
            a[:, [i, p]] = a[:, [p, i]]
            perm[[i, p]] = perm[[p, i]]
            vn1[p], vn2[p] = vn1[i], vn2[i]
        # dlarfg on a[i:, i]
        alpha = a[i, i]
        xnorm = np.linalg.norm(a[i + 1:, i]) if i + 1 < m else 0.0
        if xnorm == 0.0:
            tau, beta = 0.0, alpha
        else:
            beta = -np.copysign(np.hypot(alpha, xnorm), alpha)
            tau = (beta - alpha) / beta
            a[i + 1:, i] *= 1.0 / (alpha - beta)
        a[i, i] = beta
        taus.append(tau)
        diag.append(abs(beta))
        if lead is None:
            lead = abs(beta)
        # truncation (linalg.py:75-85) decided on the fly
        if sigma > 0.0 and lead > 0.0 and abs(beta) < sigma * lead:
            rank = i
            break
        if sigma > 0.0 and lead == 0.0:
            rank = 0
            break
        if i + 1 < n and tau != 0.0:
            v = np.concatenate([[1.0], a[i + 1:, i]])
            wv = v @ a[i:, i + 1:]
            a[i:, i + 1:] -= tau * np.outer(v, wv)
        for jj in range(i + 1, n):
            if vn1[jj] != 0.0:
                temp = max(0.0, 1.0 - (abs(a[i, jj]) / vn1[jj]) ** 2)
                temp2 = temp * (vn1[jj] / vn2[jj]) ** 2
                if temp2 <= TOL3Z:
                    vn1[jj] = np.linalg.norm(a[i + 1:, jj]) if i + 1 < m else 0.0
                    vn2[jj] = vn1[jj]
                else:
                    vn1[jj] *= np.sqrt(temp)
    r = np.triu(a[:rank, :rank])
    # dorg2r: thin Q from the first `rank` reflectors
    q = np.zeros((m, rank))
    q[:rank, :rank] = np.eye(rank)
    for i in range(rank - 1, -1, -1):
        v = np.concatenate([[1.0], a[i + 1:, i]])
        q[i:, i:] -= taus[i] * np.outer(v, v @ q[i:, i:])
    signs = np.sign(np.diag(r))
    signs[signs == 0.0] = 1.0
    d = np.asarray(diag[:rank])
    ratios = d / d[0] if rank and d[0] > 0 else np.zeros(rank)
    out = (q * signs, r * signs[:, None], perm[:rank].copy(), np.sort(perm[rank:]), ratios)
    return out + (np.asarray(gaps),) if record_gaps else out


# ---------------------------------------------------------------------------
# filtering, preconditioned operator, recovery (filtering.py:92-183)

def filter_system(sysd, sigma, qr=qr_column_pivot):
    """Per-block truncated QRCP; returns list of dict(rows, kept, dropped, q,
    r) with kept/dropped as GLOBAL column ids, plus offsets."""
    out, counts = [], [0]
    k = None
    for j, (rows, mat) in enumerate(sysd["blocks"]):
        k = mat.shape[1]
        q, r, kept, dropped, _ = qr(mat, sigma)[:5]
        if kept.size == 0:
            raise RuntimeError(f"subdomain {j}: all {k} columns dropped at sigma={sigma}")
        out.append(dict(rows=rows, kept=j * k + kept, dropped=j * k + dropped, q=q, r=r))
        counts.append(counts[-1] + kept.size)
    return out, np.asarray(counts)


def q_operator(fblocks, offsets, row_count):
    """CSR of the orthonormal blocks (`filtering.py:133-144`)."""
    rows, cols, vals = [], [], []
    for b, lo in zip(fblocks, offsets):
        kc = b["kept"].size
        rows.append(np.repeat(b["rows"], kc))
        cols.append(np.tile(np.arange(lo, lo + kc), b["rows"].size))
        vals.append(b["q"].ravel())
    return scipy.sparse.coo_matrix(
        (np.concatenate(vals), (np.concatenate(rows), np.concatenate(cols))),
        shape=(row_count, int(offsets[-1]))).tocsr()


def raw_operator(sysd):
    rows, cols, vals = [], [], []
    for j, (r, mat) in enumerate(sysd["blocks"]):
        k = mat.shape[1]
        rows.append(np.repeat(r, k))
        cols.append(np.tile(np.arange(j * k, (j + 1) * k), r.size))
        vals.append(mat.ravel())
    return scipy.sparse.coo_matrix(
        (np.concatenate(vals), (np.concatenate(rows), np.concatenate(cols))),
        shape=(sysd["row_count"], sysd["column_count"])).tocsr()


def recover_solution(fblocks, offsets, y, column_count):
    """a[kept_j] = R_j^{-1} y_j, dropped -> 0 (`filtering.py:169-183`)."""
    a = np.zeros(column_count)
    for b, lo in zip(fblocks, offsets):
        kc = b["kept"].size
        a[b["kept"]] = scipy.linalg.solve_triangular(b["r"], y[lo:lo + kc], lower=False)
    return a


# ---------------------------------------------------------------------------
# LSQR (solvers.py:87-145)

class DivergenceError(RuntimeError):
    pass


def lsqr(matvec, rmatvec, ncols, rhs, max_iters, observe=None):
    """Golub-Kahan LSQR from zero, fixed budget, exact-breakdown stops.
    Returns (x, iterations, phibar, breakdown, phibar_trace)."""
    x = np.zeros(ncols)
    trace = []
    beta = float(np.linalg.norm(rhs))
    if beta == 0.0:
        return x, 0, 0.0, False, trace
    u = rhs / beta
    v = rmatvec(u)
    alpha = float(np.linalg.norm(v))
    if alpha == 0.0:
        return x, 0, beta, True, trace
    v = v / alpha
    w = v.copy()
    phibar, rhobar = beta, alpha
    its, brk = 0, False
    for it in range(1, max_iters + 1):
        u = matvec(v) - alpha * u
        beta = float(np.linalg.norm(u))
        if beta > 0.0:
            u = u / beta
        rho = float(np.hypot(rhobar, beta))
        c, s = rhobar / rho, beta / rho
        phi = c * phibar
        phibar = s * phibar
        x = x + (phi / rho) * w
        its = it
        if not np.isfinite(x).all():
            raise DivergenceError(f"non-finite iterate at iteration {it}")
        trace.append(phibar)
        if observe is not None:
            observe(it, x, phibar)
        if beta == 0.0:
            brk = True
            break
        vn = rmatvec(u) - beta * v
        alpha = float(np.linalg.norm(vn))
        if alpha == 0.0:
            brk = True
            break
        v = vn / alpha
        theta = s * alpha
        rhobar = -c * alpha
        w = v - (theta / rho) * w
    return x, its, float(phibar), brk, trace


def lsqr_stopping_rule(op_csr, rhs, atol, btol, iter_lim, conlim=1e8):
    """Iteration count under scipy's atol/btol rule: the
    reference lsqr has none, so the rule's oracle is scipy's lsqr on the
    reference operator."""
    res = scipy.sparse.linalg.lsqr(op_csr, rhs, atol=atol, btol=btol,
                                   iter_lim=iter_lim, conlim=conlim)
    return res[0], int(res[2]), int(res[1])


# ---------------------------------------------------------------------------
# demo reproduction: runner._solve_one with the test-lattice monitor
# (runner.py:265-293, solvers.py:47-69, assembly.py:244-318)

def random_source(seed, stream=0):
    """`linalg.py:21-30`: PCG64 over SeedSequence(seed, spawn_key=(stream,))."""
    ss = np.random.SeedSequence(entropy=seed, spawn_key=(stream,))
    return np.random.Generator(np.random.PCG64(ss))


def test_lattice(problem, dec):
    per_dim = problem.test_points_per_count * dec.count_per_dim
    axes = [np.linspace(problem.domain.bounds[i, 0], problem.domain.bounds[i, 1], per_dim)
            for i in range(dec.dim)]
    mesh = np.meshgrid(*axes, indexing="ij")
    pts = np.stack([m.ravel() for m in mesh], axis=1)
    truth = problem.exact(pts)
    return pts, truth, float(np.std(truth))


def solution_csr(dec, basis, pts, problem=None):
    """assembly.py:244-272 (P only; the lift is `lift_values`)."""
    rows, cols, vals = [], [], []
    k = basis.feature_count
    mask = problem.mask_value(pts) if problem is not None and problem.mask_value else None
    for j in range(dec.subdomain_count):
        inside = np.nonzero(support(dec, j, pts))[0]
        if inside.size == 0:
            continue
        p = pts[inside]
        w = window_jet(dec, j, p, 0)[0]
        if mask is not None:
            w = w * mask[inside]
        phi = feature_jet(basis, j, p, 0)[0]
        rows.append(np.repeat(inside, k))
        cols.append(np.tile(np.arange(j * k, (j + 1) * k), inside.size))
        vals.append((w[:, None] * phi).ravel())
    return scipy.sparse.coo_matrix(
        (np.concatenate(vals), (np.concatenate(rows), np.concatenate(cols))),
        shape=(pts.shape[0], basis.column_count)).tocsr()


def lift_values(problem, pts):
    return problem.lift_value(pts) if problem.lift_value else np.zeros(np.atleast_2d(pts).shape[0])


def run_rrqr_lsqr(problem, dec, basis, sigma, max_iters, interior_per_dim=None):
    """One seed of `runner._solve_one` for solver rrqr-lsqr, eval_stride 1.
    Returns dict(error, best_iteration, iterations, residual, drop_fraction,
    kept, coeffs)."""
    sysd = assemble(problem, dec, basis, interior_per_dim)
    fb, off = filter_system(sysd, sigma)
    q = q_operator(fb, off, sysd["row_count"])
    pts, truth, spread = test_lattice(problem, dec)
    phi = solution_csr(dec, basis, pts, problem)
    lift = lift_values(problem, pts)
    kept = np.concatenate([b["kept"] for b in fb])
    sinv = scipy.sparse.block_diag(
        [scipy.linalg.solve_triangular(b["r"], np.eye(b["kept"].size)) for b in fb],
        format="csc")
    t_mat = (phi[:, kept] @ sinv).tocsr()
    best = dict(err=np.inf, it=-1, x=None)

    def observe(it, x, _phibar):
        err = float(np.mean(np.abs(t_mat @ x + lift - truth)) / spread)
        if err < best["err"]:
            best.update(err=err, it=it, x=x.copy())
    x, its, phibar, _, _ = lsqr(lambda v: q @ v, lambda r: q.T @ r, int(off[-1]),
                                sysd["rhs"], max_iters, observe)
    y = best["x"] if best["x"] is not None else x
    coeffs = recover_solution(fb, off, y, sysd["column_count"])
    err = float(np.mean(np.abs(phi @ coeffs + lift - truth)) / spread)
    return dict(error=err, best_iteration=best["it"], iterations=its, residual=phibar,
                drop_fraction=1.0 - off[-1] / sysd["column_count"], kept=int(off[-1]),
                coeffs=coeffs)


# ---------------------------------------------------------------------------
# N4 baselines (solvers.py:150-239): additive Schwarz, CG on the normal equations

def as_preconditioner(blocks, column_ranges, cutoff=1e-14):
    """solvers.py:181-192: per block (pseudo-)inverse of A_j^T A_j through
    numpy's eigh (LAPACK dsyevd, as the reference). Returns (ranges,
    inverses, degenerate)."""
    invs, degenerate = [], []
    for j, mat in enumerate(blocks):
        gram = mat.T @ mat
        evals, evecs = np.linalg.eigh(gram)
        top = float(evals[-1]) if evals.size else 0.0
        keep = evals > cutoff * top if top > 0.0 else np.zeros_like(evals, dtype=bool)
        if not keep.all():
            degenerate.append(j)
        inv_vals = np.where(keep, 1.0 / np.where(keep, evals, 1.0), 0.0)
        invs.append((evecs * inv_vals) @ evecs.T)
    return list(column_ranges), invs, degenerate


def as_apply(ranges, invs, vec):
    out = np.empty_like(vec)
    for cols, inv in zip(ranges, invs):
        out[cols] = inv @ vec[cols]
    return out


def cg_normal(matvec, rmatvec, ncols, rhs, max_iters, stride=1, precond=None):
    """solvers.py:195-239. Returns (x, iterations, final residual, records,
    breakdown) with records (it, residual, residual) at recorded iterations."""
    x = np.zeros(ncols)
    r = rmatvec(rhs)
    z = precond(r) if precond else r
    p = z.copy()
    rz = float(r @ z)
    records, breakdown, iterations = [], False, 0
    for it in range(1, max_iters + 1):
        q = rmatvec(matvec(p))
        pq = float(p @ q)
        if pq <= 0.0 or not np.isfinite(pq):
            breakdown = True
            break
        step = rz / pq
        x = x + step * p
        r = r - step * q
        iterations = it
        if not np.isfinite(x).all():
            raise DivergenceError(f"non-finite iterate at iteration {it}")
        if not (stride > 1 and it % stride != 0):
            res = float(np.linalg.norm(matvec(x) - rhs))
            records.append((it, res, res))
        z = precond(r) if precond else r
        rz_next = float(r @ z)
        if rz == 0.0:
            breakdown = True
            break
        p = z + (rz_next / rz) * p
        rz = rz_next
    return x, iterations, float(np.linalg.norm(matvec(x) - rhs)), records, breakdown
