"""Parity of the CUDA path against the CPU oracle and the reference goldens.

All tests here need a B200 (`-m gpu`). The oracle (`oracle/featlsq_oracle.py`,
pinned to the reference in tests/test_oracle_golden.py) is the checker.
Tolerances (BASELINE.json north star):
  * rows, kept/dropped sequences, ranks: identical;
  * assembled entries: max |dA| <= 1e-13 max |A_j| per block (libm ulps);
  * R_j: ||dR||_F <= 1e-10 ||R||_F (entry-wise is not achievable, §0 F5);
  * Q_j: ||Q^T Q - I||_max <= 1e-12, ||Q R - A[:, kept]||_max <= 1e-12 max|A|;
  * operator products: <= 1e-12 relative;
  * LSQR after a converged fixed budget: relative L2 of y <= 1e-8, of M a <= 1e-8.
"""

import json
import os

import numpy as np
import pytest

from oracle import featlsq_oracle as O

pytestmark = pytest.mark.gpu

CFGS = ["cfg1", "cfg2", "cfg3", "cfg4", "cfg5"]


@pytest.fixture(scope="module")
def fl():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2506_17626_b200 as fl
    return fl


def _wl(name):
    from paper_2506_17626_b200 import workloads
    return workloads.build(name) if name == "cfg1" else workloads.build_small(name)


_cache = {}


def runs(fl, name):
    if name not in _cache:
        wl = _wl(name)
        ref = O.assemble(wl.problem, wl.dec, wl.basis, wl.interior_per_dim)
        fb, off = O.filter_system(ref, wl.sigma)
        sysd = fl.assemble(wl.problem, wl.dec, wl.basis, interior_per_dim=wl.interior_per_dim)
        fs = fl.filter_system(sysd, wl.sigma)
        _cache[name] = (wl, ref, fb, off, sysd, fs)
    return _cache[name]


@pytest.mark.parametrize("name", CFGS)
def test_assembly_matches_oracle(fl, name):
    wl, ref, _, _, sysd, _ = runs(fl, name)
    assert sysd.shape == (ref["row_count"], ref["column_count"])
    assert np.array_equal(sysd.rhs, ref["rhs"])
    for blk, (rows, mat) in zip(sysd.blocks, ref["blocks"]):
        assert np.array_equal(blk.rows, rows)
        assert blk.matrix.shape == mat.shape
        scale = max(np.abs(mat).max(), 1e-300)
        assert np.abs(blk.matrix - mat).max() <= 1e-13 * scale


@pytest.mark.parametrize("name", CFGS)
def test_filtering_matches_golden_and_oracle(fl, name, golden_dir):
    g = np.load(os.path.join(golden_dir, f"{name}.npz"))
    wl, ref, fb, off, sysd, fs = runs(fl, name)
    assert np.array_equal([len(k) for k in fs.kept_list], g["kept_len"])
    assert np.array_equal(fs.kept_columns, g["kept"])
    assert np.array_equal(np.concatenate(fs.dropped_list), g["dropped"])
    assert np.array_equal(fs.offsets, off)
    for blk, ob, sb in zip(fs.blocks, fb, ref["blocks"]):
        r, q = blk.r_factor, blk.q_factor
        assert np.linalg.norm(r - ob["r"]) <= 1e-10 * np.linalg.norm(ob["r"])
        assert np.all(np.diag(r) > 0)
        k = r.shape[0]
        assert np.abs(q.T @ q - np.eye(k)).max() <= 1e-12
        a = sb[1]
        local = blk.kept_columns - blk.subdomain * a.shape[1]
        assert np.abs(q @ r - a[:, local]).max() <= 1e-12 * np.abs(a).max()
    np.testing.assert_allclose([np.linalg.norm(b.r_factor) for b in fs.blocks], g["r_fro"],
                               rtol=1e-10)


@pytest.mark.parametrize("name", CFGS)
def test_preconditioned_products_match_oracle(fl, name):
    """K3 vs a host CSR of the same Q blocks: <= 1e-12. Against the
    oracle's own Q (a different correct QR) the blocks differ by ~1e-6 in
    their last kept columns, so that comparison is bounded
    at 1e-5."""
    wl, ref, fb, off, sysd, fs = runs(fl, name)
    op = fl.precondition(fs)
    own = op.csr()
    q = O.q_operator(fb, off, ref["row_count"])
    rng = np.random.default_rng(5)
    y = rng.standard_normal(op.shape[1])
    r = rng.standard_normal(op.shape[0])
    got = op.apply(y)
    assert np.linalg.norm(got - own @ y) <= 1e-12 * np.linalg.norm(own @ y)
    assert np.linalg.norm(got - q @ y) <= 1e-5 * np.linalg.norm(q @ y)
    got = op.apply_transpose(r)
    assert np.linalg.norm(got - own.T @ r) <= 1e-12 * np.linalg.norm(own.T @ r)
    assert np.linalg.norm(got - q.T @ r) <= 1e-5 * np.linalg.norm(q.T @ r)
    # raw system products (assembly.py:91-104)
    a = rng.standard_normal(sysd.column_count)
    M = O.raw_operator(ref)
    got, want = fl.apply(sysd, a), M @ a
    assert np.linalg.norm(got - want) <= 1e-12 * np.linalg.norm(want)
    got, want = fl.apply_transpose(sysd, r), M.T @ r
    assert np.linalg.norm(got - want) <= 1e-12 * np.linalg.norm(want)


@pytest.mark.parametrize("name", CFGS)
def test_recovery_matches_oracle(fl, name):
    wl, ref, fb, off, sysd, fs = runs(fl, name)
    y = np.random.default_rng(6).standard_normal(fs.kept_total)
    a_dev = fl.recover_solution(fs, y)
    a_ref = O.recover_solution(fb, off, y, ref["column_count"])
    dropped = np.concatenate(fs.dropped_list)
    assert np.all(a_dev[dropped] == 0.0)
    # Q y == M a holds to ~eps * kappa(R_j) (kappa(R_j) ~ 1e10 at sigma = 1e-10),
    # for the device's factors and for the oracle's alike; the reference's own
    # 1e-8 check (tests/test_filtering.py:143-149) is at sigma = 1e-4, see
    # test_filter_sigma_properties
    M = O.raw_operator(ref)
    ma = M @ a_dev
    qy = fl.precondition(fs).apply(y)
    mr = M @ a_ref
    qr = O.q_operator(fb, off, ref["row_count"]) @ y
    dev_gap = np.linalg.norm(ma - qy) / np.linalg.norm(qy)
    ref_gap = np.linalg.norm(mr - qr) / np.linalg.norm(qr)
    assert dev_gap <= 1e-5 and dev_gap <= 10 * max(ref_gap, 1e-12)
    assert np.linalg.norm(ma - mr) <= 1e-5 * np.linalg.norm(mr)
    # identical factor: device back substitution == scipy dtrtrs to 1e-12
    for blk in list(fs.blocks)[:4]:
        yy = np.random.default_rng(blk.subdomain).standard_normal(blk.kept_count)
        got = fl.back_substitute(blk.r_factor, yy)
        import scipy.linalg
        want = scipy.linalg.solve_triangular(blk.r_factor, yy)
        assert np.linalg.norm(got - want) <= 1e-12 * np.linalg.norm(want) * max(
            1.0, np.linalg.cond(blk.r_factor) * 1e-16 * 1e4)


@pytest.mark.parametrize("name", CFGS)
def test_lsqr_same_operator_matches_reference(fl, name, golden_dir):
    """Same operator, different summation order: device LSQR run on the
    oracle's Q blocks (uploaded) against the oracle's lsqr on the same Q —
    the first 100 residual estimates within 1e-9, the 100-step iterate within
    1e-6. Beyond ~100-300 steps two fp64 implementations that differ only in
    summation order drift apart mid-run before re-converging,
    so mid-run iterates are not a gate. Against the reference golden (whose
    Q differs from the oracle's by the assembly ulps amplified through
    kappa(R), ~1e-6) and with the device's own Q, the records agree to 1e-5."""
    from paper_2506_17626_b200 import _device as D
    g = np.load(os.path.join(golden_dir, f"{name}.npz"))
    wl, ref, fb, off, sysd, fs = runs(fl, name)
    oq = D.blocks_from_host(ref["row_count"], [b["rows"] for b in fb], [b["q"] for b in fb])
    res = fl.lsqr(oq, ref["rhs"], 100)
    tr = np.array([r[1] for r in res.monitor.records])
    q = O.q_operator(fb, off, ref["row_count"])
    x100, _, _, _, tr_o = O.lsqr(lambda v: q @ v, lambda r: q.T @ r, q.shape[1], ref["rhs"], 100)
    np.testing.assert_allclose(tr, tr_o, rtol=1e-9)
    assert np.linalg.norm(res.solution - x100) <= 1e-6 * np.linalg.norm(x100)
    np.testing.assert_allclose(tr, g["lsqr_records"][:100], rtol=1e-5)
    own = fl.lsqr(fl.precondition(fs), sysd.rhs, 100)
    tro = np.array([r[1] for r in own.monitor.records])
    np.testing.assert_allclose(tro, g["lsqr_records"][:100], rtol=1e-5)


def test_lsqr_converged_cfg1_matches_oracle(fl):
    """cfg1 at the paper's 10 000-iteration budget (converged regime, SURVEY
    §8(c)): y and M a within 1e-8 of the oracle's run."""
    wl, ref, fb, off, sysd, fs = runs(fl, "cfg1")
    q = O.q_operator(fb, off, ref["row_count"])
    x_o, its_o, *_ = O.lsqr(lambda v: q @ v, lambda r: q.T @ r, q.shape[1], ref["rhs"], 10000)
    res = fl.lsqr(fl.precondition(fs), sysd.rhs, 10000)
    assert res.iterations_run == its_o
    assert np.linalg.norm(res.solution - x_o) <= 1e-8 * np.linalg.norm(x_o)
    M = O.raw_operator(ref)
    ma = M @ fl.recover_solution(fs, res.solution)
    mo = M @ O.recover_solution(fb, off, x_o, ref["column_count"])
    assert np.linalg.norm(ma - mo) <= 1e-8 * np.linalg.norm(mo)


def test_lsqr_stopping_rule_cfg1_reports_iterations(fl):
    """scipy atol=btol=1e-12 rule on the device vs scipy on the same Q blocks.
    Where the rule fires at ~1e4 iterations depends on rounding (§0 F3):
    1-ulp perturbations of the operator move scipy's own count by ~±1.5%, so
    the device count must fall inside that ensemble's range widened by 3%."""
    wl, ref, fb, off, sysd, fs = runs(fl, "cfg1")
    pop = fl.precondition(fs)
    q = pop.csr()
    rng = np.random.default_rng(0)
    counts = []
    for k in range(6):
        qq = q.copy()
        if k:
            qq.data = qq.data * (1 + 2.0 ** -52 * rng.standard_normal(qq.data.size))
        _, its_o, istop_o = O.lsqr_stopping_rule(qq, ref["rhs"], 1e-12, 1e-12, 20000)
        counts.append(its_o)
    res = fl.lsqr(pop, sysd.rhs, 20000, atol=1e-12, btol=1e-12)
    assert res.istop in (1, 2, 3)
    assert 0.97 * min(counts) <= res.iterations_run <= 1.03 * max(counts), (res.iterations_run, counts)


# ---------------------------------------------------------------- QR unit cases
def test_qr_column_pivot_golden_cases(fl, golden_dir):
    g = np.load(os.path.join(golden_dir, "qrcp.npz"))
    for i in range(int(g["count"])):
        a, s = g[f"a{i}"], float(g[f"sigma{i}"])
        pq = fl.qr_column_pivot(a, s)
        assert np.array_equal(pq.kept, g[f"kept{i}"]), i
        assert np.array_equal(pq.dropped, g[f"dropped{i}"]), i
        rr = g[f"r{i}"]
        if rr.size and np.linalg.norm(rr) > 0:
            assert np.linalg.norm(pq.r_factor - rr) <= 1e-10 * np.linalg.norm(rr), i
            assert np.abs(pq.q_factor.T @ pq.q_factor - np.eye(pq.kept.size)).max() <= 1e-12
            assert np.abs(pq.q_factor @ pq.r_factor - a[:, pq.kept]).max() <= 1e-12 * np.abs(a).max()


def test_qr_rank_matches_svd_oracle(fl):
    """tests/test_linalg.py:39-58 property on the device kernel."""
    rng = fl.RandomSource(11).generator()
    sigma = 1e-6
    for _ in range(40):
        rows = int(rng.integers(10, 40))
        cols = int(rng.integers(5, min(rows, 25) + 1))
        rank = int(rng.integers(1, cols + 1))
        sv = np.empty(cols)
        sv[:rank] = rng.uniform(0.5, 2.0, rank)
        sv[rank:] = sigma * 10.0 ** rng.uniform(-4.0, -1.0, cols - rank)
        u, _ = np.linalg.qr(rng.standard_normal((rows, cols)))
        v, _ = np.linalg.qr(rng.standard_normal((cols, cols)))
        a = (u * np.sort(sv)[::-1]) @ v.T
        svd_rank = int(np.sum(np.linalg.svd(a, compute_uv=False) > sigma * sv.max()))
        assert abs(fl.qr_column_pivot(a, sigma).kept.size - svd_rank) <= 1


def test_qr_edge_cases(fl):
    assert fl.qr_column_pivot(np.zeros((5, 3)), 1e-8).kept.size == 0
    assert fl.qr_column_pivot(np.zeros((5, 3)), 0.0).kept.size == 3
    assert fl.qr_column_pivot(np.diag([1.0, 0.5, 0.25]), 0.5).kept.size == 2
    with pytest.raises(fl.InvalidInputError):
        fl.qr_column_pivot(np.eye(3), 1.0)
    a = np.eye(3)
    a[0, 0] = np.nan
    with pytest.raises(fl.InvalidInputError):
        fl.qr_column_pivot(a, 0.1)
    base = np.random.default_rng(0).standard_normal((12, 5))
    dup = np.concatenate([base, base[:, 2:3]], axis=1)
    assert fl.qr_column_pivot(dup, 1e-8).kept.size == 5


@pytest.mark.parametrize("K", [160, 192, 224, 256, 704])
def test_qr_column_pivot_both_routes_match_scipy(fl, K):
    """K = 160 / 224 take route R with the 32-wide branches (K2a panel +
    wy_apply<32> loop, the 32-wide K2c loop), K = 192 / 256 the 64-wide
    updates and the fused K2c; K = 704 exceeds route R's shared-memory bound
    and takes the direct kernel (filtering.rrqr_route, the same selection
    filter_system makes). All reproduce LAPACK's kept sequence on a
    gapped-spectrum matrix, R norm-wise and Q's own gates (linalg.py:58-97)."""
    from paper_2506_17626_b200 import _device as D
    from paper_2506_17626_b200.filtering import rrqr_route
    rng = np.random.default_rng(K)
    m = 900
    u, _ = np.linalg.qr(rng.standard_normal((m, K)))
    w, _ = np.linalg.qr(rng.standard_normal((K, K)))
    s = np.logspace(0, -14, K)
    a = (u * s) @ w.T
    route = rrqr_route(D.BlockLayout(m, K, [np.arange(m)]))
    assert route == ("direct" if K > 640 else "blocked")
    _, r_ref, kept_ref, _, _ = O.qr_column_pivot(a, 1e-10)
    got = fl.qr_column_pivot(a, 1e-10)
    assert np.array_equal(got.kept, kept_ref)
    assert np.linalg.norm(got.r_factor - r_ref) <= 1e-10 * np.linalg.norm(r_ref)
    q, r = got.q_factor, got.r_factor
    assert np.abs(q.T @ q - np.eye(q.shape[1])).max() <= 1e-12
    assert np.abs(q @ r - a[:, got.kept]).max() <= 1e-12 * np.abs(a).max()


@pytest.mark.parametrize("m,K", [(2500, 128), (4001, 160), (7003, 128), (11770, 192), (13001, 128),
                                 (30011, 64),
                                 # row counts around the leading-dimension padding (16) and the
                                 # staging threshold (2944 rows) of the panel kernel
                                 (129, 128), (143, 128), (144, 128), (145, 128), (257, 256), (1000, 160),
                                 (2944, 128), (2945, 128), (5888, 128), (5889, 128), (11776, 128),
                                 (11777, 128)])
def test_route_r_tall_blocks_match_scipy(fl, m, K):
    """Route R's panel kernel stages its 8-column inner panels in shared
    memory for blocks of up to 2944 rows and factors taller blocks in place;
    both, with row counts that are odd, 2 mod 4 or at the thresholds,
    reproduce LAPACK's factorisation (linalg.py:58-97). (30011, 64) is a
    narrow block beyond the direct kernel's on-chip bound."""
    from paper_2506_17626_b200 import _device as D
    from paper_2506_17626_b200.filtering import rrqr_route
    rng = np.random.default_rng(m + K)
    u, _ = np.linalg.qr(rng.standard_normal((m, K)))
    w, _ = np.linalg.qr(rng.standard_normal((K, K)))
    a = (u * np.logspace(0, -13, K)) @ w.T
    assert rrqr_route(D.BlockLayout(m, K, [np.arange(m)])) == "blocked"
    _, r_ref, kept_ref, _, _ = O.qr_column_pivot(a, 1e-10)
    got = fl.qr_column_pivot(a, 1e-10)
    assert np.array_equal(got.kept, kept_ref)
    assert np.linalg.norm(got.r_factor - r_ref) <= 1e-10 * np.linalg.norm(r_ref)
    q, r = got.q_factor, got.r_factor
    assert np.abs(q.T @ q - np.eye(q.shape[1])).max() <= 1e-12
    assert np.abs(q @ r - a[:, got.kept]).max() <= 1e-12 * np.abs(a).max()


def test_rhs_evaluated_off_thread(fl):
    """`assemble` hands the right-hand side (the problem's forcing / lift
    callables over every point, assembly.py:179-192) to a worker thread; the
    `rhs` attribute joins on first access, equals the oracle's, and re-raises
    what a callable raised."""
    import dataclasses
    import threading
    from paper_2506_17626_b200 import workloads
    wl = workloads.build("cfg1")
    seen = []

    def forcing(p):
        seen.append(threading.current_thread().name)
        return wl.problem.forcing(p)
    prob = dataclasses.replace(wl.problem, forcing=forcing)
    sysd = fl.assemble(prob, wl.dec, wl.basis, interior_per_dim=wl.interior_per_dim)
    ref = O.assemble(wl.problem, wl.dec, wl.basis, wl.interior_per_dim)
    assert np.array_equal(sysd.rhs, ref["rhs"]) and sysd.rhs is sysd.rhs
    assert seen == ["featlsq-rhs"]

    def broken(p):
        raise ValueError("forcing failed")
    sysd = fl.assemble(dataclasses.replace(wl.problem, forcing=broken), wl.dec, wl.basis,
                       interior_per_dim=wl.interior_per_dim)
    fs = fl.filter_system(sysd, wl.sigma)   # the blocks do not depend on the right-hand side
    assert fs.kept_total > 0
    with pytest.raises(ValueError, match="forcing failed"):
        sysd.rhs


def test_tall_blocks_end_to_end(fl):
    """Blocks of 40 000 rows (beyond what the panel kernel, the direct RRQR
    and the transposed product kernels stage on chip): K1, route R with
    in-place inner panels, the split LSQR kernels with gathered rows, and
    recovery against the oracle (the reference has no block-size bound)."""
    from paper_2506_17626_b200 import _device as D, workloads
    wl = workloads.build("cfg1", S=4, M=128, n=60000, overlap=2.0)
    sysd = fl.assemble(wl.problem, wl.dec, wl.basis, interior_per_dim=wl.interior_per_dim)
    assert max(b.rows.size for b in sysd.blocks) > 30000
    ref = O.assemble(wl.problem, wl.dec, wl.basis, wl.interior_per_dim)
    for blk, (rows, mat) in zip(sysd.blocks, ref["blocks"]):
        assert np.array_equal(blk.rows, rows)
        assert np.abs(blk.matrix - mat).max() <= 1e-13 * np.abs(mat).max()
    fs = fl.filter_system(sysd, wl.sigma)
    fb, off = O.filter_system(ref, wl.sigma)
    assert np.array_equal(fs.kept_columns, np.concatenate([b["kept"] for b in fb]))
    for blk, ob in zip(fs.blocks, fb):
        assert np.linalg.norm(blk.r_factor - ob["r"]) <= 1e-10 * np.linalg.norm(ob["r"])
        q = blk.q_factor
        assert np.abs(q.T @ q - np.eye(q.shape[1])).max() <= 1e-12
    rng = np.random.default_rng(0)
    M = O.raw_operator(ref)
    a, r = rng.standard_normal(sysd.column_count), rng.standard_normal(sysd.row_count)
    assert np.linalg.norm(fl.apply(sysd, a) - M @ a) <= 1e-12 * np.linalg.norm(M @ a)
    assert np.linalg.norm(fl.apply_transpose(sysd, r) - M.T @ r) <= 1e-12 * np.linalg.norm(M.T @ r)
    # same operator (the oracle's Q blocks, uploaded): the residual estimates
    # agree to 1e-9 until the Krylov space of this rank-57 system is
    # exhausted (iteration ~28; the same happens with 20 000-row blocks,
    # which fit the staging buffers), and stay within a few percent after
    oq = D.blocks_from_host(ref["row_count"], [b["rows"] for b in fb], [b["q"] for b in fb])
    res = fl.lsqr(oq, ref["rhs"], 50)
    q = O.q_operator(fb, off, ref["row_count"])
    x50, _, _, _, tr_o = O.lsqr(lambda v: q @ v, lambda u: q.T @ u, q.shape[1], ref["rhs"], 50)
    got = np.array([rec[1] for rec in res.monitor.records])
    np.testing.assert_allclose(got[:25], tr_o[:25], rtol=1e-9)
    np.testing.assert_allclose(got, tr_o, rtol=5e-2)
    own = fl.lsqr(fl.precondition(fs), sysd.rhs, 50)
    coeffs = fl.recover_solution(fs, own.solution)
    assert np.isfinite(coeffs).all() and np.all(coeffs[np.concatenate(fs.dropped_list)] == 0.0)


@pytest.mark.parametrize("K", [160, 256])
def test_route_r_rejects_non_finite(fl, K):
    """Route R flags a block holding NaN or Inf with rank -1 (the finiteness
    test of linalg.py:49-55); qr_column_pivot and filter_system raise
    InvalidInputError like the reference (filtering.py:100 -> linalg.py:66)."""
    from paper_2506_17626_b200 import workloads
    rng = np.random.default_rng(1)
    for bad in (np.nan, np.inf):
        a = rng.standard_normal((400, K))
        a[123, K // 2] = bad
        with pytest.raises(fl.InvalidInputError, match="non-finite"):
            fl.qr_column_pivot(a, 1e-10)
    from paper_2506_17626_b200.filtering import rrqr_route
    wl = workloads.build_small("cfg2" if K == 160 else "cfg3", M=K)
    sysd = fl.assemble(wl.problem, wl.dec, wl.basis, interior_per_dim=wl.interior_per_dim)
    assert rrqr_route(sysd.store.layout) == "blocked"
    blk = sysd.blocks[7]
    mat = blk.matrix.copy()
    mat[3, 5] = np.nan
    sysd.blocks[7] = fl.SubdomainBlock(blk.subdomain, blk.rows, blk.columns, mat)
    with pytest.raises(fl.InvalidInputError, match="non-finite"):
        fl.filter_system(sysd, wl.sigma)


# ---------------------------------------------------------------- LSQR unit cases
@pytest.fixture(scope="module")
def tall(golden_dir):
    g = np.load(os.path.join(golden_dir, "lsqr_dense.npz"))
    return g["a"], g["b"], g


def test_lsqr_dense_matches_reference(fl, tall):
    a, b, g = tall
    res = fl.lsqr(a, b, 200)
    assert np.allclose(res.solution, g["x200"], atol=1e-12)
    assert np.allclose(res.solution, np.linalg.pinv(a) @ b, atol=1e-8)
    mon = fl.ConvergenceMonitor()
    res = fl.lsqr(a, b, 60, mon)
    assert res.residual_norm == pytest.approx(np.linalg.norm(a @ res.solution - b), rel=1e-6)
    res_tr = [r for _, r, _ in mon.records]
    assert all(r2 <= r1 + 1e-12 for r1, r2 in zip(res_tr, res_tr[1:]))


def test_lsqr_breakdowns(fl):
    res = fl.lsqr(np.eye(4), np.zeros(4), 10)
    assert res.iterations_run == 0 and res.residual_norm == 0.0
    assert np.array_equal(res.solution, np.zeros(4))
    res = fl.lsqr(np.array([[1.0], [0.0]]), np.array([0.0, 1.0]), 10)
    assert res.breakdown and res.iterations_run == 0
    assert res.residual_norm == pytest.approx(1.0)
    b = np.array([1.0, 2.0, 3.0])
    res = fl.lsqr(np.eye(3), b, 50)
    assert res.breakdown and res.iterations_run <= 3
    assert np.allclose(res.solution, b, atol=1e-12)


def test_lsqr_divergence_and_shape(fl):
    a = np.full((3, 3), np.nan)
    with pytest.raises(fl.DivergenceError, match="iteration 1"):
        fl.lsqr(fl.Operator(lambda v: a @ v, lambda r: a.T @ r, (3, 3)), np.ones(3), 5)
    with pytest.raises(fl.InvalidInputError):
        fl.lsqr(np.eye(3), np.ones(4), 5)


def test_monitor_stride_and_best_iterate(fl, tall):
    a, b, _ = tall
    mon = fl.ConvergenceMonitor(stride=10)
    fl.lsqr(a, b, 35, mon)
    assert [it for it, _, _ in mon.records] == [10, 20, 30]
    a3 = np.diag([1.0, 2.0, 3.0])
    snap = {}

    def error_fn(x):
        if 1 not in snap:
            snap[1] = x.copy()
        return float(np.linalg.norm(x - snap[1]))
    mon = fl.ConvergenceMonitor(error_fn=error_fn)
    res = fl.lsqr(a3, np.ones(3), 30, mon)
    assert mon.best_iteration == 1
    assert np.allclose(res.best_solution, snap[1], atol=0)


def test_lsqr_deterministic(fl):
    wl, ref, fb, off, sysd, fs = runs(fl, "cfg2")
    op = fl.precondition(fs)
    r1 = fl.lsqr(op, sysd.rhs, 200)
    r2 = fl.lsqr(op, sysd.rhs, 200)
    assert np.array_equal(r1.solution, r2.solution)


# ---------------------------------------------------------------- boundary behaviour
def test_degenerate_block_and_mutation(fl):
    p = fl.oscillator_problem(30.0)
    dec = fl.decompose(p.domain, 4, 2.9)
    basis = fl.init_basis(dec, 4, 1, "tanh", np.random.default_rng(0))
    system = fl.assemble(p, dec, basis)
    blk = system.blocks[0]
    system.blocks[0] = fl.SubdomainBlock(blk.subdomain, blk.rows, blk.columns,
                                         np.zeros_like(blk.matrix))
    with pytest.raises(fl.DegenerateSubdomainError, match="subdomain 0"):
        fl.filter_system(system, 1e-8)


def test_filter_sigma_properties(fl):
    p = fl.oscillator_problem(30.0)
    dec = fl.decompose(p.domain, 8, 2.9)
    basis = fl.init_basis(dec, 8, 1, "tanh", np.random.default_rng(0))
    system = fl.assemble(p, dec, basis)
    kept = [fl.filter_system(system, s).kept_total for s in (0.0, 1e-4, 1e-2, 0.3)]
    assert kept[0] == system.column_count and kept == sorted(kept, reverse=True)
    loose, tight = fl.filter_system(system, 1e-4), fl.filter_system(system, 1e-2)
    for lo, hi in zip(loose.blocks, tight.blocks):
        assert np.array_equal(hi.kept_columns, lo.kept_columns[:hi.kept_count])
    fs = fl.filter_system(system, 0.0)
    rng = np.random.default_rng(8)
    a_true = rng.standard_normal(system.column_count)
    y = np.concatenate([b.r_factor @ a_true[b.kept_columns] for b in fs.blocks])
    assert np.allclose(fl.recover_solution(fs, y), a_true, atol=1e-8)
    op = fl.precondition(fs)
    # tests/test_filtering.py:143-149: Q y and M a agree when a = recover(y)
    yy = np.random.default_rng(6).standard_normal(loose.kept_total)
    assert np.allclose(fl.precondition(loose).apply(yy),
                       fl.apply(system, fl.recover_solution(loose, yy)), atol=1e-8)
    import scipy.linalg
    s_inv = scipy.linalg.block_diag(*[np.linalg.inv(b.r_factor) for b in loose.blocks])
    assert np.allclose(fl.precondition(loose).materialize(), loose.materialize() @ s_inv, atol=1e-10)
    assert op.shape == (system.row_count, system.column_count)


def test_oscillator_demo_matches_committed_report(fl, golden_dir):
    """The reference demo (oscillator, S=20, K=8, sigma=1e-8, 10 000 LSQR
    iterations, per-iteration test-lattice monitor, best iterate kept).

    * Device path end to end: drop fractions identical, iterations identical,
      final residual within 1e-6 (converged state).
    * LSQR arithmetic: the device loop run on the reference's own Q blocks
      (the oracle's, which reproduce the committed report exactly) gives the
      committed final residual within 1e-6.
    * The best-iterate error (device factors or reference factors) is only
      bounded by the spread of correct implementations: it is read off a
      mid-run dip of the test-error curve that summation order alone moves by
      up to 2x (measured with the reference algorithm itself,
      see below).
    """
    import scipy.linalg
    import scipy.sparse
    from paper_2506_17626_b200 import _device as D
    rep = json.load(open(os.path.join(golden_dir, "oscillator_report.json")))
    p = fl.oscillator_problem(60.0)
    dec = fl.decompose(p.domain, 20, 2.9)
    pts, truth, spread = O.test_lattice(p, dec)
    for s in rep["seeds"][:2]:
        basis = fl.init_basis(dec, 8, 1, "tanh", fl.RandomSource(s["seed"]).generator())
        system = fl.assemble(p, dec, basis)
        fs = fl.filter_system(system, 1e-8)
        assert fs.drop_fraction == pytest.approx(s["drop_fraction"], abs=1e-15)
        phi = O.solution_csr(dec, basis, pts)

        def err_of(blocks, kept, y):
            sinv = scipy.sparse.block_diag(
                [scipy.linalg.solve_triangular(r, np.eye(r.shape[0])) for r in blocks],
                format="csc")
            return (phi[:, kept] @ sinv).tocsr()

        # device LSQR on the oracle's Q (reference factors)
        ref = O.assemble(p, dec, basis, 160)
        fb, off = O.filter_system(ref, 1e-8)
        t_ref = err_of([b["r"] for b in fb], np.concatenate([b["kept"] for b in fb]), None)
        oq = D.blocks_from_host(ref["row_count"], [b["rows"] for b in fb], [b["q"] for b in fb])
        mon_o = fl.ConvergenceMonitor(lambda y: float(np.mean(np.abs(t_ref @ y - truth)) / spread))
        res_o = fl.lsqr(oq, ref["rhs"], rep["config"]["max_iters"], mon_o)
        # even on identical factors the best-iterate error is read off a
        # mid-run dip that summation order alone moves: the reference algorithm
        # with a dense instead of a CSR matvec gives 3.59e-3 (seed 0) and
        # 6.19e-4 (seed 1) against the committed 7.12e-3 / 4.63e-4, with the
        # final residual equal to 1e-11 — so the gate is that spread (x2.5)
        assert 0.4 * s["error"] <= mon_o.best_error <= 2.5 * s["error"]
        assert res_o.residual_norm == pytest.approx(s["residual_norm"], rel=1e-6)

        # device path with its own factors
        t_mat = err_of([b.r_factor for b in fs.blocks], fs.kept_columns, None)
        mon = fl.ConvergenceMonitor(lambda y: float(np.mean(np.abs(t_mat @ y - truth)) / spread))
        res = fl.lsqr(fl.precondition(fs), system.rhs, rep["config"]["max_iters"], mon)
        coeffs = fl.recover_solution(fs, res.best_solution)
        err = float(np.mean(np.abs(phi @ coeffs - truth)) / spread)
        print(f"seed {s['seed']}: same-Q best {mon_o.best_error:.6e} it {mon_o.best_iteration} | "
              f"own-Q error {err:.6e} it {mon.best_iteration} (ref {s['error']:.6e} it "
              f"{s['best_iteration']}) residual {res.residual_norm:.6e} (ref {s['residual_norm']:.6e})")
        assert res.iterations_run == s["iterations_run"]
        assert res.residual_norm == pytest.approx(s["residual_norm"], rel=1e-6)
        assert 0.4 * s["error"] <= err <= 2.5 * s["error"]


@pytest.mark.parametrize("name", ["cfg2", "cfg4"])
def test_fallback_paths_agree(fl, name, monkeypatch):
    """The two-pass LSQR kernels (used when a column does not fit on chip)
    and the direct RRQR kernel (used outside route R's bounds) give the same
    results as the default fused / blocked paths on the same input."""
    wl, ref, fb, off, sysd, fs = runs(fl, name)
    op = fl.precondition(fs)
    fused = fl.lsqr(op, sysd.rhs, 60)
    monkeypatch.setenv("FEATLSQ_LSQR", "split")
    split = fl.lsqr(op, sysd.rhs, 60)
    monkeypatch.delenv("FEATLSQ_LSQR")
    np.testing.assert_allclose([r[1] for r in split.monitor.records],
                               [r[1] for r in fused.monitor.records], rtol=1e-10)
    assert np.linalg.norm(split.solution - fused.solution) <= 1e-8 * np.linalg.norm(fused.solution)
    monkeypatch.setenv("FEATLSQ_RRQR", "direct")
    fd = fl.filter_system(sysd, wl.sigma)
    monkeypatch.delenv("FEATLSQ_RRQR")
    assert np.array_equal(fd.kept_columns, fs.kept_columns)
    for a, b in zip(fd.blocks, fs.blocks):
        assert np.linalg.norm(a.r_factor - b.r_factor) <= 1e-10 * np.linalg.norm(b.r_factor)


def test_blocked_route_sigma_zero_keeps_all(fl):
    """Route R with sigma = 0 keeps min(m, K) = K columns of every block
    (linalg.py:75-85), in LAPACK's pivot order down to the rounding floor:
    once |R_ii| / |R_00| is ~1e-16 the remaining pivots are decided by
    rounding noise in any implementation, so the order is compared while
    the reference's ratio is above 1e-12."""
    from paper_2506_17626_b200.filtering import rrqr_route
    wl, ref, fb, off, sysd, fs = runs(fl, "cfg2")
    assert rrqr_route(sysd.store.layout) == "blocked"
    full = fl.filter_system(sysd, 0.0)
    K = wl.basis.feature_count
    assert np.all(full.ranks == K)
    for j in (0, len(full.kept_list) // 2):
        got = full.kept_list[j] - j * K
        assert np.array_equal(np.sort(got), np.arange(K))
        _, _, kept_ref, _, ratios = O.qr_column_pivot(ref["blocks"][j][1], 0.0)
        n = int(np.sum(ratios > 1e-12))
        assert n >= 5 and np.array_equal(got[:n], kept_ref[:n])
