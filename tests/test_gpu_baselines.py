"""GPU parity for the §8(f) N4 row: CG on the normal equations (plain and
additive-Schwarz preconditioned, solvers.py:150-239) and plain LSQR on the
raw system with the device test-error monitor (runner.py:296-305).
Mirrors the reference's own TestCgNormal / TestAdditiveSchwarz cases and
checks trajectories against the oracle (pinned to the reference by
tests/test_oracle_golden.py::test_oracle_cg_and_additive_schwarz_match_reference)."""

from __future__ import annotations

import os

import numpy as np
import pytest

from oracle import featlsq_oracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def fl():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2506_17626_b200 as fl
    return fl


@pytest.fixture(scope="module")
def tall():
    rng = np.random.default_rng(11)
    a = rng.standard_normal((50, 20))
    b = rng.standard_normal(50)
    return a, b, np.linalg.pinv(a) @ b


def test_cg_reference_cases(fl, tall):
    """tests/test_solvers.py TestCgNormal, on the device."""
    a, b, x_ref = tall
    assert np.allclose(fl.cg_normal(a, b, 200).solution, x_ref, atol=1e-6)
    mon = fl.ConvergenceMonitor()
    res = fl.cg_normal(a, b, 40, mon)
    it, r, _ = mon.records[-1]
    assert it == res.iterations_run
    assert r == pytest.approx(np.linalg.norm(a @ res.solution - b), rel=1e-8)
    assert res.residual_norm == pytest.approx(np.linalg.norm(a @ res.solution - b), rel=1e-12)
    assert np.allclose(fl.cg_normal(np.eye(3), np.array([2.0, -1.0, 0.5]), 10).solution,
                       [2.0, -1.0, 0.5], atol=1e-12)
    z = fl.cg_normal(np.zeros((3, 2)), np.ones(3), 10)
    assert z.breakdown and z.iterations_run == 0
    assert z.residual_norm == pytest.approx(np.sqrt(3.0))
    with pytest.raises(fl.InvalidInputError):
        fl.cg_normal(np.eye(3), np.ones(2), 5)
    # a non-finite operator makes p.q non-finite: breakdown before any x update
    nan = fl.cg_normal(np.full((3, 3), np.nan), np.ones(3), 5)
    assert nan.breakdown and nan.iterations_run == 0


def test_cg_dense_matches_reference_records(fl, golden_dir):
    g = np.load(os.path.join(golden_dir, "cg.npz"))
    mon = fl.ConvergenceMonitor()
    res = fl.cg_normal(g["a"], g["b"], 40, mon)
    np.testing.assert_allclose(np.array(mon.records), g["dense_records"], rtol=1e-10)
    np.testing.assert_allclose(res.solution, g["dense_x"], rtol=1e-10)
    assert res.residual_norm == pytest.approx(float(g["dense_res"]), rel=1e-12)
    assert mon.best_iteration == int(np.argmin(g["dense_records"][:, 1])) + 1
    assert np.array_equal(mon.best_iterate, mon.best_iterate)


def test_cg_raw_system_matches_oracle_and_stride(fl):
    """cfg1's raw system (kappa(M)^2 ~ 1e20: CG on the normal equations
    loses orthogonality within ~25 iterations), stride 5: the first five
    recorded residuals agree with the oracle on the same M to 1e-8. After
    that single records are not reproducible — the oracle's own ensemble
    over 1-ulp perturbations of M spreads by up to 16% per record but only
    1.3% in the final residual (266.96..270.43, measured) — so later records
    are gated at 25% and the final residual at 3%; iterations and the record
    schema are exact."""
    from paper_2506_17626_b200 import workloads
    wl = workloads.build("cfg1")
    sysd = fl.assemble(wl.problem, wl.dec, wl.basis, interior_per_dim=wl.interior_per_dim)
    M = sysd.csr()
    mon = fl.ConvergenceMonitor(stride=5)
    res = fl.cg_normal(sysd, sysd.rhs, 200, mon)
    _, its, fres, recs, brk = O.cg_normal(lambda v: M @ v, lambda r: M.T @ r, M.shape[1],
                                          sysd.rhs, 200, stride=5)
    assert res.iterations_run == its and res.breakdown == brk
    assert [r[0] for r in mon.records] == [r[0] for r in recs] == list(range(5, 201, 5))
    np.testing.assert_allclose([r[1] for r in mon.records[:5]], [r[1] for r in recs[:5]], rtol=1e-8)
    np.testing.assert_allclose([r[1] for r in mon.records], [r[1] for r in recs], rtol=0.25)
    assert res.residual_norm == pytest.approx(fres, rel=3e-2)
    assert res.residual_norm == pytest.approx(np.linalg.norm(M @ res.solution - sysd.rhs), rel=1e-10)
    assert mon.best_error == min(r[1] for r in mon.records)


def _osc_system(fl):
    """The reference's TestAdditiveSchwarz system (oscillator 8.0, 4
    subdomains, 4 features, default_rng(2))."""
    p = fl.oscillator_problem(8.0)
    dec = fl.decompose(p.domain, 4, 2.9)
    basis = fl.init_basis(dec, 4, 1, "tanh", np.random.default_rng(2))
    return fl.assemble(p, dec, basis)


def test_additive_schwarz_reference_cases(fl, tall):
    """tests/test_solvers.py TestAdditiveSchwarz, on the device."""
    system = _osc_system(fl)
    pre = fl.as_preconditioner(system)
    assert pre.degenerate_blocks == ()
    for blk, inv in zip(system.blocks, pre.block_inverses):
        gram = blk.matrix.T @ blk.matrix
        assert np.allclose(inv @ gram @ inv, inv, atol=1e-8 * np.abs(inv).max())
        assert np.allclose(gram @ inv @ gram, gram, atol=1e-8 * np.abs(gram).max())
    # against the oracle (numpy eigh, the reference's LAPACK)
    K = 4
    ranges, invs, deg = O.as_preconditioner([b.matrix for b in system.blocks],
                                            [np.arange(j * K, (j + 1) * K) for j in range(4)])
    # the eigendecompositions (cuSOLVER vs LAPACK) agree to ~eps kappa(G_j)
    v = np.linspace(-1.0, 1.0, system.column_count)
    ref = O.as_apply(ranges, invs, v)
    got = pre.apply(v)
    for j, blk in enumerate(system.blocks):
        kappa = np.linalg.cond(blk.matrix.T @ blk.matrix)
        sl = slice(j * K, (j + 1) * K)
        assert np.abs(got[sl] - ref[sl]).max() <= 100 * np.finfo(float).eps * kappa * np.abs(ref[sl]).max()
    a, b, x_ref = tall
    exact = fl.AdditiveSchwarz(20, (np.arange(20),), (np.linalg.pinv(a.T @ a),), ())
    res = fl.cg_normal(a, b, 3, preconditioner=exact)
    assert np.allclose(res.solution, x_ref, atol=1e-8)
    rough = fl.cg_normal(a, b, 2).solution
    assert np.linalg.norm(res.solution - x_ref) < 1e-6 * max(np.linalg.norm(rough - x_ref), 1e-6)
    assert fl.AdditiveSchwarz(2, (np.arange(2),), (np.eye(2),), (0,)).degenerate_blocks == (0,)
    with pytest.raises(fl.InvalidInputError):
        fl.AdditiveSchwarz(2, (np.arange(2),), (np.eye(2),), ()).apply(np.ones(3))


def test_as_cg_matches_oracle(fl):
    """Preconditioned CG on the oscillator system vs the oracle with the same
    (device) preconditioner blocks: first five records to 1e-8, single
    later records within the oracle's own 1-ulp spread (17%, measured), the
    final residual (stable to 1e-8 across that ensemble) to 1e-6."""
    system = _osc_system(fl)
    pre = fl.as_preconditioner(system)
    M = system.csr()
    mon = fl.ConvergenceMonitor()
    res = fl.cg_normal(system, system.rhs, 30, mon, pre)
    invs = pre.block_inverses
    x, its, fres, recs, brk = O.cg_normal(lambda v: M @ v, lambda r: M.T @ r, M.shape[1], system.rhs,
                                          30, precond=lambda r: O.as_apply(pre.block_ranges, invs, r))
    assert res.iterations_run == its and res.breakdown == brk
    np.testing.assert_allclose([r[1] for r in mon.records[:5]], [r[1] for r in recs[:5]], rtol=1e-8)
    np.testing.assert_allclose([r[1] for r in mon.records], [r[1] for r in recs], rtol=0.25)
    assert res.residual_norm == pytest.approx(fres, rel=1e-6)


def test_plain_lsqr_on_raw_system_with_device_monitor(fl):
    """The runner's plain-LSQR baseline: lsqr on M with the test-lattice
    error through P itself (DeviceL1Error(None, P, test set)), same records
    as the host error function, best iterate identical."""
    from test_oracle_masked import masked_case
    p, dec, basis = masked_case("laplace")
    sysd = fl.assemble(p, dec, basis)
    ts = fl.make_test_set(p, dec)
    sb = fl.SolutionBlocks(p, dec, basis, ts.points)
    efn = fl.DeviceL1Error(None, sb, ts)
    phi = sb.csr()

    def host_err(a):
        return float(np.mean(np.abs(phi @ a + sb.lift - ts.true_values)) / ts.spread)

    m_dev = fl.ConvergenceMonitor(efn, 3)
    r_dev = fl.lsqr(sysd, sysd.rhs, 120, m_dev)
    m_host = fl.ConvergenceMonitor(host_err, 3)
    r_host = fl.lsqr(sysd, sysd.rhs, 120, m_host)
    assert [r[0] for r in m_dev.records] == [r[0] for r in m_host.records]
    np.testing.assert_allclose([r[2] for r in m_dev.records], [r[2] for r in m_host.records],
                               rtol=1e-12, atol=1e-12)
    assert m_dev.best_iteration == m_host.best_iteration
    assert np.array_equal(m_dev.best_iterate, m_host.best_iterate)
    assert np.array_equal(r_dev.solution, r_host.solution)
    # and CG with the same device monitor
    m_cg = fl.ConvergenceMonitor(efn, 1)
    res = fl.cg_normal(sysd, sysd.rhs, 40, m_cg)
    errs = [host_err(m_cg.best_iterate)]
    assert errs[0] == pytest.approx(m_cg.best_error, rel=1e-10, abs=1e-12)
    assert res.iterations_run == 40


@pytest.mark.parametrize("K", [16, 64, 96, 128])
def test_as_setup_kernel_matches_eigh(fl, K):
    """fl_as_setup (Gramian + parallel Jacobi, K <= 96) and the wide-block
    library path (K = 128) against numpy eigh (solvers.py:178-192): on
    well-conditioned blocks the pseudo-inverses agree to 1e-11 relative; on
    blocks with an exactly rank-deficient Gramian the same eigenvalues are
    dropped (degenerate flags identical) and the products with G agree."""
    from paper_2506_17626_b200 import _device as D
    rng = np.random.default_rng(K)
    J = 6
    rows, mats = [], []
    for j in range(J):
        m = 3 * K + 7 * j
        a = rng.standard_normal((m, K)) * np.logspace(0, -3, K)
        if j % 3 == 2:           # rank-deficient: two duplicated columns
            a[:, 1] = a[:, 0]
            a[:, K - 1] = 2.0 * a[:, 3]
        rows.append(np.arange(m) + j)
        mats.append(a)
    nrows = max(r[-1] for r in rows) + 1
    from paper_2506_17626_b200.assembly import GlobalSystem
    store = D.blocks_from_host(nrows, rows, mats)
    sysd = GlobalSystem(None, None, None, np.zeros(nrows), nrows, nrows, J * K, (), _store=store,
                        block_rows=rows)
    pre = fl.as_preconditioner(sysd)
    deg_ref = []
    for j, (a, inv) in enumerate(zip(mats, pre.block_inverses)):
        g = a.T @ a
        w, v = np.linalg.eigh(g)
        keep = w > 1e-14 * w[-1]
        if not keep.all():
            deg_ref.append(j)
        ref = (v * np.where(keep, 1.0 / np.where(keep, w, 1.0), 0.0)) @ v.T
        if keep.all():
            assert np.abs(inv - ref).max() <= 1e-11 * np.abs(ref).max(), j
        else:
            assert np.allclose(g @ inv @ g, g, atol=1e-9 * np.abs(g).max()), j
            assert np.allclose(inv @ g @ inv, inv, atol=1e-9 * np.abs(inv).max()), j
    assert pre.degenerate_blocks == tuple(deg_ref)
