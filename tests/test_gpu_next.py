"""GPU parity for the §8(f) rows: N2 hard-constrained (mask/lift) assembly
in K1, N3 device `solution_matrix`/`evaluate_solution`, N1 the device
test-lattice monitor (K6) and its best iterate. Checked against goldens from
the reference (tests/golden/masked_*.npz, laplace_report.json) and against
the oracle pinned by tests/test_oracle_masked.py.
"""

from __future__ import annotations

import json
import os

import numpy as np
import pytest

from oracle import featlsq_oracle as O

pytestmark = pytest.mark.gpu

from test_oracle_masked import CASES, masked_case  # noqa: E402


@pytest.fixture(scope="module")
def fl():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2506_17626_b200 as fl
    return fl


@pytest.mark.parametrize("name", sorted(CASES))
def test_masked_assembly_matches_reference(fl, name, golden_dir):
    g = np.load(os.path.join(golden_dir, f"masked_{name}.npz"))
    p, dec, basis = masked_case(name)
    sysd = fl.assemble(p, dec, basis)
    assert sysd.shape == (int(g["row_count"]), int(g["column_count"]))
    assert np.array_equal(np.concatenate(sysd.lattice_axes), g["axes"])
    np.testing.assert_allclose(sysd.rhs, g["rhs"], rtol=1e-13, atol=1e-14 * np.abs(g["rhs"]).max())
    blocks = sysd.blocks
    assert np.array_equal(np.concatenate([b.rows for b in blocks]), g["block_rows"])
    for k, j in enumerate(g["full_idx"]):
        ref = g[f"full{k}"]
        assert np.abs(blocks[j].matrix - ref).max() <= 1e-13 * np.abs(ref).max()
    dig = np.stack([[np.abs(b.matrix).sum(), (b.matrix ** 2).sum(), np.abs(b.matrix).max()]
                    for b in blocks])
    np.testing.assert_allclose(dig, g["block_digest"][:, 1:], rtol=1e-12)


@pytest.mark.parametrize("name", sorted(CASES))
def test_solution_matrix_matches_reference(fl, name, golden_dir):
    """N3: P at arbitrary points (assembly.py:244-272), P c + lift vs the reference."""
    g = np.load(os.path.join(golden_dir, f"masked_{name}.npz"))
    p, dec, basis = masked_case(name)
    phi, lift = fl.solution_matrix(p, dec, basis, g["points"])
    assert phi.shape == (g["points"].shape[0], basis.column_count)
    assert phi.nnz == int(g["phi_nnz"])
    np.testing.assert_array_equal(lift, g["lift"])
    scale = np.abs(g["pc"]).max()
    assert np.abs(phi @ g["c"] - g["pc"]).max() <= 1e-13 * scale
    pred = fl.evaluate_solution(p, dec, basis, g["c"], g["points"])
    assert np.abs(pred - (g["pc"] + g["lift"])).max() <= 1e-13 * scale
    with pytest.raises(fl.InvalidInputError):
        fl.evaluate_solution(p, dec, basis, g["c"][:-1], g["points"])


def test_solution_matrix_mask_free_matches_oracle(fl):
    from paper_2506_17626_b200 import workloads
    wl = workloads.build("cfg1")
    pts = np.linspace(0.0, 1.0, 777)[:, None]
    phi, lift = fl.solution_matrix(wl.problem, wl.dec, wl.basis, pts)
    ref = O.solution_csr(wl.dec, wl.basis, pts)
    assert np.array_equal(np.sort(phi.indices), np.sort(ref.indices)) and phi.nnz == ref.nnz
    assert abs(phi - ref).max() <= 1e-13 * abs(ref).max()
    assert np.array_equal(lift, np.zeros(777))


def _laplace_pipeline(fl):
    p, dec, basis = masked_case("laplace")
    sysd = fl.assemble(p, dec, basis)
    fs = fl.filter_system(sysd, 1e-8)
    ts = fl.make_test_set(p, dec)
    return p, dec, basis, sysd, fs, ts


def _oracle_t(fs, p, dec, basis, ts):
    """The runner's T = P[:, kept] S^-1 (runner.py:265-276) from the DEVICE's
    own R factors, with the reference's arithmetic (dtrtrs on I, CSR products)."""
    import scipy.linalg
    import scipy.sparse
    phi = O.solution_csr(dec, basis, ts.points, p)
    sinv = scipy.sparse.block_diag(
        [scipy.linalg.solve_triangular(b.r_factor, np.eye(b.kept_count)) for b in fs.blocks],
        format="csc")
    return (phi[:, fs.kept_columns] @ sinv).tocsr(), O.lift_values(p, ts.points)


def test_device_error_fn_matches_oracle(fl):
    """N1: e(y) through the device T equals the runner's host T e(y) to 1e-12
    (relative; here e ~ 1, the iterates are far from the solution)."""
    from paper_2506_17626_b200.monitor import test_error_fn
    p, dec, basis, sysd, fs, ts = _laplace_pipeline(fl)
    efn = test_error_fn(fs, p, dec, basis, ts)
    t_mat, lift = _oracle_t(fs, p, dec, basis, ts)
    rng = np.random.default_rng(3)
    for _ in range(3):
        y = rng.standard_normal(fs.kept_total) * 1e-2
        e_ref = float(np.mean(np.abs(t_mat @ y + lift - ts.true_values)) / ts.spread)
        assert efn(y) == pytest.approx(e_ref, rel=1e-12)


def test_device_monitor_in_loop_matches_host_monitor(fl):
    """N1: the in-loop monitor (K6) records the same errors (to 1e-12), best
    iteration and best iterate as the host path evaluating the same iterates
    with the runner's host T."""
    from paper_2506_17626_b200.monitor import test_error_fn
    p, dec, basis, sysd, fs, ts = _laplace_pipeline(fl)
    efn = test_error_fn(fs, p, dec, basis, ts)
    t_mat, lift = _oracle_t(fs, p, dec, basis, ts)

    def host_err(y):
        return float(np.mean(np.abs(t_mat @ y + lift - ts.true_values)) / ts.spread)

    op = fl.precondition(fs)
    for stride in (1, 7):
        m_dev = fl.ConvergenceMonitor(efn, stride)
        r_dev = fl.lsqr(op, sysd.rhs, 300, m_dev)
        m_host = fl.ConvergenceMonitor(host_err, stride)
        r_host = fl.lsqr(op, sysd.rhs, 300, m_host)
        assert [r[0] for r in m_dev.records] == [r[0] for r in m_host.records]
        np.testing.assert_allclose([r[1] for r in m_dev.records], [r[1] for r in m_host.records],
                                   rtol=1e-13)
        # e is spread-normalised; T y ~ 1 while e ~ 1e-3, so the two T
        # arithmetics (forward substitution vs dtrtrs(I) + CSR) agree to 1e-12 in e
        np.testing.assert_allclose([r[2] for r in m_dev.records], [r[2] for r in m_host.records],
                                   rtol=1e-12, atol=1e-12)
        assert m_dev.best_iteration == m_host.best_iteration
        assert m_dev.best_error == pytest.approx(m_host.best_error, rel=1e-12)
        assert np.array_equal(m_dev.best_iterate, m_host.best_iterate)
        assert np.array_equal(r_dev.solution, r_host.solution)


def test_laplace_demo_through_device_path(fl, golden_dir):
    """N1+N2+N3 end to end: the reference's committed laplace demo (3000
    iterations, monitor every iteration) through the device pipeline. Drop
    fraction and iteration count exact; the best
    test error and residual move with rounding, so they are
    gated a few times wider than the oracle's own 1-ulp-perturbation spread;
    the best iteration is exact, and the recovered solution's error is
    recomputed from the device coefficients."""
    from paper_2506_17626_b200.monitor import test_error_fn
    rep = json.load(open(os.path.join(golden_dir, "laplace_report.json")))
    s = rep["seeds"][0]
    p, dec, basis, sysd, fs, ts = _laplace_pipeline(fl)
    assert sysd.shape == (rep["rows"], rep["columns"]) and fs.kept_total == rep["kept"]
    assert ts.points.shape[0] == rep["test_points"]
    assert fs.drop_fraction == s["drop_fraction"]
    mon = fl.ConvergenceMonitor(test_error_fn(fs, p, dec, basis, ts), 1)
    res = fl.lsqr(fl.precondition(fs), sysd.rhs, rep["config"]["max_iters"], mon)
    assert res.iterations_run == s["iterations_run"]
    print("device laplace demo:", res.residual_norm, mon.best_error, mon.best_iteration)
    # the oracle's own 1-ulp-perturbation ensemble spans 1.5e-5 (relative) in
    # the 3000-iteration residual and 4e-6 in the best error (best iteration
    # 1032 throughout); the device Q differs from the oracle's by more (F5)
    assert res.residual_norm == pytest.approx(s["residual_norm"], rel=2e-4)
    assert mon.best_iteration == s["best_iteration"]
    assert mon.best_error == pytest.approx(s["error"], rel=1e-4)
    coeffs = fl.recover_solution(fs, res.best_solution)
    pred = fl.evaluate_solution(p, dec, basis, coeffs, ts.points)
    err = fl.l1_error(pred, ts)
    assert err == pytest.approx(mon.best_error, rel=1e-6)


@pytest.mark.parametrize("name", ["lap_sigmoid", "lap_sin", "osc_sigmoid", "osc_sin"])
def test_activations_assembly_matches_reference(fl, name, golden_dir):
    """K1 with sin / sigmoid features (basis.py:24-40) against the reference."""
    from test_oracle_masked import activation_case
    g = np.load(os.path.join(golden_dir, "activations.npz"))
    p, dec, basis = activation_case(name)
    sysd = fl.assemble(p, dec, basis)
    assert np.array_equal(np.concatenate([b.rows for b in sysd.blocks]), g[name + "_rows"])
    np.testing.assert_allclose(sysd.rhs, g[name + "_rhs"], rtol=1e-13,
                               atol=1e-14 * np.abs(g[name + "_rhs"]).max())
    vals = np.concatenate([b.matrix.ravel() for b in sysd.blocks])
    assert np.abs(vals - g[name + "_vals"]).max() <= 1e-13 * np.abs(g[name + "_vals"]).max()


def test_assembly_layout_cache_keyed_by_geometry():
    """The cached lattice row structure is reused only for identical geometry:
    a decomposition with another overlap gets its own rows (and the assembled
    system matches a fresh, uncached assembly)."""
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2506_17626_b200 as fl
    from paper_2506_17626_b200 import assembly as A, workloads
    from paper_2506_17626_b200.domains import decompose
    wl = workloads.build("cfg1")
    s1 = fl.assemble(wl.problem, wl.dec, wl.basis, interior_per_dim=wl.interior_per_dim)
    s2 = fl.assemble(wl.problem, wl.dec, wl.basis, interior_per_dim=wl.interior_per_dim)
    assert [r.tolist() for r in s1.block_rows] == [r.tolist() for r in s2.block_rows]
    A._LAYOUT_CACHE.clear()
    s3 = fl.assemble(wl.problem, wl.dec, wl.basis, interior_per_dim=wl.interior_per_dim)
    assert [r.tolist() for r in s1.block_rows] == [r.tolist() for r in s3.block_rows]
    np.testing.assert_array_equal(s1.rhs, s3.rhs)
    # another overlap: different supports, so different rows
    dec2 = decompose(wl.dec.domain, wl.dec.count_per_dim, wl.dec.overlap_ratio * 1.3)
    k1 = A._cached_layout(wl.problem, wl.dec, s1.lattice_axes, [a.size for a in s1.lattice_axes], 64, [])
    k2 = A._cached_layout(wl.problem, dec2, s1.lattice_axes, [a.size for a in s1.lattice_axes], 64, [])
    assert k1[-1] is not k2[-1]
    assert sum(r.size for r in k2[5]) > sum(r.size for r in k1[5])
