"""The behaviours the reference's own assembly / filtering tests pin
(pkg/tests/test_assembly.py, test_filtering.py), exercised on the device
path: lattice placement (mask-free endpoints, cell-centred masked lattices,
no zero rows, interior overrides), block storage products and adjoint
identity, the residual oracle (M a - h equals the finite-difference residual
of the predicted field), input validation, prediction and test sets."""

from __future__ import annotations

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def fl():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2506_17626_b200 as fl
    return fl


@pytest.fixture(scope="module")
def osc(fl):
    p = fl.oscillator_problem(8.0)
    dec = fl.decompose(p.domain, 4, 2.9)
    basis = fl.init_basis(dec, 4, 1, "tanh", np.random.default_rng(0))
    return p, dec, basis, fl.assemble(p, dec, basis)


@pytest.fixture(scope="module")
def lap(fl):
    p = fl.laplace_problem(1)
    dec = fl.decompose(p.domain, 4, 2.9)
    basis = fl.init_basis(dec, 4, 1, "tanh", np.random.default_rng(1))
    return p, dec, basis, fl.assemble(p, dec, basis)


def test_lattices(fl, osc, lap):
    sysd = osc[3]
    ax = sysd.lattice_axes[0]
    assert ax.size == 16 and ax[0] == 0.0 and ax[-1] == 1.0
    for ax in lap[3].lattice_axes:           # 4 * (ceil(sqrt 4) + 1) cell centres
        assert ax.size == 12
        assert ax[0] == pytest.approx(0.5 / 12, abs=1e-15)
        assert ax[-1] == pytest.approx(1.0 - 0.5 / 12, abs=1e-15)
    assert np.linalg.norm(lap[3].materialize(), axis=1).min() > 0.0
    p, dec, basis, _ = osc
    s7 = fl.assemble(p, dec, basis, interior_per_dim=7)
    assert s7.interior_count == 7 and s7.lattice_axes[0].size == 7
    with pytest.raises(fl.InvalidInputError):
        fl.assemble(p, dec, basis, interior_per_dim=1)
    p2, dec2, basis2, _ = lap
    s69 = fl.assemble(p2, dec2, basis2, interior_per_dim=(6, 9))
    assert s69.interior_count == 54
    assert [a.size for a in s69.lattice_axes] == [6, 9]
    with pytest.raises(fl.InvalidInputError):
        fl.assemble(p2, dec2, basis2, interior_per_dim=(6, 9, 4))
    p0 = fl.oscillator_problem(60.0)
    d0 = fl.decompose(p0.domain, 20, 2.9)
    s0 = fl.assemble(p0, d0, fl.init_basis(d0, 8, 1, "tanh", np.random.default_rng(0)))
    assert s0.shape == (162, 160) and s0.interior_count == 160


def test_block_storage(fl, osc):
    _, _, basis, sysd = osc
    dense = sysd.materialize()
    rng = np.random.default_rng(7)
    for _ in range(3):
        x = rng.standard_normal(sysd.column_count)
        y = rng.standard_normal(sysd.row_count)
        assert np.allclose(fl.apply(sysd, x), dense @ x, atol=1e-12)
        assert float(y @ fl.apply(sysd, x)) == pytest.approx(float(fl.apply_transpose(sysd, y) @ x),
                                                              rel=1e-12)
    cols = np.concatenate([b.columns for b in sysd.blocks])
    assert np.array_equal(np.sort(cols), np.arange(sysd.column_count))
    for b in sysd.blocks:
        assert b.matrix.shape == (b.rows.size, b.columns.size)
    with pytest.raises(fl.InvalidInputError):
        fl.apply(sysd, np.zeros(sysd.column_count + 1))
    with pytest.raises(fl.InvalidInputError):
        fl.apply_transpose(sysd, np.zeros(sysd.row_count - 1))
    with pytest.raises(fl.CapExceededError):
        sysd.materialize(size_cap=4)


def test_residual_oracle_oscillator(fl, osc):
    """M a - h is the weighted residual of u = evaluate_solution(a):
    u'' + 4u' + 64u on the lattice (/sqrt N), u(0) - 1 and u'(0)."""
    p, dec, basis, sysd = osc
    a = np.random.default_rng(3).standard_normal(sysd.column_count)
    alg = fl.apply(sysd, a) - sysd.rhs
    t = sysd.lattice_axes[0][:, None]
    h = 1e-5

    def u(pts):
        return fl.evaluate_solution(p, dec, basis, a, pts)
    u0, up, um = u(t), u(t + h), u(t - h)
    res = ((up - 2 * u0 + um) / h ** 2 + 4.0 * (up - um) / (2 * h) + 64.0 * u0) / np.sqrt(t.size)
    assert np.allclose(alg[:t.size], res, atol=1e-5)
    z = np.zeros((1, 1))
    assert alg[t.size] == pytest.approx(float(u(z)[0] - 1.0), abs=1e-12)
    assert alg[t.size + 1] == pytest.approx(float((u(z + h)[0] - u(z - h)[0]) / (2 * h)), abs=1e-5)


def test_residual_oracle_laplace(fl, lap):
    """Masked problem: M a - h = (-lap u - f) / sqrt N with u including the mask."""
    p, dec, basis, sysd = lap
    a = np.random.default_rng(4).standard_normal(sysd.column_count)
    alg = fl.apply(sysd, a) - sysd.rhs
    mesh = np.meshgrid(*sysd.lattice_axes, indexing="ij")
    pts = np.stack([m.ravel() for m in mesh], axis=1)
    h = 1e-4

    def u(q):
        return fl.evaluate_solution(p, dec, basis, a, q)
    lapu = np.zeros(pts.shape[0])
    for ax in range(2):
        e = np.zeros(2)
        e[ax] = h
        lapu += (u(pts + e) - 2 * u(pts) + u(pts - e)) / h ** 2
    assert np.allclose(alg, (-lapu - p.forcing(pts)) / np.sqrt(pts.shape[0]), atol=1e-4)


def test_validation(fl, osc):
    p, dec, _, _ = osc
    other = fl.decompose(fl.Domain(np.array([[0.0, 2.0]])), 4, 2.9)
    with pytest.raises(fl.InvalidInputError, match="domains differ"):
        fl.assemble(p, other, fl.init_basis(other, 4, 1, "tanh", np.random.default_rng(0)))
    five = fl.decompose(p.domain, 5, 2.9)
    with pytest.raises(fl.InvalidInputError, match="different decomposition"):
        fl.assemble(p, dec, fl.init_basis(five, 4, 1, "tanh", np.random.default_rng(0)))
    rebuilt = fl.decompose(p.domain, dec.count_per_dim, dec.overlap_ratio)
    assert fl.assemble(p, rebuilt, osc[2]).shape == (18, 16)
    thin = fl.decompose(p.domain, 4, 0.5)
    with pytest.raises(fl.CoverageError):
        fl.assemble(p, thin, fl.init_basis(thin, 4, 1, "tanh", np.random.default_rng(0)))


def test_prediction_and_test_sets(fl, osc, lap):
    p, dec, basis, sysd = osc
    rng = np.random.default_rng(5)
    a = rng.standard_normal(sysd.column_count)
    pts = rng.uniform(0, 1, (40, 1))
    phi, lift = fl.solution_matrix(p, dec, basis, pts)
    assert np.allclose(phi @ a + lift, fl.evaluate_solution(p, dec, basis, a, pts), atol=1e-14)
    with pytest.raises(fl.InvalidInputError):
        fl.evaluate_solution(p, dec, basis, np.zeros(3), np.zeros((2, 1)))
    wp = fl.wave_problem(0.2)
    wd = fl.decompose(wp.domain, 4, 2.9)
    wb = fl.init_basis(wd, 4, 1, "tanh", np.random.default_rng(2))
    wpts = np.array([[0.0, 0.0, 0.0], [0.1, -0.2, 0.0]])
    got = fl.evaluate_solution(wp, wd, wb, np.zeros(wb.column_count), wpts)
    assert np.allclose(got, wp.lift_value(wpts), atol=1e-14)
    assert got[0] == pytest.approx(1.0, abs=1e-9)
    ts = fl.make_test_set(p, dec)
    assert ts.points.shape == (200, 1) and ts.points[0, 0] == 0.0 and ts.points[-1, 0] == 1.0
    assert ts.spread == pytest.approx(np.std(ts.true_values))
    assert fl.make_test_set(lap[0], lap[1]).points.shape == (576, 2)
    with pytest.raises(fl.InvalidInputError, match="exact or reference"):
        fl.make_test_set(wp, wd)
    assert fl.l1_error(ts.true_values, ts) == 0.0
    assert fl.l1_error(ts.true_values + 0.5, ts) == pytest.approx(0.5 / ts.spread, rel=1e-12)
    with pytest.raises(fl.InvalidInputError):
        fl.l1_error(ts.true_values[:-1], ts)


def test_filter_reference_cases(fl, osc):
    """tests/test_filtering.py behaviours: sigma = 0 keeps everything, kept
    sets grow as sigma shrinks and nest in pivot order, offsets partition the
    kept columns, the filtered matrix is a column subset, summary fields."""
    sysd = osc[3]
    K = osc[2].feature_count
    full = fl.filter_system(sysd, 0.0)
    assert full.kept_total == sysd.column_count and full.drop_fraction == 0.0
    prev = None
    for sigma in (1e-2, 1e-4, 1e-8):
        fs = fl.filter_system(sysd, sigma)
        if prev is not None:
            assert fs.kept_total >= prev.kept_total
            for a, b in zip(prev.kept_list, fs.kept_list):
                assert np.array_equal(b[:a.size], a)   # prefix in pivot order
        assert np.array_equal(np.diff(fs.offsets), [k.size for k in fs.kept_list])
        for k, d in zip(fs.kept_list, fs.dropped_list):
            assert np.intersect1d(k, d).size == 0 and k.size + d.size == K
        dense = sysd.materialize()
        assert np.array_equal(fs.materialize(), dense[:, fs.kept_columns])
        s = fs.summary()
        assert s["kept_total"] == fs.kept_total and s["sigma"] == sigma
        prev = fs
    op = fl.precondition(prev)
    with pytest.raises(fl.InvalidInputError):
        op.apply(np.zeros(op.shape[1] + 1))
    with pytest.raises(fl.InvalidInputError):
        op.apply_transpose(np.zeros(op.shape[0] + 1))
    with pytest.raises(fl.InvalidInputError):
        fl.recover_solution(prev, np.zeros(prev.kept_total + 1))
