"""Pin the CPU oracle against the reference's own outputs (CPU only).

Goldens come from `tests/golden/make_golden.py`, which ran the reference
package itself; `oscillator_report.json` is extracted from the reference's
committed demo artifact. Once pinned here, the oracle is the checker the
GPU parity tests use at sizes the goldens do not cover.
"""

import json
import os

import numpy as np
import pytest

from oracle import featlsq_oracle as O
from paper_2506_17626_b200 import workloads
from featlsq.basis import init_basis
from featlsq.domains import decompose
from featlsq.problems import oscillator_problem

CFGS = ["cfg1", "cfg2", "cfg3", "cfg4", "cfg5"]


def _wl(name):
    return workloads.build(name) if name == "cfg1" else workloads.build_small(name)


@pytest.fixture(scope="module")
def oracle_runs():
    cache = {}

    def get(name):
        if name not in cache:
            wl = _wl(name)
            sysd = O.assemble(wl.problem, wl.dec, wl.basis, wl.interior_per_dim)
            fb, off = O.filter_system(sysd, wl.sigma)
            cache[name] = (wl, sysd, fb, off)
        return cache[name]
    return get


@pytest.mark.parametrize("name", CFGS)
def test_assembly_matches_reference(name, oracle_runs, golden_dir):
    g = np.load(os.path.join(golden_dir, f"{name}.npz"))
    wl, sysd, _, _ = oracle_runs(name)
    assert sysd["row_count"] == int(g["row_count"])
    assert sysd["column_count"] == int(g["column_count"])
    lens = np.array([r.size for r, _ in sysd["blocks"]])
    assert np.array_equal(lens, g["block_rows_len"])
    assert np.array_equal(np.concatenate([r for r, _ in sysd["blocks"]]), g["block_rows"])
    np.testing.assert_allclose(sysd["rhs"], g["rhs"], rtol=1e-14, atol=1e-14 * np.abs(g["rhs"]).max())
    dig = np.stack([[m.sum(), np.abs(m).sum(), (m * m).sum(), np.abs(m).max()]
                    for _, m in sysd["blocks"]])
    np.testing.assert_allclose(dig[:, 1:], g["block_digest"][:, 1:], rtol=1e-13)
    for key in g.files:
        if key.startswith("block") and key.endswith("_matrix"):
            j = int(key[5:-7])
            ref = g[key]
            got = sysd["blocks"][j][1]
            assert np.abs(got - ref).max() <= 1e-13 * np.abs(ref).max()


@pytest.mark.parametrize("name", CFGS)
def test_filtering_matches_reference(name, oracle_runs, golden_dir):
    g = np.load(os.path.join(golden_dir, f"{name}.npz"))
    _, _, fb, off = oracle_runs(name)
    assert np.array_equal([b["kept"].size for b in fb], g["kept_len"])
    assert np.array_equal(np.concatenate([b["kept"] for b in fb]), g["kept"])
    assert np.array_equal(np.concatenate([b["dropped"] for b in fb]), g["dropped"])
    np.testing.assert_allclose([np.linalg.norm(b["r"]) for b in fb], g["r_fro"], rtol=1e-12)


@pytest.mark.parametrize("name", CFGS)
def test_lsqr_and_recovery_match_reference(name, oracle_runs, golden_dir):
    g = np.load(os.path.join(golden_dir, f"{name}.npz"))
    _, sysd, fb, off = oracle_runs(name)
    q = O.q_operator(fb, off, sysd["row_count"])
    x, its, phibar, brk, trace = O.lsqr(lambda v: q @ v, lambda r: q.T @ r, int(off[-1]),
                                        sysd["rhs"], int(g["lsqr_iters"]))
    assert its == int(g["lsqr_iterations_run"])
    np.testing.assert_allclose(trace, g["lsqr_records"], rtol=1e-9)
    assert np.linalg.norm(x - g["lsqr_y"]) <= 1e-8 * np.linalg.norm(g["lsqr_y"])
    a = O.recover_solution(fb, off, g["lsqr_y"], sysd["column_count"])
    ma = O.raw_operator(sysd) @ a
    assert np.linalg.norm(ma - g["m_times_a"]) <= 1e-8 * np.linalg.norm(g["m_times_a"])


def test_lapack_rule_restatement_matches_reference_qr(golden_dir):
    """qrcp_dlaqp2 (numpy restatement of LAPACK's pivot rule) reproduces the
    reference qr_column_pivot: ranks, kept sequences, R norm-wise."""
    g = np.load(os.path.join(golden_dir, "qrcp.npz"))
    for i in range(int(g["count"])):
        a, s = g[f"a{i}"], float(g[f"sigma{i}"])
        q, r, kept, dropped, _ = O.qrcp_dlaqp2(a, s)
        assert np.array_equal(kept, g[f"kept{i}"]), i
        assert np.array_equal(dropped, g[f"dropped{i}"]), i
        rr = g[f"r{i}"]
        if rr.size:
            assert np.linalg.norm(r - rr) <= 1e-10 * max(np.linalg.norm(rr), 1e-300) + 1e-300, i
            if np.linalg.norm(rr) > 0:
                assert np.abs(q.T @ q - np.eye(kept.size)).max() < 1e-12


@pytest.mark.parametrize("name", ["cfg1", "cfg2"])
def test_lapack_rule_restatement_on_workload_blocks(name, oracle_runs):
    _, sysd, fb, _ = oracle_runs(name)
    for j in (0, 3, len(fb) // 2, len(fb) - 1):
        _, r, kept, _, _ = O.qrcp_dlaqp2(sysd["blocks"][j][1], 1e-10)
        k = sysd["blocks"][j][1].shape[1]
        assert np.array_equal(kept + j * k, fb[j]["kept"])
        assert np.linalg.norm(r - fb[j]["r"]) <= 1e-10 * np.linalg.norm(fb[j]["r"])


def test_dense_lsqr_matches_reference(golden_dir):
    g = np.load(os.path.join(golden_dir, "lsqr_dense.npz"))
    a, b = g["a"], g["b"]
    x, *_ = O.lsqr(lambda v: a @ v, lambda r: a.T @ r, a.shape[1], b, 200)
    np.testing.assert_allclose(x, g["x200"], rtol=0, atol=1e-13)
    x, its, *_ = O.lsqr(lambda v: v, lambda r: r, 3, np.array([1.0, 2.0, 3.0]), 50)
    assert its == int(g["ident_iters"])


def test_oscillator_demo_seed_reproduces_committed_report(golden_dir):
    """Two seeds of the reference's committed demo (10 000 LSQR iterations,
    per-iteration test-lattice monitor) reproduce exactly."""
    rep = json.load(open(os.path.join(golden_dir, "oscillator_report.json")))
    p = oscillator_problem(60.0)
    dec = decompose(p.domain, 20, 2.9)
    for s in rep["seeds"][:2]:
        basis = init_basis(dec, 8, 1, "tanh", O.random_source(s["seed"]))
        out = O.run_rrqr_lsqr(p, dec, basis, 1e-8, rep["config"]["max_iters"])
        assert out["best_iteration"] == s["best_iteration"]
        assert out["iterations"] == s["iterations_run"]
        assert out["drop_fraction"] == pytest.approx(s["drop_fraction"], abs=1e-15)
        assert out["error"] == pytest.approx(s["error"], rel=1e-9)
        assert out["residual"] == pytest.approx(s["residual_norm"], rel=1e-9)
    assert rep["kept"] == 157


def test_oracle_cg_and_additive_schwarz_match_reference(golden_dir):
    """N4: CG on the normal equations (dense case and cfg1's raw system, plain
    and additive-Schwarz preconditioned) against the reference's own runs."""
    g = np.load(os.path.join(golden_dir, "cg.npz"))
    a, b = g["a"], g["b"]
    x, its, res, recs, brk = O.cg_normal(lambda v: a @ v, lambda r: a.T @ r, 20, b, 40)
    np.testing.assert_allclose(np.array(recs), g["dense_records"], rtol=1e-12)
    np.testing.assert_allclose(x, g["dense_x"], rtol=1e-12)
    wl = workloads.build("cfg1")
    sysd = O.assemble(wl.problem, wl.dec, wl.basis, wl.interior_per_dim)
    M = O.raw_operator(sysd)
    x, its, res, recs, _ = O.cg_normal(lambda v: M @ v, lambda r: M.T @ r, M.shape[1],
                                       sysd["rhs"], 200, stride=5)
    np.testing.assert_allclose(np.array(recs)[:, 1], g["plain_records"][:, 1], rtol=1e-6)
    K = wl.basis.feature_count
    ranges, invs, deg = O.as_preconditioner([m for _, m in sysd["blocks"]],
                                            [np.arange(j * K, (j + 1) * K) for j in range(len(sysd["blocks"]))])
    assert deg == list(g["as_degenerate"])
    v = np.linspace(-1, 1, M.shape[1])
    np.testing.assert_allclose(O.as_apply(ranges, invs, v), g["as_apply"], rtol=1e-9,
                               atol=1e-9 * np.abs(g["as_apply"]).max())
