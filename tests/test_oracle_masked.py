"""Oracle pinning for the §8(f) rows (CPU): hard-constrained (mask/lift)
assembly, the solution matrix at test points, and the test-lattice monitor.

tests/golden/masked_{laplace,wave}.npz come from the reference itself
(tests/golden/make_golden.py masked); laplace_report.json is extracted from
the reference's committed demo artifact
(pkg/demos/out/laplace/laplace-multiscale/report.json).
"""

import json
import os

import numpy as np
import pytest

from oracle import featlsq_oracle as O
from featlsq.basis import init_basis
from featlsq.domains import decompose
from featlsq.problems import laplace_problem, wave_problem

CASES = {"laplace": (lambda: laplace_problem(3), 16, 2.9, 16),
         "wave": (lambda: wave_problem(0.4), 4, 2.9, 8)}


def masked_case(name):
    make, S, ov, K = CASES[name]
    p = make()
    dec = decompose(p.domain, S, ov)
    basis = init_basis(dec, K, 1, "tanh", O.random_source(0))
    return p, dec, basis


@pytest.mark.parametrize("name", sorted(CASES))
def test_masked_inputs_match_reference(name, golden_dir):
    g = np.load(os.path.join(golden_dir, f"masked_{name}.npz"))
    p, dec, basis = masked_case(name)
    assert np.array_equal(basis.weights[0], g["w"]) and np.array_equal(basis.biases[0], g["b"])


@pytest.mark.parametrize("name", sorted(CASES))
def test_oracle_masked_assembly_matches_reference(name, golden_dir):
    g = np.load(os.path.join(golden_dir, f"masked_{name}.npz"))
    p, dec, basis = masked_case(name)
    sysd = O.assemble(p, dec, basis, None)
    assert np.array_equal(np.concatenate(sysd["axes"]), g["axes"])
    assert sysd["row_count"] == int(g["row_count"])
    assert np.array_equal(np.array([r.size for r, _ in sysd["blocks"]]), g["block_rows_len"])
    assert np.array_equal(np.concatenate([r for r, _ in sysd["blocks"]]), g["block_rows"])
    np.testing.assert_allclose(sysd["rhs"], g["rhs"], rtol=1e-13, atol=1e-14 * np.abs(g["rhs"]).max())
    for k, j in enumerate(g["full_idx"]):
        ref = g[f"full{k}"]
        assert np.abs(sysd["blocks"][j][1] - ref).max() <= 1e-13 * np.abs(ref).max()
    dig = np.stack([[m.sum(), np.abs(m).sum(), (m * m).sum(), np.abs(m).max()]
                    for _, m in sysd["blocks"]])
    np.testing.assert_allclose(dig[:, 1:], g["block_digest"][:, 1:], rtol=1e-12)


@pytest.mark.parametrize("name", sorted(CASES))
def test_oracle_solution_matrix_matches_reference(name, golden_dir):
    g = np.load(os.path.join(golden_dir, f"masked_{name}.npz"))
    p, dec, basis = masked_case(name)
    phi = O.solution_csr(dec, basis, g["points"], p)
    assert phi.nnz == int(g["phi_nnz"])
    lift = O.lift_values(p, g["points"])
    np.testing.assert_array_equal(lift, g["lift"])
    scale = np.abs(g["pc"]).max()
    assert np.abs(phi @ g["c"] - g["pc"]).max() <= 1e-13 * scale


def test_laplace_demo_reproduces_committed_report(golden_dir):
    """The reference's committed laplace demo (masked assembly, 3000 LSQR
    iterations, per-iteration test-lattice monitor) reproduces exactly."""
    rep = json.load(open(os.path.join(golden_dir, "laplace_report.json")))
    p, dec, basis = masked_case("laplace")
    s = rep["seeds"][0]
    out = O.run_rrqr_lsqr(p, dec, basis, rep["config"]["sigma"], rep["config"]["max_iters"])
    assert out["best_iteration"] == s["best_iteration"]
    assert out["iterations"] == s["iterations_run"]
    assert out["drop_fraction"] == s["drop_fraction"]
    assert out["error"] == pytest.approx(s["error"], rel=1e-12)
    assert out["residual"] == pytest.approx(s["residual_norm"], rel=1e-12)


ACT_CASES = {"osc_sin": ("osc", "sin"), "osc_sigmoid": ("osc", "sigmoid"),
             "lap_sigmoid": ("lap", "sigmoid"), "lap_sin": ("lap", "sin")}


def activation_case(name):
    from featlsq.problems import oscillator_problem
    kind, act = ACT_CASES[name]
    if kind == "osc":
        p, S, K = oscillator_problem(60.0), 20, 8
    else:
        p, S, K = laplace_problem(3), 4, 16
    dec = decompose(p.domain, S, 2.9)
    return p, dec, init_basis(dec, K, 1, act, O.random_source(0))


@pytest.mark.parametrize("name", sorted(ACT_CASES))
def test_oracle_activations_match_reference(name, golden_dir):
    """sin / sigmoid feature jets (basis.py:24-40) through the oracle's
    assembly against the reference's."""
    g = np.load(os.path.join(golden_dir, "activations.npz"))
    p, dec, basis = activation_case(name)
    sysd = O.assemble(p, dec, basis, None)
    assert np.array_equal(np.concatenate([r for r, _ in sysd["blocks"]]), g[name + "_rows"])
    np.testing.assert_allclose(sysd["rhs"], g[name + "_rhs"], rtol=1e-13,
                               atol=1e-14 * np.abs(g[name + "_rhs"]).max())
    vals = np.concatenate([m.ravel() for _, m in sysd["blocks"]])
    assert np.abs(vals - g[name + "_vals"]).max() <= 1e-13 * np.abs(g[name + "_vals"]).max()
