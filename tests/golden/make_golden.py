"""Generate the golden fixtures by running the REFERENCE package itself.

Run in the build container (where /root/reference exists):

    PYTHONPATH=/root/reference/pkg/src:/root/repo python tests/golden/make_golden.py

Writes tests/golden/*.npz. The GPU box never runs this; tests only read the
committed .npz files. Inputs are rebuilt from `paper_2506_17626_b200.workloads`
with fixed seeds, converted to the reference's own value types, and pushed
through the reference stage API (`assemble` assembly.py:124, `filter_system`
filtering.py:92, `precondition` :165, `lsqr` solvers.py:87,
`recover_solution` filtering.py:169, `qr_column_pivot` linalg.py:58).
"""

from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

import featlsq  # noqa: E402
from featlsq import assembly as r_asm  # noqa: E402
from featlsq import basis as r_basis  # noqa: E402
from featlsq import domains as r_dom  # noqa: E402
from featlsq import filtering as r_filt  # noqa: E402
from featlsq import linalg as r_lin  # noqa: E402
from featlsq import problems as r_prob  # noqa: E402
from featlsq import solvers as r_sol  # noqa: E402

from paper_2506_17626_b200 import workloads  # noqa: E402

LSQR_ITERS = 300


def to_reference(wl):
    """Rebuild a workload with the reference's own classes."""
    p = wl.problem
    dom = r_dom.Domain(p.domain.bounds)
    dec = r_dom.decompose(dom, wl.dec.count_per_dim, wl.dec.overlap_ratio)
    op = lambda o: r_prob.LinearOperator2(o.value_coef, o.first_coefs, o.second_coefs)  # noqa
    cons = tuple(r_prob.ConstraintRows(c.label, op(c.operator), c.points, c.targets, c.weight)
                 for c in p.constraints)
    prob = r_prob.ProblemSpec(p.name, dom, op(p.operator), p.forcing, cons,
                              exact=p.exact, test_points_per_count=p.test_points_per_count)
    b = wl.basis
    basis = r_basis.FeatureBasis(dec, b.feature_count, 1, b.activation, b.weights, b.biases)
    return prob, dec, basis


def block_digest(mat):
    """Size-independent fingerprints of one block."""
    m = np.asarray(mat)
    return np.array([m.sum(), np.abs(m).sum(), (m * m).sum(), np.abs(m).max()])


def workload_golden(name, wl, full_blocks=()):
    prob, dec, basis = to_reference(wl)
    system = r_asm.assemble(prob, dec, basis, interior_per_dim=wl.interior_per_dim)
    fs = r_filt.filter_system(system, wl.sigma)
    op = r_filt.precondition(fs)
    res = r_sol.lsqr(op, system.rhs, LSQR_ITERS)
    coeffs = r_filt.recover_solution(fs, res.solution)
    out = dict(
        rhs=system.rhs, row_count=system.row_count, column_count=system.column_count,
        block_rows_len=np.array([b.rows.size for b in system.blocks]),
        block_rows=np.concatenate([b.rows for b in system.blocks]),
        block_digest=np.stack([block_digest(b.matrix) for b in system.blocks]),
        kept_len=np.array([b.kept_count for b in fs.blocks]),
        kept=np.concatenate([b.kept_columns for b in fs.blocks]),
        dropped=np.concatenate([b.dropped_columns for b in fs.blocks]),
        r_fro=np.array([np.linalg.norm(b.r_factor) for b in fs.blocks]),
        r_diag=np.concatenate([np.diag(b.r_factor) for b in fs.blocks]),
        lsqr_iters=LSQR_ITERS, lsqr_y=res.solution, lsqr_phibar=res.residual_norm,
        lsqr_records=np.array([r[1] for r in res.monitor.records]),
        lsqr_iterations_run=res.iterations_run, coeffs=coeffs,
        m_times_a=r_asm.apply(system, coeffs),
        sigma=wl.sigma,
    )
    for j in full_blocks:
        out[f"block{j}_matrix"] = system.blocks[j].matrix
        out[f"block{j}_q"] = fs.blocks[j].q_factor
        out[f"block{j}_r"] = fs.blocks[j].r_factor
    np.savez_compressed(os.path.join(HERE, f"{name}.npz"), **out)
    print(name, system.shape, "kept", fs.kept_total, "drop", round(fs.drop_fraction, 4))


def qr_golden():
    """Reference qr_column_pivot on seeded matrices exercising the pivot rule:
    gapped spectra, duplicate columns, exact ties, zero and wide matrices."""
    rng = np.random.default_rng(2024)
    cases = []

    def spectrum(rows, cols, svals):
        u, _ = np.linalg.qr(rng.standard_normal((rows, cols)))
        v, _ = np.linalg.qr(rng.standard_normal((cols, cols)))
        return (u * np.asarray(svals)) @ v.T
    for t in range(24):
        rows = int(rng.integers(10, 90))
        cols = int(rng.integers(4, min(rows, 70) + 1))
        rank = int(rng.integers(1, cols + 1))
        sv = np.empty(cols)
        sv[:rank] = rng.uniform(0.5, 2.0, rank)
        sv[rank:] = 1e-6 * 10.0 ** rng.uniform(-4, -1, cols - rank)
        cases.append((spectrum(rows, cols, np.sort(sv)[::-1]), 1e-6))
    base = rng.standard_normal((12, 5))
    cases.append((np.concatenate([base, base[:, 2:3]], axis=1), 1e-8))   # duplicate column
    cases.append((np.diag([1.0, 0.5, 0.25]), 0.5))                        # tie at threshold
    cases.append((np.zeros((5, 3)), 1e-8))                                # zero matrix
    cases.append((np.zeros((5, 3)), 0.0))                                 # zero, sigma 0
    cases.append((rng.standard_normal((6, 11)), 1e-3))                    # wide
    cases.append((np.ones((7, 4)), 1e-8))                                 # all-equal norms
    cases.append((rng.standard_normal((40, 40)), 0.0))                    # square, sigma 0
    out = {}
    for i, (a, s) in enumerate(cases):
        pq = r_lin.qr_column_pivot(a, s)
        out[f"a{i}"] = a
        out[f"sigma{i}"] = s
        out[f"kept{i}"] = pq.kept
        out[f"dropped{i}"] = pq.dropped
        out[f"r{i}"] = pq.r_factor
        out[f"q{i}"] = pq.q_factor
    out["count"] = len(cases)
    np.savez_compressed(os.path.join(HERE, "qrcp.npz"), **out)
    print("qrcp cases", len(cases))


def lsqr_golden():
    rng = np.random.default_rng(11)
    a = rng.standard_normal((50, 20))
    b = rng.standard_normal(50)
    res = r_sol.lsqr(a, b, 200)
    res60 = r_sol.lsqr(a, b, 60)
    ident = r_sol.lsqr(np.eye(3), np.array([1.0, 2.0, 3.0]), 50)
    np.savez_compressed(os.path.join(HERE, "lsqr_dense.npz"), a=a, b=b, x200=res.solution,
                        x60=res60.solution, phibar60=res60.residual_norm,
                        ident_iters=ident.iterations_run, ident_x=ident.solution)


def oscillator_golden():
    """The reference's own demo config, one seed, through the reference stages
    (the committed report.json pins the full 5-seed run)."""
    prob = r_prob.oscillator_problem(60.0)
    dec = r_dom.decompose(prob.domain, 20, 2.9)
    basis = r_basis.init_basis(dec, 8, 1, "tanh", r_lin.RandomSource(0).generator())
    system = r_asm.assemble(prob, dec, basis)
    fs = r_filt.filter_system(system, 1e-8)
    res = r_sol.lsqr(r_filt.precondition(fs), system.rhs, 2000)
    np.savez_compressed(
        os.path.join(HERE, "oscillator_seed0.npz"),
        w=basis.weights[0], b=basis.biases[0], rhs=system.rhs,
        kept=np.concatenate([b.kept_columns for b in fs.blocks]),
        kept_len=np.array([b.kept_count for b in fs.blocks]),
        matrix=np.concatenate([b.matrix.ravel() for b in system.blocks]),
        y2000=res.solution, phibar2000=res.residual_norm)


def demo_report_golden():
    """Per-seed numbers of the reference's committed oscillator demo run
    (pkg/demos/out/oscillator/oscillator-baseline/report.json)."""
    import json
    src = os.path.join(os.path.dirname(os.path.dirname(featlsq.__file__)), "..", "demos",
                       "out", "oscillator", "oscillator-baseline", "report.json")
    with open(src) as fh:
        rep = json.load(fh)
    keep = dict(rows=rep["rows"], columns=rep["columns"], kept=rep["kept"],
                config={k: rep["config"][k] for k in
                        ("omega0", "count_per_dim", "overlap", "features", "sigma",
                         "max_iters", "seeds")},
                seeds=[{k: s[k] for k in ("seed", "error", "best_iteration", "iterations_run",
                                          "residual_norm", "drop_fraction")}
                       for s in rep["seeds"]])
    with open(os.path.join(HERE, "oscillator_report.json"), "w") as fh:
        json.dump(keep, fh, indent=1)


def masked_golden():
    """Hard-constrained problems through the reference: the laplace demo
    config (pkg/demos/out/laplace/laplace-multiscale, seed 0) and a small
    wave problem (mask x ramp plus Gaussian-pulse lift): assembly digests,
    rhs, two full blocks, and P c + lift at the test points for a fixed c."""
    import json
    cases = {
        "laplace": (r_prob.laplace_problem(3), 16, 2.9, 16, None),
        "wave": (r_prob.wave_problem(0.4), 4, 2.9, 8, None),
    }
    for name, (prob, S, ov, K, ipd) in cases.items():
        dec = r_dom.decompose(prob.domain, S, ov)
        basis = r_basis.init_basis(dec, K, 1, "tanh", r_lin.RandomSource(0).generator())
        system = r_asm.assemble(prob, dec, basis, interior_per_dim=ipd)
        if name == "laplace":
            ts = r_asm.make_test_set(prob, dec)
            pts = ts.points
        else:
            rng = np.random.default_rng(5)
            pts = np.column_stack([rng.uniform(-0.95, 0.95, (600, 2)), rng.uniform(0.02, 0.98, 600)])
        phi, lift = r_asm.solution_matrix(prob, dec, basis, pts)
        c = np.random.default_rng(7).standard_normal(basis.column_count)
        full = (0, len(system.blocks) // 2)
        np.savez_compressed(
            os.path.join(HERE, f"masked_{name}.npz"),
            w=basis.weights[0], b=basis.biases[0], rhs=system.rhs, axes=np.concatenate(system.lattice_axes),
            row_count=system.row_count, column_count=system.column_count,
            block_rows_len=np.array([b.rows.size for b in system.blocks]),
            block_rows=np.concatenate([b.rows for b in system.blocks]),
            block_digest=np.stack([block_digest(b.matrix) for b in system.blocks]),
            full_idx=np.array(full), full0=system.blocks[full[0]].matrix, full1=system.blocks[full[1]].matrix,
            points=pts, pc=phi @ c, lift=lift, c=c, phi_nnz=phi.nnz,
            phi_digest=np.array([phi.data.sum(), np.abs(phi.data).sum(), (phi.data ** 2).sum()]))
    src = os.path.join(os.path.dirname(os.path.dirname(featlsq.__file__)), "..", "demos",
                       "out", "laplace", "laplace-multiscale", "report.json")
    with open(src) as fh:
        rep = json.load(fh)
    keep = dict(rows=rep["rows"], columns=rep["columns"], kept=rep["kept"],
                test_points=rep["test_points"],
                config={k: rep["config"][k] for k in
                        ("scale_count", "count_per_dim", "overlap", "features", "sigma",
                         "max_iters", "seeds", "eval_stride")},
                seeds=[{k: s[k] for k in ("seed", "error", "best_iteration", "iterations_run",
                                          "residual_norm", "drop_fraction")}
                       for s in rep["seeds"]])
    with open(os.path.join(HERE, "laplace_report.json"), "w") as fh:
        json.dump(keep, fh, indent=1)


def cg_golden():
    """CG on the normal equations and the additive-Schwarz preconditioner
    through the reference (solvers.py:150-239): a dense well-conditioned
    case and cfg1's raw system (plain, and with AS), 200 iterations each."""
    rng = np.random.default_rng(11)
    a = rng.standard_normal((50, 20))
    b = rng.standard_normal(50)
    dense = r_sol.cg_normal(a, b, 40, r_sol.ConvergenceMonitor())
    wl = workloads.build("cfg1")
    prob, dec, basis = to_reference(wl)
    system = r_asm.assemble(prob, dec, basis, interior_per_dim=wl.interior_per_dim)
    pre = r_sol.as_preconditioner(system)
    plain = r_sol.cg_normal(system, system.rhs, 200, r_sol.ConvergenceMonitor(stride=5))
    asc = r_sol.cg_normal(system, system.rhs, 200, r_sol.ConvergenceMonitor(), pre)
    np.savez_compressed(
        os.path.join(HERE, "cg.npz"), a=a, b=b, dense_x=dense.solution,
        dense_records=np.array(dense.monitor.records), dense_res=dense.residual_norm,
        plain_x=plain.solution, plain_records=np.array(plain.monitor.records),
        plain_res=plain.residual_norm, plain_best_it=plain.monitor.best_iteration,
        as_x=asc.solution, as_records=np.array(asc.monitor.records), as_res=asc.residual_norm,
        as_degenerate=np.array(pre.degenerate_blocks, dtype=np.int64),
        as_apply=pre.apply(np.linspace(-1, 1, system.column_count)))


def activations_golden():
    """sin and sigmoid feature networks (basis.py:24-40) through the reference
    assembly: 1D soft-constrained oscillator and 2D masked laplace."""
    cases = {
        "osc_sin": (r_prob.oscillator_problem(60.0), 20, 2.9, 8, "sin"),
        "osc_sigmoid": (r_prob.oscillator_problem(60.0), 20, 2.9, 8, "sigmoid"),
        "lap_sigmoid": (r_prob.laplace_problem(3), 4, 2.9, 16, "sigmoid"),
        "lap_sin": (r_prob.laplace_problem(3), 4, 2.9, 16, "sin"),
    }
    out = {}
    for name, (prob, S, ov, K, act) in cases.items():
        dec = r_dom.decompose(prob.domain, S, ov)
        basis = r_basis.init_basis(dec, K, 1, act, r_lin.RandomSource(0).generator())
        system = r_asm.assemble(prob, dec, basis)
        out[name + "_rhs"] = system.rhs
        out[name + "_rows"] = np.concatenate([b.rows for b in system.blocks])
        out[name + "_vals"] = np.concatenate([b.matrix.ravel() for b in system.blocks])
    np.savez_compressed(os.path.join(HERE, "activations.npz"), **out)


if __name__ == "__main__":
    if sys.argv[1:] == ["activations"]:
        activations_golden()
        sys.exit(0)
    if sys.argv[1:] == ["masked"]:
        masked_golden()
        sys.exit(0)
    if sys.argv[1:] == ["cg"]:
        cg_golden()
        sys.exit(0)
    cg_golden()
    activations_golden()
    masked_golden()
    demo_report_golden()
    print("reference featlsq", featlsq.__version__, "from", featlsq.__file__)
    for name in ("cfg1", "cfg2", "cfg3", "cfg4", "cfg5"):
        wl = workloads.build(name) if name == "cfg1" else workloads.build_small(name)
        workload_golden(name, wl, full_blocks=(0, 7) if name in ("cfg1", "cfg2") else ())
    qr_golden()
    lsqr_golden()
    oscillator_golden()
