"""The plug-in boundary on the host (no GPU needed): the drop-in's value
types and exceptions ARE featlsq's, `integrate.enable()` rebinds exactly the
stage functions in every featlsq namespace that holds them (runner.py:34-43)
and `disable()` restores them, and the bench's featlsq sampler (reference
arm) runs featlsq's own stage functions on a stratified block sample."""

from __future__ import annotations

import importlib

import numpy as np
import pytest

import featlsq
import paper_2506_17626_b200 as fl
from paper_2506_17626_b200 import errors, integrate


def test_value_types_and_errors_are_featlsq_own():
    assert fl.ConvergenceMonitor is featlsq.ConvergenceMonitor
    assert fl.Operator is featlsq.Operator
    assert fl.decompose is featlsq.decompose
    assert fl.FeatureBasis is featlsq.FeatureBasis
    assert fl.laplace_problem is featlsq.laplace_problem
    assert fl.SubdomainBlock is featlsq.assembly.SubdomainBlock
    assert fl.make_test_set is featlsq.make_test_set
    assert issubclass(fl.SolveResult, featlsq.SolveResult)
    for name in ("InvalidInputError", "SingularFactorError", "CapExceededError", "CoverageError",
                 "DegenerateSubdomainError", "DivergenceError"):
        assert getattr(errors, name) is getattr(featlsq.errors, name)


def test_enable_rebinds_and_disable_restores():
    mods = {m: importlib.import_module(f"featlsq.{m}")
            for m in ("assembly", "filtering", "solvers", "linalg", "runner")}
    before = {(m, n): getattr(mod, n) for m, mod in mods.items() for n in dir(mod)
              if n in integrate._NAMES or n == "_solve_one"}
    integrate.enable()
    try:
        assert integrate.enabled()
        for name, where in integrate._NAMES.items():
            for m in where:
                assert getattr(mods[m], name) is getattr(fl, name), (m, name)
            if hasattr(featlsq, name):
                assert getattr(featlsq, name) is getattr(fl, name)
        assert mods["runner"]._solve_one is integrate._solve_one
        # the names the runner binds at import (runner.py:34-43)
        for name in ("assemble", "filter_system", "precondition", "recover_solution", "lsqr",
                     "cg_normal", "as_preconditioner", "solution_matrix"):
            assert getattr(mods["runner"], name).__module__.startswith("paper_2506_17626_b200")
        integrate.enable()  # idempotent
    finally:
        integrate.disable()
    assert not integrate.enabled()
    for (m, n), obj in before.items():
        assert getattr(mods[m], n) is obj, (m, n)


def test_reference_sampler_runs_featlsq_stages():
    import bench
    from paper_2506_17626_b200 import workloads
    wl = workloads.build("cfg1")
    out = bench.ref_sample(wl, 100, 2, seed=3)
    assert out["kind"] == "reference" and out["value"] > 0
    st = out["stages"]
    assert len(st["sample_blocks"]) == 4          # 2 interior + 2 boundary (1-D strata)
    assert st["solve_s"] > 0 and st["lsqr_ms_per_iter"] > 0
    # the decomposition view: featlsq's assemble on the sample sees only it
    sd = bench.SampledDecomposition(wl.dec, [3, 7])
    assert sd.subdomain_count == 2 and sd.multi_index(1) == wl.dec.multi_index(7)
    assert sd.count_per_dim == wl.dec.count_per_dim
    assert np.array_equal(sd.centers, wl.dec.centers)
    # both bench arms describe the workload with the same helper: the
    # reference arm's row count (featlsq's own) is the product arm's
    ref = featlsq.assembly.assemble(wl.problem, wl.dec, wl.basis, interior_per_dim=wl.interior_per_dim)
    assert out["rows"] == ref.row_count

    class A:
        config = "cfg1"
    cfg = bench.config_of(A, wl, 100, 1, out["rows"])
    assert set(cfg) == {"workload", "lsqr_iters_per_solve", "sigma", "rows", "cols", "l2", "parallelism"}
    assert cfg["rows"] == ref.row_count and cfg["cols"] == ref.column_count


def test_install_reference_is_git_ignored():
    import os
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    ignored = open(os.path.join(root, ".gitignore")).read().split()
    assert "baseline/_ref/" in ignored
    if os.path.exists(os.path.join(root, ".gpurunignore")):
        assert "baseline" not in open(os.path.join(root, ".gpurunignore")).read()


@pytest.mark.parametrize("name", ["cfg1", "cfg2", "cfg3", "cfg5"])
def test_block_rows_work_model_matches_assembly(name):
    """bench._block_rows (the reference arm's work model) counts the same
    rows per block as featlsq's assemble does (reduced sizes for 2-D/3-D)."""
    import bench
    from paper_2506_17626_b200 import workloads
    wl = workloads.build(name) if name in ("cfg1", "cfg2") else workloads.build_small(name)
    m, _ = bench._block_rows(wl)
    ref = featlsq.assembly.assemble(wl.problem, wl.dec, wl.basis, interior_per_dim=wl.interior_per_dim)
    assert np.array_equal(m, [b.rows.size for b in ref.blocks])
