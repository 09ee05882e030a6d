"""featlsq's OWN tests, run unmodified against the drop-in,
and the reference runner reaching the device monitor K6 through the shim.

The reference package and its test files are installed into baseline/_ref
by scripts/install_reference.py (git-ignored, shipped to the GPU box with
the repo); nothing of them is committed. Each file runs in a child pytest
with `-p paper_2506_17626_b200.pytest_plugin`, which calls
`integrate.enable()` before collection, so every `from featlsq.<module>
import <stage function>` in those files binds the device implementation.
"""

from __future__ import annotations

import json
import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "baseline", "_ref")
REF_TESTS = os.path.join(REF, "featlsq_tests")

# the reference test files that exercise the replaced stage functions
# (assembly.py:124, filtering.py:92/165/169, linalg.py:58/100, solvers.py:87/178/195)
SUITES = ["test_filtering.py", "test_solvers.py", "test_assembly.py", "test_linalg.py"]


@pytest.fixture(scope="module")
def fl():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2506_17626_b200 as fl
    return fl


@pytest.mark.parametrize("name", SUITES)
def test_reference_suite_unmodified(fl, name):
    path = os.path.join(REF_TESTS, name)
    assert os.path.exists(path), f"{path} missing: run scripts/install_reference.py"
    env = dict(os.environ)
    env["PYTHONPATH"] = os.pathsep.join([ROOT, REF, env.get("PYTHONPATH", "")])
    cmd = [sys.executable, "-m", "pytest", "-p", "paper_2506_17626_b200.pytest_plugin",
           "-p", "no:cacheprovider", "--rootdir", REF_TESTS, path]
    res = subprocess.run(cmd, capture_output=True, text=True, env=env, cwd=REF_TESTS,
                         timeout=1800)
    out = res.stdout + res.stderr
    print(out[-3000:])
    assert "featlsq stage functions -> paper_2506_17626_b200" in out, "shim not active"
    assert res.returncode == 0, out[-3000:]


def test_reference_whole_suite(fl):
    """featlsq's complete test suite (13 files: acceptance, analysis, runner,
    CLI/config, FD wave, ... — 312 tests) under its own pytest configuration
    (`pkg/pyproject.toml`: addopts "-m 'not extended'") with the drop-in
    enabled: every stage function and `run_experiment` run on the device."""
    env = dict(os.environ)
    env["PYTHONPATH"] = os.pathsep.join([ROOT, REF, env.get("PYTHONPATH", "")])
    cmd = [sys.executable, "-m", "pytest", "-p", "paper_2506_17626_b200.pytest_plugin",
           "-p", "no:cacheprovider", "--rootdir", REF_TESTS, "-m", "not extended",
           "-o", "markers=extended: long-running acceptance checks", REF_TESTS]
    res = subprocess.run(cmd, capture_output=True, text=True, env=env, cwd=REF_TESTS,
                         timeout=1800)
    out = res.stdout + res.stderr
    print(out[-2000:])
    assert "featlsq stage functions -> paper_2506_17626_b200" in out, "shim not active"
    assert res.returncode == 0, out[-3000:]
    assert " 312 passed" in out


def test_runner_uses_device_monitor(fl, golden_dir):
    """`run_experiment` on the oscillator demo config (demos/oscillator_baseline.py)
    through the shim: `runner._solve_one` builds the K6 monitor, so no iterate
    crosses PCIe — the D2H bytes of a run grow by the two per-iteration trace
    entries only (phi-bar and test error), not by x — and the report
    reproduces the committed demo report within the spread measured for the
    best-iterate error (tests/test_gpu_parity.py: x0.4..x2.5 on identical
    factors) with the drop fractions exact."""
    from featlsq import runner
    from paper_2506_17626_b200 import _device as D
    from paper_2506_17626_b200 import integrate, monitor
    rep = json.load(open(os.path.join(golden_dir, "oscillator_report.json")))
    c = rep["config"]
    integrate.enable()
    try:
        assert runner._solve_one is integrate._solve_one

        def run(iters, seeds):
            cfg = runner.ExperimentConfig(
                problem="oscillator", omega0=c["omega0"], count_per_dim=c["count_per_dim"],
                overlap=c["overlap"], features=c["features"], depth=1, activation="tanh",
                sigma=c["sigma"], solver="rrqr-lsqr", max_iters=iters, seeds=tuple(seeds),
                cond_seeds=0, label="osc")
            before = D.XFER["d2h"]
            out = runner.run_experiment(cfg)
            return out, D.XFER["d2h"] - before

        seen = []
        orig = monitor.DeviceL1Error.__init__

        def spy(self, *a, **k):
            seen.append(1)
            orig(self, *a, **k)
        monitor.DeviceL1Error.__init__ = spy
        try:
            short, d2h_short = run(2000, [0])
            full, d2h_full = run(c["max_iters"], [0])
        finally:
            monitor.DeviceL1Error.__init__ = orig
        assert len(seen) == 2, "runner did not build the device monitor"
        extra = d2h_full - d2h_short
        per_it = extra / (c["max_iters"] - 2000)
        n = rep["kept"]
        assert per_it <= 2 * 8 + 1, f"{per_it:.1f} B/iteration D2H (x is {8 * n} B)"
        s0 = rep["seeds"][0]
        got = full.seeds[0]
        assert got.drop_fraction == pytest.approx(s0["drop_fraction"], abs=1e-15)
        assert full.kept_count == rep["kept"]
        assert got.iterations_run == s0["iterations_run"]
        assert 0.4 * s0["error"] <= got.error <= 2.5 * s0["error"]
        assert len(got.records) == c["max_iters"]
        print(f"runner via shim: error {got.error:.4e} (ref {s0['error']:.4e}) best it "
              f"{got.best_iteration} (ref {s0['best_iteration']}) residual {got.residual_norm:.6e} "
              f"(ref {s0['residual_norm']:.6e}); D2H {per_it:.2f} B/iteration")
    finally:
        integrate.disable()
