"""Full-size converged-LSQR golden for cfg3 from the REFERENCE itself (slow, CPU).

    PYTHONPATH=/root/reference/pkg/src:/root/repo python tests/golden/make_golden_lsqr_full.py cfg3 10000

Runs the reference's own stage chain on the full BASELINE cfg3 system:
`assemble` (assembly.py:124) -> `filter_system` (filtering.py:92) ->
`precondition` (:165) -> `lsqr` (solvers.py:87, fixed budget, the paper's
10 000-iteration protocol) -> `recover_solution` (filtering.py:169), then
M.a (`apply`, assembly.py:91) and the prediction on the test
lattice (`evaluate_solution` assembly.py:273 at `make_test_set` points).

Keeps y, M.a, the test-lattice prediction, the phi-bar records every 100
iterations and scipy's test-2 quantity ||Q^T r|| / (||Q||_F ||r||) of the
final iterate, so the GPU test can tell whether the run is in the converged
regime where iterate-level parity is meaningful.
About 50 min on 8 cores (the reference's CSR SpMV is single-threaded).
"""

from __future__ import annotations

import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from featlsq import assembly as r_asm  # noqa: E402
from featlsq import filtering as r_filt  # noqa: E402
from featlsq import solvers as r_sol  # noqa: E402

from paper_2506_17626_b200 import workloads  # noqa: E402
from make_golden import to_reference  # noqa: E402


def main(name, iters):
    wl = workloads.build(name)
    prob, dec, basis = to_reference(wl)
    t0 = time.time()
    system = r_asm.assemble(prob, dec, basis, interior_per_dim=wl.interior_per_dim)
    t1 = time.time()
    fs = r_filt.filter_system(system, wl.sigma)
    t2 = time.time()
    op = r_filt.precondition(fs)
    q = op.csr()
    t3 = time.time()
    mon = r_sol.ConvergenceMonitor(stride=100)
    res = r_sol.lsqr(op, system.rhs, iters, monitor=mon)
    t4 = time.time()
    y = res.solution
    np.save(os.path.join("/tmp", f"lsqr_full_{name}_y.npy"), y)  # the expensive part, kept first
    a = r_filt.recover_solution(fs, y)
    ma = r_asm.apply(system, a)
    r = system.rhs - q @ y
    test2 = float(np.linalg.norm(q.T @ r) / (np.sqrt((q.multiply(q)).sum()) * np.linalg.norm(r)))
    ts = r_asm.make_test_set(prob, dec)
    pred = r_asm.evaluate_solution(prob, dec, basis, a, ts.points)
    rec = np.array(mon.records, dtype=float).reshape(-1, 3)
    np.savez_compressed(
        os.path.join(HERE, f"lsqr_full_{name}.npz"), y=y, ma=ma, pred=pred,
        records=rec[:, :2], iterations=res.iterations_run, residual=res.residual_norm,
        test2=test2, l1=r_asm.l1_error(pred, ts), kept=np.array([b.kept_count for b in fs.blocks]),
        max_iters=iters, assemble_s=t1 - t0, filter_s=t2 - t1, csr_s=t3 - t2,
        lsqr_s=t4 - t3)
    print(name, "iters", res.iterations_run, "phibar", res.residual_norm, "test2", test2,
          f"assemble {t1 - t0:.1f}s filter {t2 - t1:.1f}s lsqr {t4 - t3:.1f}s")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 10000)
