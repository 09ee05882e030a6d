"""Full-size solution parity helpers (test infrastructure, not product code).

Two LSQR runs on the SAME device-assembled BASELINE system:

* run D — the product path: device RRQR factors (route R), device LSQR;
* run L — LAPACK factors: featlsq's own `qr_column_pivot` (linalg.py:58, the
  function `filter_system` calls per block, filtering.py:100) applied on the
  host to every device-assembled block, the resulting Q-hat blocks uploaded
  and run through the same device LSQR kernels.

Both runs are snapshotted at checkpoints; at each one the solution-level
quantities of SURVEY §8(c) are compared: y, the recovered coefficients'
fitted values M a (featlsq: `GlobalSystem.apply`, assembly.py:91), the
predicted field on the test lattice (`evaluate_solution` at `make_test_set`
points, assembly.py:275/295), plus each run's residual estimate phibar, its
true residual ||Q y - b||, scipy's test-2 quantity ||Q^T r|| / (||Q||_F ||r||)
and the L1 test error (assembly.py:313).
"""

from __future__ import annotations

import os
from concurrent.futures import ThreadPoolExecutor

import numpy as np


def lapack_factors(blocks, sigma, threads=None):
    """featlsq.linalg.qr_column_pivot on every block (one BLAS thread per
    block, blocks in parallel)."""
    from featlsq import linalg as r_lin
    from threadpoolctl import threadpool_limits
    threads = threads or os.cpu_count() or 1
    with threadpool_limits(1):
        with ThreadPoolExecutor(threads) as ex:
            return list(ex.map(lambda b: r_lin.qr_column_pivot(b.matrix, sigma), blocks))


def _recover_host(pqs, y, K, J):
    import scipy.linalg
    a = np.zeros(J * K)
    o = 0
    for j, pq in enumerate(pqs):
        r = pq.kept.size
        a[j * K + pq.kept] = scipy.linalg.solve_triangular(pq.r_factor, y[o:o + r])
        o += r
    return a


def compare(name, checkpoints=(100, 1000, 3000, 10000), threads=None, log=print):
    import torch
    import paper_2506_17626_b200 as fl
    from paper_2506_17626_b200 import _device as D, solvers, workloads

    wl = workloads.build(name)
    sysd = fl.assemble(wl.problem, wl.dec, wl.basis, interior_per_dim=wl.interior_per_dim)
    fs = fl.filter_system(sysd, wl.sigma)
    op = fl.precondition(fs)
    J, K = len(fs.ranks), fs.K
    host_blocks = sysd.blocks
    pqs = lapack_factors(host_blocks, wl.sigma, threads)
    kept_same = all(np.array_equal(pq.kept, k - j * K) for j, (pq, k) in
                    enumerate(zip(pqs, fs.kept_list)))
    ref_ops = D.blocks_from_host(sysd.row_count, [b.rows for b in host_blocks],
                                 [pq.q_factor for pq in pqs])
    ts = fl.make_test_set(wl.problem, wl.dec)
    rhs = sysd.rhs
    rhs_dev = D.to_dev(rhs)
    n_q = float(fs.kept_total)           # ||Q||_F^2: orthonormal columns per block
    last = max(checkpoints)
    snaps = {}
    for tag, blocks in (("D", op.device_blocks), ("L", ref_ops)):
        run = solvers.DeviceLsqr(blocks, last)
        run.reset_state(1, track_best=False)
        run.init(rhs_dev)
        done = 0
        for c in sorted(checkpoints):
            run.iterate(done + 1, c - done)
            done = c
            st = run.read_state()
            snaps[(tag, c)] = (D.to_host(run.x)[:blocks.ncols_total].copy(), float(st.phibar))
        del run
    del host_blocks
    out = {"name": name, "kept_identical": kept_same, "J": J, "kept": int(fs.kept_total),
           "checkpoints": {}}
    for c in sorted(checkpoints):
        row = {}
        vals = {}
        for tag in ("D", "L"):
            y, ph = snaps[(tag, c)]
            if tag == "D":
                qy = op.apply(y)
                qtr = op.apply_transpose(rhs - qy)
                a = fl.recover_solution(fs, y)
            else:
                qy = D.to_host(ref_ops.apply(D.to_dev(y)))[:sysd.row_count]
                qtr = D.to_host(ref_ops.apply_t(D.to_dev(rhs - qy)))[:fs.kept_total]
                a = _recover_host(pqs, y, K, J)
            ma = fl.apply(sysd, a)
            pred = fl.evaluate_solution(wl.problem, wl.dec, wl.basis, a, ts.points)
            res = np.linalg.norm(rhs - qy)
            vals[tag] = (y, ma, pred, qy)
            row[tag] = {"phibar": ph, "residual": float(res),
                        "test2": float(np.linalg.norm(qtr) / (np.sqrt(n_q) * res)),
                        "l1_error": float(fl.l1_error(pred, ts)),
                        "ma_minus_qy": float(np.linalg.norm(ma - qy) / np.linalg.norm(qy))}

        def rel(i):
            a, b = vals["D"][i], vals["L"][i]
            return float(np.linalg.norm(a - b) / np.linalg.norm(b))
        row["rel_y"], row["rel_Ma"], row["rel_pred"], row["rel_Qy"] = rel(0), rel(1), rel(2), rel(3)
        out["checkpoints"][c] = row
        log(f"{name} it {c}: rel y {row['rel_y']:.3e} Ma {row['rel_Ma']:.3e} pred {row['rel_pred']:.3e} "
            f"Qy {row['rel_Qy']:.3e} | D phibar {row['D']['phibar']:.10e} res {row['D']['residual']:.10e} "
            f"test2 {row['D']['test2']:.2e} l1 {row['D']['l1_error']:.6e} | L phibar "
            f"{row['L']['phibar']:.10e} res {row['L']['residual']:.10e} test2 {row['L']['test2']:.2e} "
            f"l1 {row['L']['l1_error']:.6e}")
    del fs, sysd, op, ref_ops
    torch.cuda.empty_cache()
    return out
