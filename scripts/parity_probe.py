"""Diagnostic: how closely does the device path track the oracle on each
small config? Prints operator-product, LSQR-trajectory and prediction
agreement for (a) the device's own Q vs the oracle's Q and (b) the device
LSQR run on the oracle's Q (isolates LSQR arithmetic). Not a test."""

import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import featlsq_oracle as O  # noqa: E402
import paper_2506_17626_b200 as fl  # noqa: E402
from paper_2506_17626_b200 import _device as D, workloads  # noqa: E402


def rel(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def main(names, iters):
    for name in names:
        wl = workloads.build(name) if name == "cfg1" else workloads.build_small(name)
        ref = O.assemble(wl.problem, wl.dec, wl.basis, wl.interior_per_dim)
        fb, off = O.filter_system(ref, wl.sigma)
        q = O.q_operator(fb, off, ref["row_count"])
        M = O.raw_operator(ref)
        sysd = fl.assemble(wl.problem, wl.dec, wl.basis, interior_per_dim=wl.interior_per_dim)
        fs = fl.filter_system(sysd, wl.sigma)
        op = fl.precondition(fs)
        qd = op.csr()
        rng = np.random.default_rng(0)
        y = rng.standard_normal(op.shape[1])
        print(f"== {name} shape {sysd.shape} kept {fs.kept_total}")
        print(f"  apply: own-Q {rel(op.apply(y), qd @ y):.2e}  vs oracle-Q {rel(op.apply(y), q @ y):.2e}")
        qmax = max(np.abs(b.q_factor - ob['q']).max() for b, ob in zip(fs.blocks, fb))
        print(f"  max |Q_dev - Q_oracle| = {qmax:.2e}")
        oq = D.blocks_from_host(ref["row_count"], [b["rows"] for b in fb], [b["q"] for b in fb])
        for its in iters:
            t0 = time.perf_counter()
            xo, _, pho, _, tro = O.lsqr(lambda v: q @ v, lambda r: q.T @ r, q.shape[1], ref["rhs"], its)
            t_cpu = time.perf_counter() - t0
            rd = fl.lsqr(op, sysd.rhs, its)
            ro = fl.lsqr(oq, ref["rhs"], its)
            tr_d = np.array([r[1] for r in rd.monitor.records])
            tr_o = np.array([r[1] for r in ro.monitor.records])
            ma_o = M @ O.recover_solution(fb, off, xo, ref["column_count"])
            ma_d = M @ fl.recover_solution(fs, rd.solution)
            print(f"  its {its:6d}: sameQ y {rel(ro.solution, xo):.2e} trace {np.abs(tr_o/np.array(tro)-1).max():.2e} | "
                  f"ownQ y {rel(rd.solution, xo):.2e} trace {np.abs(tr_d/np.array(tro)-1).max():.2e} "
                  f"Ma {rel(ma_d, ma_o):.2e} | phibar {pho:.3e} cpu {t_cpu:.2f}s")


if __name__ == "__main__":
    names = sys.argv[1].split(",") if len(sys.argv) > 1 else ["cfg1", "cfg2", "cfg3", "cfg4", "cfg5"]
    iters = [int(x) for x in sys.argv[2].split(",")] if len(sys.argv) > 2 else [100, 300, 3000]
    main(names, iters)
