"""How many LSQR iterations a BASELINE config needs to reach the converged
regime (scipy's test-2 quantity ||Q^T r|| / (||Q||_F ||r||) below a target),
measured on the device path with the exact quantity at checkpoints.

    python scripts/converge_probe.py cfg4 200000 20000

Q-hat has orthonormal columns per block, so ||Q||_F^2 = sum_j r_j exactly.
"""

import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2506_17626_b200 as fl  # noqa: E402
from paper_2506_17626_b200 import solvers, workloads, _device as D  # noqa: E402


def main(name, max_it, chunk):
    wl = workloads.build(name)
    sysd = fl.assemble(wl.problem, wl.dec, wl.basis, interior_per_dim=wl.interior_per_dim)
    fs = fl.filter_system(sysd, wl.sigma)
    op = fl.precondition(fs)
    qf = np.sqrt(float(fs.kept_total))
    blocks, shape = solvers.device_operator(op)
    run = solvers.DeviceLsqr(blocks, max_it)
    run.reset_state(1, track_best=False, atol=1e-16, btol=1e-16, conlim=0)
    run.init(D.to_dev(sysd.rhs))
    it = 0
    t0 = time.time()
    while it < max_it:
        run.iterate(it + 1, chunk)
        it += chunk
        st = run.read_state()
        y = D.to_host(run.x)[:shape[1]]
        r = sysd.rhs - op.apply(y)
        test2 = np.linalg.norm(op.apply_transpose(r)) / (qf * np.linalg.norm(r))
        print(f"{name} it {int(st.it)} phibar {st.phibar:.10e} test2 {test2:.3e} "
              f"istop {int(st.istop)} {time.time() - t0:.0f}s", flush=True)
        if st.done:
            break


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]), int(sys.argv[3]))
