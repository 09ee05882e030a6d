"""Full-size goldens for cfg3/cfg4/cfg5 from the REFERENCE itself (slow, CPU).

    PYTHONPATH=/root/reference/pkg/src:/root/repo python tests/golden/make_golden_full.py cfg4

Runs the reference's `assemble` (assembly.py:124) and, block by block, the
reference's `qr_column_pivot` (linalg.py:58, exactly what filter_system
filtering.py:92-115 calls per block), keeping only per-block ranks, the kept
sequences (int16, pivot order) and ||R_j||_F — enough to check exact
kept-sequence parity of the device RRQR at BASELINE size without storing the
matrices.
"""

from __future__ import annotations

import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from featlsq import assembly as r_asm  # noqa: E402
from featlsq import linalg as r_lin  # noqa: E402

from paper_2506_17626_b200 import workloads  # noqa: E402
from make_golden import to_reference  # noqa: E402


def main(name):
    wl = workloads.build(name)
    prob, dec, basis = to_reference(wl)
    t0 = time.time()
    system = r_asm.assemble(prob, dec, basis, interior_per_dim=wl.interior_per_dim)
    t1 = time.time()
    ranks, kept, rfro = [], [], []
    for blk in system.blocks:
        pq = r_lin.qr_column_pivot(blk.matrix, wl.sigma)
        ranks.append(pq.kept.size)
        kept.append(pq.kept.astype(np.int16))
        rfro.append(np.linalg.norm(pq.r_factor))
    t2 = time.time()
    np.savez_compressed(os.path.join(HERE, f"full_{name}.npz"), ranks=np.array(ranks, np.int32),
                        kept=np.concatenate(kept), r_fro=np.array(rfro), sigma=wl.sigma,
                        shape=np.array(system.shape), assemble_s=t1 - t0, filter_s=t2 - t1)
    print(name, system.shape, "kept", int(np.sum(ranks)), f"assemble {t1 - t0:.1f}s filter {t2 - t1:.1f}s")


if __name__ == "__main__":
    for n in sys.argv[1:]:
        main(n)
