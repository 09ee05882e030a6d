"""Quick per-stage device timing of one config (CUDA events)."""

import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2506_17626_b200 as fl  # noqa: E402
from paper_2506_17626_b200 import workloads  # noqa: E402


def ev():
    e = torch.cuda.Event(enable_timing=True)
    e.record()
    return e


def main(name, iters):
    wl = workloads.build(name)
    torch.cuda.synchronize()
    for rep in range(2):
        e0 = ev()
        sysd = fl.assemble(wl.problem, wl.dec, wl.basis, interior_per_dim=wl.interior_per_dim)
        e1 = ev()
        fs = fl.filter_system(sysd, wl.sigma)
        e2 = ev()
        op = fl.precondition(fs)
        res = fl.lsqr(op, sysd.rhs, iters)
        e3 = ev()
        a = fl.recover_solution(fs, res.solution)
        e4 = ev()
        torch.cuda.synchronize()
        L = fs.qstore.layout
        nnzq = int(np.sum(L.m.astype(np.int64) * fs.ranks))
        nnza = int(np.sum(L.m.astype(np.int64))) * L.K
        t_it = e2.elapsed_time(e3) / 1e3 / max(iters, 1)
        bytes_it = 8 * (2 * nnzq + 2 * sysd.row_count + 6 * fs.kept_total)
        print(f"{name} rep{rep}: assemble {e0.elapsed_time(e1):.1f} ms ({8*nnza/e0.elapsed_time(e1)/1e6:.0f} GB/s) "
              f"filter {e1.elapsed_time(e2):.1f} ms  lsqr {iters} its {e2.elapsed_time(e3):.1f} ms "
              f"({t_it*1e3:.3f} ms/it, {bytes_it/t_it/1e9:.0f} GB/s)  recover {e3.elapsed_time(e4):.1f} ms  "
              f"kept {fs.kept_total}/{sysd.column_count} phibar {res.residual_norm:.4e}", flush=True)


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 50)
