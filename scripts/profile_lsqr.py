"""Build one config's preconditioned operator and run N LSQR iterations
twice (profile the second run's kernels)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2506_17626_b200 as fl  # noqa: E402
from paper_2506_17626_b200 import workloads  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "cfg4"
its = int(sys.argv[2]) if len(sys.argv) > 2 else 5
wl = workloads.build(name)
system = fl.assemble(wl.problem, wl.dec, wl.basis, interior_per_dim=wl.interior_per_dim)
fs = fl.filter_system(system, wl.sigma)
op = fl.precondition(fs)
for rep in range(2):
    res = fl.lsqr(op, system.rhs, its)
    torch.cuda.synchronize()
print(name, "phibar", res.residual_norm)
