"""Run assemble + filter_system twice for one config (the second pass is the
one to profile under ncu: skip the first pass's launches with -s)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2506_17626_b200 as fl  # noqa: E402
from paper_2506_17626_b200 import workloads  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "cfg4"
wl = workloads.build(name)
for rep in range(2):
    system = fl.assemble(wl.problem, wl.dec, wl.basis, interior_per_dim=wl.interior_per_dim)
    fs = fl.filter_system(system, wl.sigma)
    torch.cuda.synchronize()
    print(name, "kept", fs.kept_total, flush=True)
