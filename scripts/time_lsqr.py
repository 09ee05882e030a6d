"""LSQR ms/iteration of one config (device-resident, CUDA events), best of 3."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2506_17626_b200 as fl  # noqa: E402
from paper_2506_17626_b200 import _device as D, solvers, workloads  # noqa: E402

name, iters = sys.argv[1], int(sys.argv[2])
wl = workloads.build(name)
sysd = fl.assemble(wl.problem, wl.dec, wl.basis, interior_per_dim=wl.interior_per_dim)
fs = fl.filter_system(sysd, wl.sigma)
op = fl.precondition(fs)
run = solvers.DeviceLsqr(op.device_blocks, iters)
rhs = D.to_dev(sysd.rhs)
best = 1e9
for rep in range(3):
    run.reset_state(1, track_best=True)
    run.init(rhs)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    run.iterate(1, iters)
    e1.record()
    torch.cuda.synchronize()
    best = min(best, e0.elapsed_time(e1) / iters)
st = run.read_state()
print(f"{name} {os.environ.get('FEATLSQ_LIB', 'default')}: {best:.4f} ms/it phibar {st.phibar:.12e}")
