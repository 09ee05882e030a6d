"""Time the fused LSQR iteration on one config for the CTA shape given in
FEATLSQ_FUSED (unset = default table choice); also a plain streaming read
of the Q store for comparison.

    FEATLSQ_FUSED=256,1,5,2 python scripts/lsqr_shapes.py cfg4 200
"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2506_17626_b200 as fl  # noqa: E402
from paper_2506_17626_b200 import workloads  # noqa: E402
from paper_2506_17626_b200.solvers import DeviceLsqr  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "cfg4"
its = int(sys.argv[2]) if len(sys.argv) > 2 else 200
wl = workloads.build(name)
system = fl.assemble(wl.problem, wl.dec, wl.basis, interior_per_dim=wl.interior_per_dim)
fs = fl.filter_system(system, wl.sigma)
blocks = fs.qstore
L = blocks.layout
nnz = int((L.m.astype("int64") * blocks.ncols).sum())
solver = DeviceLsqr(blocks, its + 20)
rhs = torch.from_numpy(system.rhs).cuda()
solver.reset_state(1, False)
solver.init(rhs)
solver.iterate(1, 10)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
solver.iterate(11, its)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / its
st = solver.read_state()
# plain read of the used part of the Q store: sum over all blocks' r_j columns
vals = blocks.vals
e0.record()
for _ in range(5):
    s = vals.sum()
e1.record()
torch.cuda.synchronize()
ms_read = e0.elapsed_time(e1) / 5
out = dict(shape=os.environ.get("FEATLSQ_FUSED", "default"), ms_per_iter=round(ms, 4),
           GBs_Q=round(8 * nnz / ms / 1e6, 1), GBs_store_sum=round(8 * vals.numel() / ms_read / 1e6, 1),
           phibar=st.phibar, it=st.it, done=st.done)
print(json.dumps(out))

# CUDA-graph replay of the same iterations (launch gaps)
if os.environ.get("FEATLSQ_GRAPH"):
    solver.reset_state(1, False)
    solver.init(rhs)
    solver.iterate(1, 10)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        with torch.cuda.graph(g, stream=s):
            solver.iterate(11, 50)
    torch.cuda.synchronize()
    solver.reset_state(1, False)
    solver.init(rhs)
    solver.iterate(1, 10)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(its // 50):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    print(json.dumps(dict(graph_ms_per_iter=round(e0.elapsed_time(e1) / (its // 50 * 50), 4))))
