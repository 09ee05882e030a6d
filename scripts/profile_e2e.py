"""cProfile of one public-API solve (assemble -> filter_system -> precondition
-> lsqr -> recover_solution) after a warm-up solve: where the host time of
the e2e path goes."""
import cProfile
import os
import pstats
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2506_17626_b200 as fl  # noqa: E402
from paper_2506_17626_b200 import workloads  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "cfg4"
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 1000
wl = workloads.build(name)


def step():
    t = [time.perf_counter()]
    system = fl.assemble(wl.problem, wl.dec, wl.basis, interior_per_dim=wl.interior_per_dim)
    t.append(time.perf_counter())
    fs = fl.filter_system(system, wl.sigma)
    t.append(time.perf_counter())
    res = fl.lsqr(fl.precondition(fs), system.rhs, iters)
    t.append(time.perf_counter())
    fl.recover_solution(fs, res.solution)
    torch.cuda.synchronize()
    t.append(time.perf_counter())
    return [round(b - a, 4) for a, b in zip(t, t[1:])]


print("warm", step())
print("timed", step())
pr = cProfile.Profile()
pr.enable()
print("profiled", step())
pr.disable()
pstats.Stats(pr).sort_stats("cumulative").print_stats(40)
