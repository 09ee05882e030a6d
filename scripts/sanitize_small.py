"""Small end-to-end runs for compute-sanitizer (memcheck/racecheck): cfg2
(K = 128: route R with the fused K2c) and a K = 160 route-R case (32-wide
updates), a few LSQR iterations each."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2506_17626_b200 as fl  # noqa: E402
from paper_2506_17626_b200 import workloads  # noqa: E402

wl = workloads.build("cfg2")
system = fl.assemble(wl.problem, wl.dec, wl.basis, interior_per_dim=wl.interior_per_dim)
fs = fl.filter_system(system, wl.sigma)
res = fl.lsqr(fl.precondition(fs), system.rhs, 20)
a = fl.recover_solution(fs, res.solution)
print("cfg2 kept", fs.kept_total, "phibar", res.residual_norm)
rng = np.random.default_rng(0)
m, K = 600, 160
u, _ = np.linalg.qr(rng.standard_normal((m, K)))
w, _ = np.linalg.qr(rng.standard_normal((K, K)))
mat = (u * np.logspace(0, -14, K)) @ w.T
got = fl.qr_column_pivot(mat, 1e-10)
print("K=160 kept", got.kept.size)
