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
# round 2 kernels: K1 on a 2-D and a 3-D problem (tabulated path + constraint
# rows), the additive-Schwarz setup kernel, masked assembly
wl3 = workloads.build_small("cfg3")
s3 = fl.assemble(wl3.problem, wl3.dec, wl3.basis, interior_per_dim=wl3.interior_per_dim)
wl5 = workloads.build_small("cfg5")
s5 = fl.assemble(wl5.problem, wl5.dec, wl5.basis, interior_per_dim=wl5.interior_per_dim)
pre = fl.as_preconditioner(system)
p = fl.laplace_problem(1)
dec = fl.decompose(p.domain, 4, 2.9)
basis = fl.init_basis(dec, 16, 1, "tanh", np.random.default_rng(1))
sl = fl.assemble(p, dec, basis)
pre2 = fl.as_preconditioner(sl)
print("asm3", s3.shape, "asm5", s5.shape, "as blocks", len(pre.block_ranges), len(pre2.block_ranges))
