"""Feature-basis codes for the assembly kernel.

`FeatureBasis` and `init_basis` are featlsq's own (`featlsq/basis.py:43-96`,
re-exported). Layout consumed by K1: weights[0] is (J, K, d), biases[0] is
(J, K); columns of subdomain j are j*K .. (j+1)*K-1. Only depth 1 is on the
accelerated path (the BASELINE configs and the paper's problems are depth 1);
the feature jets (`basis.py:99-133`) are evaluated inside the kernel.
"""

from __future__ import annotations

from ._featlsq import ref_basis

FeatureBasis = ref_basis.FeatureBasis
init_basis = ref_basis.init_basis

# activation name -> kernel code (include/featlsq_b200.h FL_ACT_*)
ACTIVATIONS = {"tanh": 0, "sin": 1, "sigmoid": 2}
