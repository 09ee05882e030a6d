"""Subdomain-grid helpers for the device assembly.

The value types and `decompose` are featlsq's own (`featlsq/domains.py:26-103`,
re-exported here); the window arithmetic (`domains.py:109-184`) lives in the
assembly kernel (`csrc/assemble.cu`). The host only evaluates the strict
support test on the 1-D lattice axes to derive each subdomain's row runs.
"""

from __future__ import annotations

import numpy as np

from ._featlsq import ref_domains

Domain = ref_domains.Domain
Decomposition = ref_domains.Decomposition
decompose = ref_domains.decompose


def support_runs(dec, axes) -> np.ndarray:
    """Per (subdomain-index-along-dim, dim): the contiguous lattice run
    [lo, lo+count) with |axis - mu| < half strictly (`assembly.py:201-204`,
    `domains.py:176-184`). Returns int64 (dim, count_per_dim, 2)."""
    d = dec.dim
    out = np.zeros((d, dec.count_per_dim, 2), dtype=np.int64)
    for i in range(d):
        half = dec.half_widths[i]
        for s in range(dec.count_per_dim):
            mu = dec.centers[i, s]
            idx = np.nonzero(np.abs(axes[i] - mu) < half)[0]
            if idx.size:
                # the strict support of a window is an interval, and a sorted
                # lattice meets it in one contiguous run
                assert idx[-1] - idx[0] + 1 == idx.size
                out[i, s] = (idx[0], idx.size)
    return out
