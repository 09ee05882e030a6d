"""Host jets -> the per-point (value, d/dx_a, d2/dx_a2) triples K1 consumes.

Mask and lift jets are the problem's own callables returning featlsq
`Jet2`s (`featlsq/jets.py:16-122`, re-exported); they are evaluated once
per point on the host and passed to the kernel as triples.
"""

from __future__ import annotations

import numpy as np

from ._featlsq import ref_jets

Jet2 = ref_jets.Jet2
radial_jet = ref_jets.radial_jet


def triples(jet_fn, points, dim: int) -> np.ndarray:
    """(P, dim, 3) array of (value, first, second) of jet_fn(points, a) for
    every axis a — the per-point layout K1 consumes."""
    pts = np.atleast_2d(np.asarray(points, dtype=float))
    out = np.empty((pts.shape[0], dim, 3))
    for a in range(dim):
        j = jet_fn(pts, a)
        out[:, a, 0] = np.broadcast_to(j.value, pts.shape[:1])
        out[:, a, 1] = np.broadcast_to(j.first, pts.shape[:1])
        out[:, a, 2] = np.broadcast_to(j.second, pts.shape[:1])
    return out
