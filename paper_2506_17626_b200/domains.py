"""Host value objects for the overlapping subdomain grid.

Same fields and formulas as `featlsq/domains.py:26-103` (`Domain`,
`Decomposition`, `decompose`), so a decomposition built here and one built by
the reference are interchangeable inputs to `assemble`. The window
arithmetic itself (`domains.py:109-184`) lives in the assembly kernel
(`csrc/assemble.cu`); the host only evaluates the strict support test on the
1-D lattice axes to derive row runs.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .errors import InvalidInputError, UnsupportedDecompositionError


@dataclass(frozen=True)
class Domain:
    """Axis-aligned box, bounds[i] = (low_i, high_i) (`domains.py:26-48`)."""

    bounds: np.ndarray

    def __post_init__(self):
        b = np.atleast_2d(np.asarray(self.bounds, dtype=float))
        if b.ndim != 2 or b.shape[1] != 2:
            raise InvalidInputError(f"bounds must be (d, 2), got {b.shape}")
        if not np.isfinite(b).all():
            raise InvalidInputError("bounds must be finite")
        if np.any(b[:, 1] <= b[:, 0]):
            raise InvalidInputError("each dimension needs high > low")
        object.__setattr__(self, "bounds", b)

    @property
    def dim(self) -> int:
        return self.bounds.shape[0]

    @property
    def widths(self) -> np.ndarray:
        return self.bounds[:, 1] - self.bounds[:, 0]


@dataclass(frozen=True)
class Decomposition:
    """Regular grid of overlapping subdomains (`domains.py:51-82`).

    centers (dim, count), half_widths (dim,); flat subdomain index is C-order
    over the per-dimension center indices.
    """

    domain: Domain
    count_per_dim: int
    overlap_ratio: float
    centers: np.ndarray
    half_widths: np.ndarray

    @property
    def dim(self) -> int:
        return self.domain.dim

    @property
    def subdomain_count(self) -> int:
        return self.count_per_dim ** self.dim

    def multi_index(self, j: int) -> tuple[int, ...]:
        if not 0 <= j < self.subdomain_count:
            raise InvalidInputError(f"subdomain index {j} out of range")
        return tuple(int(v) for v in
                     np.unravel_index(j, (self.count_per_dim,) * self.dim))


def decompose(domain: Domain, count_per_dim: int, overlap_ratio: float) -> Decomposition:
    """Centers low + spacing*s, half-width overlap/2*spacing (`domains.py:85-103`)."""
    if count_per_dim < 2:
        raise UnsupportedDecompositionError(
            f"need at least 2 subdomains per dimension, got {count_per_dim}")
    if overlap_ratio <= 0.0:
        raise UnsupportedDecompositionError(
            f"overlap_ratio must be positive, got {overlap_ratio}")
    spacing = domain.widths / (count_per_dim - 1)
    offsets = np.arange(count_per_dim, dtype=float)
    centers = domain.bounds[:, 0][:, None] + spacing[:, None] * offsets[None, :]
    half_widths = 0.5 * overlap_ratio * spacing
    return Decomposition(domain, count_per_dim, overlap_ratio, centers, half_widths)


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
