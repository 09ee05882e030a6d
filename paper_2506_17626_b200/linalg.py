"""Single-matrix entry points of the dense kernels (reference:
featlsq/linalg.py:21-112), routed through the same CUDA kernels as the
batched path: `qr_column_pivot` is K2 on a one-block store, `back_substitute`
is K5 on one block.
"""

from __future__ import annotations

import ctypes as C
import numpy as np

from . import _device as D
from . import _lib
from ._featlsq import ref_assembly, ref_linalg
from .errors import InvalidInputError, SingularFactorError

DENSE_SIZE_CAP = 20_000


# featlsq's own value types (`linalg.py:21-46`) and lattice rule (`assembly.py:32-40`)
RandomSource = ref_linalg.RandomSource
PivotedQR = ref_linalg.PivotedQR
lattice_counts = ref_assembly.lattice_counts


def _check_matrix(a, name="matrix") -> np.ndarray:
    a = np.asarray(a, dtype=float)
    if a.ndim != 2:
        raise InvalidInputError(f"{name} must be 2-D, got shape {a.shape}")
    if not np.isfinite(a).all():
        raise InvalidInputError(f"{name} contains non-finite entries")
    return a


def qr_column_pivot(a: np.ndarray, sigma_rel: float) -> PivotedQR:
    """Truncated column-pivoted QR of one matrix on the device (`linalg.py:58-97`)."""
    a = _check_matrix(a)
    if not 0.0 <= sigma_rel < 1.0:
        raise InvalidInputError(f"sigma_rel must be in [0, 1), got {sigma_rel}")
    rows, cols = a.shape
    if cols == 0:
        e = np.empty(0, dtype=int)
        return PivotedQR(np.empty((rows, 0)), np.empty((0, 0)), e, e, np.empty(0))
    from .filtering import factor_store
    from .solvers import _dense_blocks
    blocks = _dense_blocks(a)
    # the same K2 as filter_system on a one-block store (route R for K >= 128)
    work, R, perm, rank, diag = factor_store(blocks, float(sigma_rel))
    blocks = D.DeviceBlocks(blocks.layout, work, blocks.ncols, blocks.col_off)
    r = int(D.to_host(rank)[0])
    if r < 0:
        raise InvalidInputError("matrix contains non-finite entries")
    p = D.to_host(perm)[:cols].astype(int)
    q = blocks.block_host(0, ncols=r) if r else np.zeros((rows, 0))
    rr = D.to_host(R)[:cols * cols].reshape(cols, cols)[:r, :r].T.copy()
    return PivotedQR(q, rr, p[:r].copy(), np.sort(p[r:]), D.to_host(diag)[:r].copy())


def back_substitute(r: np.ndarray, y: np.ndarray) -> np.ndarray:
    """Solve r x = y for upper-triangular r on the device (`linalg.py:100-112`)."""
    r = _check_matrix(r, "triangular factor")
    if r.shape[0] != r.shape[1]:
        raise InvalidInputError(f"triangular factor must be square, got {r.shape}")
    y = np.asarray(y, dtype=float)
    if y.shape[0] != r.shape[0]:
        raise InvalidInputError(f"rhs length {y.shape[0]} != factor size {r.shape[0]}")
    n = r.shape[0]
    if n == 0:
        return np.zeros_like(y)
    if np.any(np.diag(r) == 0.0):
        raise SingularFactorError("zero diagonal entry in triangular factor")
    cols = y.reshape(n, -1)
    t = D.torch()
    Rd = D.to_dev(np.ascontiguousarray(r.T).ravel())        # column-major, ld = n
    rank = D.to_dev(np.array([n], np.int32))
    perm = D.to_dev(np.arange(n, dtype=np.int32))
    yoff = D.to_dev(np.zeros(1, np.int64))
    out = np.empty_like(cols)
    for c in range(cols.shape[1]):
        yd = D.to_dev(np.ascontiguousarray(cols[:, c]))
        coeffs = t.empty(n, dtype=t.float64, device=yd.device)
        sing = t.full((1,), 2 ** 31 - 1, dtype=t.int32, device=yd.device)
        _lib.check(_lib.lib().fl_backsub_scatter(1, n, D.ptr(Rd), D.ptr(rank), D.ptr(perm),
                                                 D.ptr(yoff), D.ptr(yd), D.ptr(coeffs),
                                                 D.ptr(sing), D.stream_ptr()), "fl_backsub_scatter")
        out[:, c] = D.to_host(coeffs)
    return out.reshape(y.shape)
