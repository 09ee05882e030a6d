"""Exception taxonomy of the drop-in path: featlsq's own classes
(`featlsq/errors.py:4-41`), so callers catch exactly what they catch around
the reference, plus `DeviceError` for CUDA failures (no reference analogue).
"""

from __future__ import annotations

from ._featlsq import ref_errors as _ref

InvalidInputError = _ref.InvalidInputError
SingularFactorError = _ref.SingularFactorError
CapExceededError = _ref.CapExceededError
UnsupportedDecompositionError = _ref.UnsupportedDecompositionError
CoverageError = _ref.CoverageError
DegenerateSubdomainError = _ref.DegenerateSubdomainError
DivergenceError = _ref.DivergenceError


class DeviceError(RuntimeError):
    """The CUDA extension reported a launch or runtime failure."""
