"""Exception taxonomy of the drop-in path.

Mirrors `featlsq/errors.py:4-41` name for name so callers catch the same
classes. When the reference package is importable in the caller's process,
each class also derives from the reference class of the same name, so an
`except featlsq.errors.DivergenceError` around the drop-in still fires.
"""

from __future__ import annotations

try:  # pragma: no cover - depends on the caller's environment
    from featlsq import errors as _ref  # type: ignore
except Exception:  # noqa: BLE001
    _ref = None


def _bases(name: str, fallback: type) -> tuple:
    ref = getattr(_ref, name, None) if _ref is not None else None
    return (ref,) if ref is not None else (fallback,)


class InvalidInputError(*_bases("InvalidInputError", ValueError)):
    """Malformed argument: wrong shape, non-finite entries, bad range."""


class SingularFactorError(*_bases("SingularFactorError", RuntimeError)):
    """A triangular factor has a zero diagonal entry."""


class CapExceededError(*_bases("CapExceededError", ValueError)):
    """Matrix dimensions exceed the configured dense-factorization cap."""


class UnsupportedDecompositionError(*_bases("UnsupportedDecompositionError", ValueError)):
    """Decomposition parameters outside the supported family."""


class CoverageError(*_bases("CoverageError", RuntimeError)):
    """A collocation point is covered by zero subdomains."""


class DegenerateSubdomainError(*_bases("DegenerateSubdomainError", RuntimeError)):
    """Filtering removed every column of some subdomain block."""


class DivergenceError(*_bases("DivergenceError", RuntimeError)):
    """An iterative solve produced non-finite iterates."""


class DeviceError(RuntimeError):
    """The CUDA extension reported a launch or runtime failure."""
