"""Host-side second-order jets along one axis (reference: featlsq/jets.py).

Only the user-facing problem definitions use these (mask and lift jets of
hard-constrained problems, evaluated once per point on the host and handed
to K1 as per-point (value, d/dx_a, d2/dx_a2) triples); the per-entry jets of
the assembly itself live in registers inside csrc/assemble.cu.

Arithmetic follows the reference term by term (jets.py:55-63 product,
:76-80 reciprocal, :82-107 chain rules) so that host-evaluated masks match
the reference to the last bit where numpy evaluates in the same order.
"""

from __future__ import annotations

import numpy as np


def _arr(x):
    return np.asarray(x, dtype=float)


class Jet2:
    """(value, first, second) of one scalar field w.r.t. one coordinate."""

    __slots__ = ("value", "first", "second")

    def __init__(self, value, first, second):
        self.value, self.first, self.second = _arr(value), _arr(first), _arr(second)

    # -- construction ------------------------------------------------------
    @staticmethod
    def variable(x) -> "Jet2":
        x = _arr(x)
        return Jet2(x, np.ones_like(x), np.zeros_like(x))

    @staticmethod
    def constant(c) -> "Jet2":
        c = _arr(c)
        return Jet2(c, np.zeros_like(c), np.zeros_like(c))

    # -- arithmetic ----------------------------------------------------------
    def __add__(self, o):
        if isinstance(o, Jet2):
            return Jet2(self.value + o.value, self.first + o.first, self.second + o.second)
        return Jet2(self.value + o, self.first, self.second)

    __radd__ = __add__

    def __neg__(self):
        return Jet2(-self.value, -self.first, -self.second)

    def __sub__(self, o):
        return self + (-o if isinstance(o, Jet2) else -_arr(o))

    def __rsub__(self, o):
        return (-self) + o

    def __mul__(self, o):
        if not isinstance(o, Jet2):
            return Jet2(self.value * o, self.first * o, self.second * o)
        v = self.value * o.value
        f = self.first * o.value + self.value * o.first
        s = self.second * o.value + 2.0 * self.first * o.first + self.value * o.second
        return Jet2(v, f, s)

    __rmul__ = __mul__

    def reciprocal(self) -> "Jet2":
        iv = 1.0 / self.value
        return Jet2(iv, -self.first * iv * iv, (2.0 * self.first * self.first * iv - self.second) * iv * iv)

    def __truediv__(self, o):
        if isinstance(o, Jet2):
            return self * o.reciprocal()
        return self * (1.0 / _arr(o))

    def __rtruediv__(self, o):
        return self.reciprocal() * o

    # -- chain rules -------------------------------------------------------
    def tanh(self) -> "Jet2":
        t = np.tanh(self.value)
        g = 1.0 - t * t
        return Jet2(t, g * self.first, -2.0 * t * g * self.first * self.first + g * self.second)

    def exp(self) -> "Jet2":
        e = np.exp(self.value)
        return Jet2(e, e * self.first, e * (self.first * self.first + self.second))

    def sin(self) -> "Jet2":
        sn, cs = np.sin(self.value), np.cos(self.value)
        return Jet2(sn, cs * self.first, -sn * self.first * self.first + cs * self.second)

    def cos(self) -> "Jet2":
        sn, cs = np.sin(self.value), np.cos(self.value)
        return Jet2(cs, -sn * self.first, -cs * self.first * self.first - sn * self.second)

    def square(self) -> "Jet2":
        return self * self


def radial_jet(offsets, axis: int) -> Jet2:
    """Jet of r = ||offsets|| w.r.t. coordinate `axis` (jets.py:110-121)."""
    off = _arr(offsets)
    r = np.sqrt(np.sum(off * off, axis=-1))
    dr = off[..., axis] / r
    return Jet2(r, dr, (1.0 - dr * dr) / r)


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
