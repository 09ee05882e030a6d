"""Synthetic BASELINE workloads (BASELINE.json `configs`).

Each config becomes (ProblemSpec, Decomposition, FeatureBasis,
interior_per_dim, sigma) built from featlsq's own value types, so the same
objects feed the device path and the CPU oracle. Weights are
W ~ U(-w, w) of shape (J, M, d) and b ~ U(-1, 1) of shape (J, M), drawn from
np.random.default_rng(seed); interior lattices are linspace with endpoints
(`assembly.py:147-158`); each boundary kind is one ConstraintRows group with
the identity operator, weight 1 and targets u(points).

The configs are synthetic stand-ins defined by BASELINE.json itself; no
public dataset is involved. `scale` shrinks S, M and n for parity tests that
the CPU oracle must finish in seconds.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from ._featlsq import featlsq

FeatureBasis = featlsq.FeatureBasis
Domain, decompose = featlsq.Domain, featlsq.decompose
ConstraintRows, LinearOperator2, ProblemSpec = (featlsq.ConstraintRows, featlsq.LinearOperator2,
                                                featlsq.ProblemSpec)

PI = np.pi


@dataclass
class Workload:
    name: str
    problem: ProblemSpec
    dec: object
    basis: FeatureBasis
    interior_per_dim: int
    sigma: float
    description: str


def _basis(dec, m, wrange, seed):
    rng = np.random.default_rng(seed)
    j, d = dec.subdomain_count, dec.dim
    w = rng.uniform(-wrange, wrange, (j, m, d))
    b = rng.uniform(-1.0, 1.0, (j, m))
    return FeatureBasis(dec, m, 1, "tanh", (w,), (b,))


def _ident(d):
    return LinearOperator2(1.0, np.zeros(d), np.zeros(d))


def _edges_2d(axis):
    n = axis.size
    zeros, ones = np.zeros(n), np.ones(n)
    return np.concatenate([
        np.stack([zeros, axis], 1), np.stack([ones, axis], 1),
        np.stack([axis, zeros], 1), np.stack([axis, ones], 1)])


def poisson_1d(S=20, M=64, n=2000, overlap=1.9, wrange=1.0, seed=0):
    """cfg1: -u'' = f, u = sin 2pi x + 0.1 sin 40pi x."""
    def exact(p):
        x = np.atleast_2d(p)[:, 0]
        return np.sin(2 * PI * x) + 0.1 * np.sin(40 * PI * x)

    def forcing(p):
        x = np.atleast_2d(p)[:, 0]
        return (2 * PI) ** 2 * np.sin(2 * PI * x) + 0.1 * (40 * PI) ** 2 * np.sin(40 * PI * x)
    dom = Domain(np.array([[0.0, 1.0]]))
    bpts = np.array([[0.0], [1.0]])
    prob = ProblemSpec("poisson1d", dom, LinearOperator2(0.0, [0.0], [-1.0]), forcing,
                       (ConstraintRows("boundary", _ident(1), bpts, exact(bpts), 1.0),),
                       exact=exact, test_points_per_count=6)
    dec = decompose(dom, S, overlap)
    return prob, dec, _basis(dec, M, wrange, seed), n


def multiscale_1d(S=200, M=128, n=40000, overlap=2.0, wrange=2.0, seed=0):
    """cfg2: -u'' = f, u = sum_{k=1..5} 2^-k sin(2^(k+1) pi x)."""
    ks = np.arange(1, 6)

    def exact(p):
        x = np.atleast_2d(p)[:, 0]
        return sum(2.0 ** -k * np.sin(2.0 ** (k + 1) * PI * x) for k in ks)

    def forcing(p):
        x = np.atleast_2d(p)[:, 0]
        return sum(2.0 ** -k * (2.0 ** (k + 1) * PI) ** 2 * np.sin(2.0 ** (k + 1) * PI * x)
                   for k in ks)
    dom = Domain(np.array([[0.0, 1.0]]))
    bpts = np.array([[0.0], [1.0]])
    prob = ProblemSpec("multiscale1d", dom, LinearOperator2(0.0, [0.0], [-1.0]), forcing,
                       (ConstraintRows("boundary", _ident(1), bpts, exact(bpts), 1.0),),
                       exact=exact, test_points_per_count=6)
    dec = decompose(dom, S, overlap)
    return prob, dec, _basis(dec, M, wrange, seed), n


def poisson_2d(S=16, M=256, n=400, overlap=2.0, wrange=1.0, seed=0):
    """cfg3: -lap u = f, u = s2(x)s2(y) + 0.1 s20(x)s20(y)."""
    def exact(p):
        p = np.atleast_2d(p)
        return (np.sin(2 * PI * p[:, 0]) * np.sin(2 * PI * p[:, 1])
                + 0.1 * np.sin(20 * PI * p[:, 0]) * np.sin(20 * PI * p[:, 1]))

    def forcing(p):
        p = np.atleast_2d(p)
        return (8 * PI ** 2 * np.sin(2 * PI * p[:, 0]) * np.sin(2 * PI * p[:, 1])
                + 0.1 * 800 * PI ** 2 * np.sin(20 * PI * p[:, 0]) * np.sin(20 * PI * p[:, 1]))
    dom = Domain(np.array([[0.0, 1.0], [0.0, 1.0]]))
    bpts = _edges_2d(np.linspace(0.0, 1.0, n))
    prob = ProblemSpec("poisson2d", dom, LinearOperator2(0.0, [0.0, 0.0], [-1.0, -1.0]),
                       forcing, (ConstraintRows("boundary", _ident(2), bpts, exact(bpts), 1.0),),
                       exact=exact, test_points_per_count=6)
    dec = decompose(dom, S, overlap)
    return prob, dec, _basis(dec, M, wrange, seed), n


def helmholtz_2d(S=32, M=512, n=800, overlap=2.0, wrange=3.0, seed=0, k=20.0):
    """cfg4: lap u + k^2 u = f, u = sum_{i=1..4} 2^-i s(2^(i+1) pi x) s(2^(i+1) pi y)."""
    iis = np.arange(1, 5)

    def exact(p):
        p = np.atleast_2d(p)
        return sum(2.0 ** -i * np.sin(2.0 ** (i + 1) * PI * p[:, 0])
                   * np.sin(2.0 ** (i + 1) * PI * p[:, 1]) for i in iis)

    def forcing(p):
        p = np.atleast_2d(p)
        return sum(2.0 ** -i * (k * k - 2 * (2.0 ** (i + 1) * PI) ** 2)
                   * np.sin(2.0 ** (i + 1) * PI * p[:, 0]) * np.sin(2.0 ** (i + 1) * PI * p[:, 1])
                   for i in iis)
    dom = Domain(np.array([[0.0, 1.0], [0.0, 1.0]]))
    bpts = _edges_2d(np.linspace(0.0, 1.0, n))
    prob = ProblemSpec("helmholtz2d", dom, LinearOperator2(k * k, [0.0, 0.0], [1.0, 1.0]),
                       forcing, (ConstraintRows("boundary", _ident(2), bpts, exact(bpts), 1.0),),
                       exact=exact, test_points_per_count=6)
    dec = decompose(dom, S, overlap)
    return prob, dec, _basis(dec, M, wrange, seed), n


def heat_2p1d(S=8, M=512, n=64, overlap=2.0, wrange=1.0, seed=0, kappa=0.01):
    """cfg5: u_t - 0.01 lap u = f on [0,1]^2 x [0,1]. The stated u's second
    mode is not an exact heat solution, so f is manufactured from it
    (SURVEY.md §8(d)): f = -0.384 pi^2 e^{-3.2 pi^2 t} s8(x) s8(y)."""
    def exact(p):
        p = np.atleast_2d(p)
        x, y, t = p[:, 0], p[:, 1], p[:, 2]
        return (np.exp(-0.08 * PI ** 2 * t) * np.sin(2 * PI * x) * np.sin(2 * PI * y)
                + 0.2 * np.exp(-3.2 * PI ** 2 * t) * np.sin(8 * PI * x) * np.sin(8 * PI * y))

    def forcing(p):
        p = np.atleast_2d(p)
        x, y, t = p[:, 0], p[:, 1], p[:, 2]
        # mode 1 is exact; mode 2: u_t - k lap u = (-3.2 + k*128) pi^2 u2
        return ((-3.2 + kappa * 128.0) * PI ** 2 * 0.2 * np.exp(-3.2 * PI ** 2 * t)
                * np.sin(8 * PI * x) * np.sin(8 * PI * y))
    dom = Domain(np.array([[0.0, 1.0], [0.0, 1.0], [0.0, 1.0]]))
    ax = np.linspace(0.0, 1.0, n)
    g1, g2 = np.meshgrid(ax, ax, indexing="ij")
    a, b = g1.ravel(), g2.ravel()
    z, o = np.zeros_like(a), np.ones_like(a)
    ic = np.stack([a, b, z], 1)
    lateral = np.concatenate([np.stack([z, a, b], 1), np.stack([o, a, b], 1),
                              np.stack([a, z, b], 1), np.stack([a, o, b], 1)])
    prob = ProblemSpec(
        "heat2p1d", dom, LinearOperator2(0.0, [0.0, 0.0, 1.0], [-kappa, -kappa, 0.0]),
        forcing,
        (ConstraintRows("initial", _ident(3), ic, exact(ic), 1.0),
         ConstraintRows("lateral", _ident(3), lateral, exact(lateral), 1.0)),
        exact=exact, test_points_per_count=4)
    dec = decompose(dom, S, overlap)
    return prob, dec, _basis(dec, M, wrange, seed), n


CONFIGS = {
    "cfg1": (poisson_1d, "1D Poisson J=20 M=64 N=2000+2, sigma 1e-10"),
    "cfg2": (multiscale_1d, "1D multiscale Poisson J=200 M=128 N=40000+2, sigma 1e-10"),
    "cfg3": (poisson_2d, "2D Poisson 16x16 M=256 400^2+1600, sigma 1e-10"),
    "cfg4": (helmholtz_2d, "2D Helmholtz k=20 32x32 M=512 800^2+3200, sigma 1e-10"),
    "cfg5": (heat_2p1d, "(2+1)D heat 8x8x8 M=512 64^3+64^2+4*64^2, sigma 1e-10"),
}

# reduced sizes the CPU oracle factors in seconds (parity-test cases)
SMALL = {
    "cfg1": dict(),
    "cfg2": dict(S=40, n=8000),
    "cfg3": dict(S=3, n=40),
    "cfg4": dict(S=3, n=48),
    "cfg5": dict(S=3, n=16),
}


def build(name: str, sigma: float = 1e-10, **overrides) -> Workload:
    fn, desc = CONFIGS[name]
    prob, dec, basis, n = fn(**overrides)
    return Workload(name, prob, dec, basis, n, sigma, desc)


def build_small(name: str, sigma: float = 1e-10, **overrides) -> Workload:
    kw = dict(SMALL[name])
    kw.update(overrides)
    return build(name, sigma, **kw)
