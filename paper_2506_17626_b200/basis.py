"""Host value object for the frozen random feature networks.

Same layout as `featlsq/basis.py:43-64`: weights[0] is (J, K, d), biases[0]
is (J, K); columns of subdomain j are j*K .. (j+1)*K-1. Only depth 1 is on the
accelerated path (the BASELINE configs and the paper's problems are depth 1);
the feature jets themselves (`basis.py:99-133`) are evaluated inside the
assembly kernel.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .errors import InvalidInputError

# activation name -> kernel code (csrc/featlsq_b200.h FL_ACT_*)
ACTIVATIONS = {"tanh": 0, "sin": 1, "sigmoid": 2}


@dataclass(frozen=True)
class FeatureBasis:
    decomposition: object
    feature_count: int
    depth: int
    activation: str
    weights: tuple
    biases: tuple

    @property
    def column_count(self) -> int:
        return self.decomposition.subdomain_count * self.feature_count

    def column_range(self, j: int) -> np.ndarray:
        k = self.feature_count
        return np.arange(j * k, (j + 1) * k)


def init_basis(dec, feature_count: int, depth: int, activation: str,
               rng: np.random.Generator) -> FeatureBasis:
    """Draw parameters subdomain by subdomain, layer by layer, from the
    uniform LeCun range (`basis.py:67-96`); same draw order, so the same
    generator state yields the same arrays as the reference."""
    if feature_count < 1:
        raise InvalidInputError(f"feature_count must be >= 1, got {feature_count}")
    if depth < 1:
        raise InvalidInputError(f"depth must be >= 1, got {depth}")
    if activation not in ACTIVATIONS:
        raise InvalidInputError(
            f"unknown activation {activation!r}, have {sorted(ACTIVATIONS)}")
    d, k, j_count = dec.dim, feature_count, dec.subdomain_count
    shapes = [(d, k, True)]
    shapes += [(k, k, True)] * (depth - 2)
    if depth >= 2:
        shapes += [(k, k, False)]
    weights, biases = [], []
    for fan_in, fan_out, has_bias in shapes:
        weights.append(np.empty((j_count, fan_out, fan_in)))
        biases.append(np.empty((j_count, fan_out)) if has_bias else None)
    for j in range(j_count):
        for layer, (fan_in, fan_out, has_bias) in enumerate(shapes):
            bound = np.sqrt(1.0 / fan_in)
            weights[layer][j] = rng.uniform(-bound, bound, size=(fan_out, fan_in))
            if has_bias:
                biases[layer][j] = rng.uniform(-bound, bound, size=fan_out)
    return FeatureBasis(dec, feature_count, depth, activation,
                        tuple(weights), tuple(biases))
