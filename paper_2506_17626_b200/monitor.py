"""Device test-lattice error monitor (K6; reference: runner.py:265-293,
solvers.py:47-69, assembly.py:313-318).

The reference runner builds T = P[:, kept] S^{-1} on the host
(`_error_matrix`) and calls `l1_error(T @ y + lift, test_set)` for every
recorded iterate. `DeviceL1Error` is the same error function with T resident
in HBM: `lsqr` recognises it as the monitor's `error_fn` and evaluates it
inside the device loop (one pass over T per recorded iteration, best iterate
kept on the device), so no iterate crosses PCIe. Called directly it is an
ordinary host function y -> e (one device evaluation).

For solvers over the raw coefficients (plain LSQR / CG on M, runner.py:
296-305) `DeviceL1Error(None, blocks, test_set)` uses P itself.
"""

from __future__ import annotations

import ctypes as C

import numpy as np

from . import _device as D
from . import _lib
from .assembly import SolutionBlocks, TestSet
from .errors import InvalidInputError


class DeviceL1Error:
    """error_fn(y) = l1_error(T y + lift, test_set) with T on the device."""

    def __init__(self, filtered, blocks: SolutionBlocks, test_set: TestSet):
        if blocks.points.shape != test_set.points.shape or not np.array_equal(blocks.points,
                                                                             test_set.points):
            raise InvalidInputError("solution blocks were evaluated at other points than the test set")
        t = D.torch()
        dev = D.require_cuda()
        P = blocks.store
        L = P.layout
        if filtered is None:
            self.T = P
        else:
            if L.J != len(filtered.ranks) or L.K != filtered.K:
                raise InvalidInputError("filtered system and solution blocks disagree on the blocks")
            vals = t.empty_like(P.vals)
            self.T = D.DeviceBlocks(L, vals, filtered.ranks.astype(np.int32), filtered.offsets[:-1])
            tiles = D.tile_table(L.m, _lib.FL_TBUILD_ROWS)
            tiles_dev = D.to_dev(tiles)
            _lib.check(_lib.lib().fl_error_blocks(
                C.byref(P.struct()), D.ptr(filtered._R), D.ptr(filtered._perm), int(filtered.K),
                C.byref(self.T.struct()), len(tiles), D.ptr(tiles_dev), D.stream_ptr()),
                "fl_error_blocks")
        self.n = int(self.T.ncols_total)
        self.test_set = test_set
        self._blocks = blocks
        self._lift = D.to_dev(blocks.lift)
        self._truth = D.to_dev(np.asarray(test_set.true_values, dtype=float))
        self._result = t.zeros(1, dtype=t.float64, device=dev)
        self._trace = t.zeros(1, dtype=t.float64, device=dev)

    def struct(self, trace=None) -> _lib.TestMonitor:
        tr = self._trace if trace is None else trace
        return _lib.TestMonitor(T=self.T.struct(), lift=D.ptr(self._lift), truth=D.ptr(self._truth),
                                spread=float(self.test_set.spread), err_trace=D.ptr(tr),
                                result=D.ptr(self._result))

    def device_error(self, y_dev) -> float:
        mon = self.struct()
        _lib.check(_lib.lib().fl_monitor_error(C.byref(mon), D.ptr(y_dev), D.stream_ptr()),
                   "fl_monitor_error")
        return float(D.to_host(self._result)[0])

    def __call__(self, y) -> float:
        y = np.asarray(y, dtype=float)
        if y.shape != (self.n,):
            raise InvalidInputError(f"iterate must have shape ({self.n},), got {y.shape}")
        return self.device_error(D.to_dev(y))


def test_error_fn(filtered, problem, dec, basis, test_set: TestSet) -> DeviceL1Error:
    """The runner's rrqr-lsqr error function (`runner.py:285-289`) on the device:
    P at the test points (K1), T = P[:, kept] S^{-1} (K6 build)."""
    return DeviceL1Error(filtered, SolutionBlocks(problem, dec, basis, test_set.points), test_set)


test_error_fn.__test__ = False  # not a pytest test


def raw_error_fn(problem, dec, basis, test_set: TestSet) -> DeviceL1Error:
    """The runner's error function for solvers over the raw coefficients
    (`runner.py:295-305`: l1_error(P a + lift)) with P on the device."""
    return DeviceL1Error(None, SolutionBlocks(problem, dec, basis, test_set.points), test_set)


raw_error_fn.__test__ = False
