"""Drop-in `assemble` / `GlobalSystem` on the device (reference:
featlsq/assembly.py:43-238).

The host does what the reference does outside its per-block numpy loop —
input validation (:132-155), the lattice (:156-158), the coverage check
(:171-177), the right-hand side from the user's forcing callable (:179-192)
and the row sets (:199-231, derived from per-dimension support runs) — and
the CUDA kernel K1 (`fl_assemble`, csrc/assemble.cu) evaluates every block
entry. Blocks stay resident in HBM; `GlobalSystem.blocks` is a lazily
materialised host view (one D2H copy on first access). Replacing an entry
of `blocks` (the reference tests do, tests/test_filtering.py:89-95) marks it
dirty and the device copy is refreshed before the next device use.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np
import scipy.sparse

from . import _device as D
from . import _lib
from .basis import ACTIVATIONS
from .domains import support_runs
from .errors import CapExceededError, CoverageError, InvalidInputError

DENSE_SIZE_CAP = 20_000


@dataclass(frozen=True)
class SubdomainBlock:
    """One subdomain's rows and columns of the global matrix (`assembly.py:43-50`)."""

    subdomain: int
    rows: np.ndarray
    columns: np.ndarray
    matrix: np.ndarray


class _BlockList(list):
    """Host view of the device blocks that records replaced entries."""

    def __init__(self, items, owner):
        super().__init__(items)
        self._owner = owner

    def __setitem__(self, idx, value):
        super().__setitem__(idx, value)
        idxs = range(len(self))[idx] if isinstance(idx, slice) else [idx]
        for i in idxs:
            self._owner._dirty.add(int(i) % len(self))


@dataclass
class GlobalSystem:
    """Same attribute surface as `assembly.py:53-88`, blocks on the device."""

    problem: object
    decomposition: object
    basis: object
    rhs: np.ndarray
    interior_count: int
    row_count: int
    column_count: int
    lattice_axes: tuple
    store: D.DeviceBlocks = field(repr=False, default=None)
    block_rows: list = field(repr=False, default=None)
    _blocks: list | None = field(default=None, repr=False)
    _dirty: set = field(default_factory=set, repr=False)
    _csr: scipy.sparse.csr_matrix | None = field(default=None, repr=False)

    @property
    def shape(self) -> tuple[int, int]:
        return (self.row_count, self.column_count)

    @property
    def blocks(self) -> list:
        if self._blocks is None:
            k = self.basis.feature_count
            mats = self.store.all_blocks_host()
            self._blocks = _BlockList(
                [SubdomainBlock(j, self.block_rows[j], np.arange(j * k, (j + 1) * k), mats[j])
                 for j in range(len(mats))], self)
        return self._blocks

    def sync_device(self) -> None:
        """Push host-side replacements of `blocks[j]` back to the device."""
        if not self._dirty:
            return
        for j in sorted(self._dirty):
            blk = self._blocks[j]
            mat = np.asarray(blk.matrix, dtype=float)
            if mat.shape != (self.store.layout.m[j], self.basis.feature_count):
                raise InvalidInputError(f"replacement block {j} has shape {mat.shape}")
            self.store.set_block(j, mat)
        self._dirty.clear()
        self._csr = None

    def csr(self) -> scipy.sparse.csr_matrix:
        """Host CSR of the raw system (analysis/tests only; `assembly.py:70-83`)."""
        if self._csr is None:
            rows, cols, vals = [], [], []
            for blk in self.blocks:
                rows.append(np.repeat(blk.rows, blk.columns.size))
                cols.append(np.tile(blk.columns, blk.rows.size))
                vals.append(blk.matrix.ravel())
            self._csr = scipy.sparse.coo_matrix(
                (np.concatenate(vals), (np.concatenate(rows), np.concatenate(cols))),
                shape=self.shape).tocsr()
        return self._csr

    def materialize(self, size_cap: int = DENSE_SIZE_CAP) -> np.ndarray:
        if max(self.shape) > size_cap:
            raise CapExceededError(f"shape {self.shape} exceeds cap {size_cap}")
        return self.csr().toarray()


def apply(system: GlobalSystem, coeffs: np.ndarray) -> np.ndarray:
    """M a on the device (`assembly.py:91-96`)."""
    coeffs = np.asarray(coeffs, dtype=float)
    if coeffs.shape != (system.column_count,):
        raise InvalidInputError(
            f"coefficients must have shape ({system.column_count},), got {coeffs.shape}")
    system.sync_device()
    return D.to_host(system.store.apply(D.to_dev(coeffs)))[:system.row_count]


def apply_transpose(system: GlobalSystem, residual: np.ndarray) -> np.ndarray:
    """M^T r on the device (`assembly.py:99-104`)."""
    residual = np.asarray(residual, dtype=float)
    if residual.shape != (system.row_count,):
        raise InvalidInputError(
            f"residual must have shape ({system.row_count},), got {residual.shape}")
    system.sync_device()
    return D.to_host(system.store.apply_t(D.to_dev(residual)))[:system.column_count]


def _member(dec, points):
    """Per-dim strict support membership, (d, S, P) booleans (`domains.py:176-184`)."""
    pts = np.atleast_2d(points)
    return np.stack([np.abs(pts[None, :, i] - dec.centers[i][:, None]) < dec.half_widths[i]
                     for i in range(dec.dim)])


def _layout_inputs(problem, dec, basis, axes, counts):
    """Per-block box runs, constraint membership and global row ids."""
    d, S, J = dec.dim, dec.count_per_dim, dec.subdomain_count
    runs = support_runs(dec, axes)                       # (d, S, 2)
    n_int = int(np.prod(counts))
    groups = []
    offset = n_int
    for con in problem.constraints:
        n_con = np.atleast_2d(con.points).shape[0]
        groups.append((offset, _member(dec, con.points)))
        offset += n_con
    row_count = offset
    multi = np.array(np.unravel_index(np.arange(J), (S,) * d)).T  # (J, d)
    box = np.zeros((J, d, 2), dtype=np.int32)
    con_idx, con_grp, con_ptr = [], [], [0]
    rows_per_block = []
    strides = np.array([int(np.prod(counts[i + 1:])) for i in range(d)], dtype=np.int64)
    for j in range(J):
        idx = multi[j]
        lo = runs[np.arange(d), idx, 0]
        cnt = runs[np.arange(d), idx, 1]
        if np.all(cnt > 0):
            box[j, :, 0], box[j, :, 1] = lo, cnt
            g = np.zeros(1, dtype=np.int64)
            for i in range(d):
                g = (g[:, None] + (lo[i] + np.arange(cnt[i], dtype=np.int64))[None, :] * strides[i]).ravel()
            rows = [g]
        else:
            rows = [np.zeros(0, np.int64)]
        for gi, (goff, mem) in enumerate(groups):
            inside = np.ones(mem.shape[2], dtype=bool)
            for i in range(d):
                inside &= mem[i, idx[i]]
            pidx = np.nonzero(inside)[0]
            rows.append(goff + pidx)
            con_idx.append(pidx)
            con_grp.append(np.full(pidx.size, gi, dtype=np.int32))
        rows_per_block.append(np.concatenate(rows))
        con_ptr.append(con_ptr[-1] + sum(x.size for x in con_idx[len(con_idx) - len(groups):]))
    return (row_count, box, np.array(con_ptr, dtype=np.int64),
            np.concatenate(con_idx).astype(np.int32) if con_idx else np.zeros(0, np.int32),
            np.concatenate(con_grp) if con_grp else np.zeros(0, np.int32),
            rows_per_block)


class AssemblyPlan:
    """Everything `assemble` derives on the host, uploaded once: the layout,
    the right-hand side and the K1 descriptor. `launch(vals)` re-runs only
    the kernel (the device-resident benchmark step uses this)."""

    def __init__(self, problem, dec, basis, interior_per_dim=None):
        _validate(problem, dec, basis)
        d = dec.dim
        counts = _lattice_counts(dec, basis, interior_per_dim)
        axes = tuple(np.linspace(dec.domain.bounds[i, 0], dec.domain.bounds[i, 1], counts[i])
                     for i in range(d))
        n_interior = int(np.prod(counts))
        _coverage(problem, dec, axes, n_interior)

        # right-hand side (assembly.py:179-192), host: user callables
        mesh = np.meshgrid(*axes, indexing="ij")
        interior = np.stack([m.ravel() for m in mesh], axis=1)
        iw = 1.0 / np.sqrt(n_interior)
        rhs_parts = [(np.asarray(problem.forcing(interior), dtype=float) - np.zeros(n_interior)) * iw]
        coef_rows = [[float(problem.operator.value_coef), iw, *problem.operator.first_coefs,
                      *problem.operator.second_coefs]]
        con_pts = []
        for con in problem.constraints:
            pts = np.atleast_2d(np.asarray(con.points, dtype=float))
            w = np.sqrt(con.weight / pts.shape[0])
            rhs_parts.append((np.asarray(con.targets, dtype=float) - np.zeros(pts.shape[0])) * w)
            op = con.operator
            coef_rows.append([float(op.value_coef), w, *op.first_coefs, *op.second_coefs])
            con_pts.append(pts)
        self.rhs = np.concatenate(rhs_parts)
        if len(problem.constraints) > 7:
            raise NotImplementedError("more than 7 constraint groups")

        row_count, box, con_ptr, con_idx, con_grp, rows_per_block = _layout_inputs(
            problem, dec, basis, axes, counts)
        goff = np.cumsum([0] + [p.shape[0] for p in con_pts])
        con_idx = con_idx + goff[con_grp].astype(np.int32) if con_idx.size else con_idx
        K = basis.feature_count
        J = dec.subdomain_count
        self.layout = D.BlockLayout(row_count, K, rows_per_block)
        self.rows_per_block = rows_per_block
        self.problem, self.dec, self.basis = problem, dec, basis
        self.axes, self.n_interior, self.row_count = axes, n_interior, row_count
        tiles = D.tile_table(self.layout.ld, _lib.FL_ASM_TILE)
        self.keep = keep = dict(
            centers=D.to_dev(np.asarray(dec.centers, float)),
            half=D.to_dev(np.asarray(dec.half_widths, float)),
            weights=D.to_dev(np.asarray(basis.weights[0], float).reshape(J, K, d)),
            biases=D.to_dev(np.asarray(basis.biases[0], float).reshape(J, K)
                            if basis.biases[0] is not None else np.zeros((J, K))),
            axes=D.to_dev(np.concatenate(axes)),
            axis_off=D.to_dev(np.cumsum([0] + [a.size for a in axes[:-1]]).astype(np.int64)),
            op_coef=D.to_dev(np.array(coef_rows, dtype=float)),
            con_pts=D.to_dev(np.concatenate(con_pts) if con_pts else np.zeros((1, d))),
            box=D.to_dev(box), con_ptr=D.to_dev(con_ptr), con_idx=D.to_dev(con_idx.astype(np.int32)),
            con_grp=D.to_dev(con_grp.astype(np.int32)), tiles=D.to_dev(tiles))
        self.desc = _lib.AssemblyDesc(
            dim=d, nsub=J, count_per_dim=dec.count_per_dim, nfeat=K,
            activation=ACTIVATIONS[basis.activation], ngroups=len(problem.constraints),
            reach=int(np.ceil(dec.overlap_ratio)) + 1,
            centers=D.ptr(keep["centers"]), half=D.ptr(keep["half"]), weights=D.ptr(keep["weights"]),
            biases=D.ptr(keep["biases"]), axes=D.ptr(keep["axes"]), axis_off=D.ptr(keep["axis_off"]),
            op_coef=D.ptr(keep["op_coef"]), con_pts=D.ptr(keep["con_pts"]), box=D.ptr(keep["box"]),
            con_ptr=D.ptr(keep["con_ptr"]), con_idx=D.ptr(keep["con_idx"]),
            con_grp=D.ptr(keep["con_grp"]), n_tiles=len(tiles), tiles=D.ptr(keep["tiles"]))

    def new_store(self) -> D.DeviceBlocks:
        t = D.torch()
        J, K = self.layout.J, self.layout.K
        vals = t.empty(max(self.layout.total, 1), dtype=t.float64, device=D.require_cuda())
        return D.DeviceBlocks(self.layout, vals, np.full(J, K, np.int32),
                              np.arange(J, dtype=np.int64) * K)

    def launch(self, store: D.DeviceBlocks) -> None:
        _lib.check(_lib.lib().fl_assemble(C.byref(self.desc), C.byref(store.struct()),
                                          D.stream_ptr()), "fl_assemble")

    def system(self, store: D.DeviceBlocks) -> GlobalSystem:
        store._asm_keepalive = self.keep
        return GlobalSystem(self.problem, self.dec, self.basis, self.rhs, self.n_interior,
                            self.row_count, self.basis.column_count, self.axes, store=store,
                            block_rows=[r.astype(int) for r in self.rows_per_block])


def _validate(problem, dec, basis):
    if basis.decomposition is not dec and (
            basis.decomposition.count_per_dim != dec.count_per_dim
            or basis.decomposition.overlap_ratio != dec.overlap_ratio
            or not np.array_equal(basis.decomposition.domain.bounds, dec.domain.bounds)):
        raise InvalidInputError("basis was initialized on a different decomposition")
    if not np.array_equal(problem.domain.bounds, dec.domain.bounds):
        raise InvalidInputError("problem and decomposition domains differ")
    if problem.mask_jets is not None or problem.lift_jets is not None:
        raise NotImplementedError(
            "hard-constraint (mask/lift) problems are not on the accelerated path yet")
    if basis.depth != 1:
        raise NotImplementedError("only depth-1 feature networks are on the accelerated path")
    if basis.activation not in ACTIVATIONS:
        raise InvalidInputError(f"unknown activation {basis.activation!r}")
    if dec.dim > 3:
        raise NotImplementedError("dimension > 3 is not on the accelerated path")


def _lattice_counts(dec, basis, interior_per_dim):
    d = dec.dim
    if interior_per_dim is None:
        from .linalg import lattice_counts
        return (lattice_counts(dec.count_per_dim, basis.feature_count, d, 0),) * d
    counts = (tuple(int(c) for c in interior_per_dim)
              if isinstance(interior_per_dim, (tuple, list))
              else (int(interior_per_dim),) * d)
    if len(counts) != d:
        raise InvalidInputError(
            f"interior_per_dim has {len(counts)} entries for a {d}-dim problem")
    if min(counts) < 2:
        raise InvalidInputError("interior_per_dim must be at least 2")
    return counts


def _coverage(problem, dec, axes, n_interior):
    """assembly.py:171-177. The lattice is a product grid, so a point is
    uncovered iff one of its coordinates is covered in no dimension."""
    d = dec.dim
    covered = [np.any(np.abs(axes[i][None, :] - dec.centers[i][:, None]) < dec.half_widths[i], axis=0)
               for i in range(d)]
    n_cov = int(np.prod([c.sum() for c in covered]))
    if n_cov < n_interior:
        raise CoverageError(f"{n_interior - n_cov} interior points covered by no subdomain")
    for con in problem.constraints:
        mem = _member(dec, con.points)
        if not np.all(np.all(mem.any(axis=1), axis=0)):
            raise CoverageError(f"constraint {con.label!r} has uncovered points")


def assemble(problem, dec, basis, interior_per_dim=None) -> GlobalSystem:
    """Build the weighted least-squares system on the device (`assembly.py:124-238`)."""
    plan = AssemblyPlan(problem, dec, basis, interior_per_dim)
    store = plan.new_store()
    plan.launch(store)
    return plan.system(store)
