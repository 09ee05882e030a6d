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
import hashlib
from dataclasses import dataclass, field

import numpy as np
import scipy.sparse

from . import _device as D
from . import _lib
from ._featlsq import ref_assembly
from .basis import ACTIVATIONS
from .domains import support_runs
from .errors import CapExceededError, CoverageError, InvalidInputError
from .jets import triples

DENSE_SIZE_CAP = 20_000


SubdomainBlock = ref_assembly.SubdomainBlock   # `assembly.py:43-50`


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


def adopt_system(system) -> GlobalSystem:
    """A featlsq `GlobalSystem` with host blocks (`assembly.py:53-88`, e.g.
    built by the reference `assemble` or by hand) as a device-resident
    system: its blocks are uploaded once into a block store. Device systems
    pass through unchanged."""
    if isinstance(system, GlobalSystem):
        return system
    if not all(hasattr(system, a) for a in ("blocks", "rhs", "row_count", "column_count")):
        raise InvalidInputError(f"cannot interpret {type(system)} as a GlobalSystem")
    blocks = list(system.blocks)
    k = system.basis.feature_count
    for j, blk in enumerate(blocks):
        if not np.array_equal(np.asarray(blk.columns), np.arange(j * k, (j + 1) * k)):
            raise InvalidInputError(f"block {j} does not hold columns {j * k}..{(j + 1) * k - 1}")
    store = D.blocks_from_host(system.row_count, [np.asarray(b.rows) for b in blocks],
                               [np.asarray(b.matrix, dtype=float) for b in blocks])
    out = GlobalSystem(system.problem, system.decomposition, system.basis,
                       np.asarray(system.rhs, dtype=float), system.interior_count,
                       system.row_count, system.column_count, system.lattice_axes,
                       store=store, block_rows=[np.asarray(b.rows) for b in blocks])
    out._blocks = _BlockList(blocks, out)
    return out


def apply(system: GlobalSystem, coeffs: np.ndarray) -> np.ndarray:
    """M a on the device (`assembly.py:91-96`)."""
    coeffs = np.asarray(coeffs, dtype=float)
    if coeffs.shape != (system.column_count,):
        raise InvalidInputError(
            f"coefficients must have shape ({system.column_count},), got {coeffs.shape}")
    system = adopt_system(system)
    system.sync_device()
    return D.to_host(system.store.apply(D.to_dev(coeffs)))[:system.row_count]


def apply_transpose(system: GlobalSystem, residual: np.ndarray) -> np.ndarray:
    """M^T r on the device (`assembly.py:99-104`)."""
    residual = np.asarray(residual, dtype=float)
    if residual.shape != (system.row_count,):
        raise InvalidInputError(
            f"residual must have shape ({system.row_count},), got {residual.shape}")
    system = adopt_system(system)
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


def _lift_values(problem, operator, points) -> np.ndarray:
    """Operator applied to the lift jets (`assembly.py:117-121`), zeros without a lift."""
    pts = np.atleast_2d(points)
    if problem.lift_jets is None:
        return np.zeros(pts.shape[0])
    jets = [problem.lift_jets(pts, a) for a in range(problem.domain.dim)]
    return _apply_operator(operator, jets)


def _apply_operator(op, jets) -> np.ndarray:
    """`problems.py:39-47` (same term order), for duck-typed operators."""
    out = op.value_coef * jets[0].value
    for a, jet in enumerate(jets):
        out = out + op.first_coefs[a] * jet.first + op.second_coefs[a] * jet.second
    return out


def _make_desc(dec, basis, layout, axes, coef_rows, con_pts, box, con_ptr, con_idx, con_grp,
               ngroups, mask_int, mask_con, counts):
    """Upload the K1 inputs and build the `fl_assembly_desc`."""
    d, J, K = dec.dim, dec.subdomain_count, basis.feature_count
    tiles = D.tile_table(layout.ld, _lib.FL_ASM_TILE)
    keep = dict(
        centers=D.to_dev(np.asarray(dec.centers, float)),
        half=D.to_dev(np.asarray(dec.half_widths, float)),
        weights=D.to_dev(np.asarray(basis.weights[0], float).reshape(J, K, d)),
        biases=D.to_dev(np.asarray(basis.biases[0], float).reshape(J, K)
                        if basis.biases[0] is not None else np.zeros((J, K))),
        axes=D.to_dev(np.concatenate(axes) if len(axes) else np.zeros(1)),
        axis_off=D.to_dev(np.cumsum([0] + [a.size for a in axes[:-1]]).astype(np.int64)
                          if len(axes) else np.zeros(d, np.int64)),
        op_coef=D.to_dev(np.array(coef_rows, dtype=float)),
        con_pts=D.to_dev(con_pts if con_pts.shape[0] else np.zeros((1, d))),
        box=D.to_dev(box), con_ptr=D.to_dev(con_ptr), con_idx=D.to_dev(con_idx.astype(np.int32)),
        con_grp=D.to_dev(con_grp.astype(np.int32)), tiles=D.to_dev(tiles))
    if mask_int is not None:
        keep["mask_int"] = D.to_dev(mask_int)
    if mask_con is not None:
        keep["mask_con"] = D.to_dev(mask_con)
    stride = (C.c_int64 * 3)(*([int(np.prod(counts[i + 1:])) for i in range(d)] + [0] * (3 - d)))
    desc = _lib.AssemblyDesc(
        dim=d, nsub=J, count_per_dim=dec.count_per_dim, nfeat=K,
        activation=ACTIVATIONS[basis.activation], ngroups=ngroups,
        reach=int(np.ceil(dec.overlap_ratio)) + 1,
        centers=D.ptr(keep["centers"]), half=D.ptr(keep["half"]), weights=D.ptr(keep["weights"]),
        biases=D.ptr(keep["biases"]), axes=D.ptr(keep["axes"]), axis_off=D.ptr(keep["axis_off"]),
        op_coef=D.ptr(keep["op_coef"]), con_pts=D.ptr(keep["con_pts"]), box=D.ptr(keep["box"]),
        con_ptr=D.ptr(keep["con_ptr"]), con_idx=D.ptr(keep["con_idx"]),
        con_grp=D.ptr(keep["con_grp"]), n_tiles=len(tiles), tiles=D.ptr(keep["tiles"]),
        mask_int=D.ptr(keep.get("mask_int")), mask_con=D.ptr(keep.get("mask_con")),
        lattice_stride=stride)
    return keep, desc


class AssemblyPlan:
    """Everything `assemble` derives on the host, uploaded once: the layout,
    the right-hand side and the K1 descriptor. `launch(vals)` re-runs only
    the kernel (the device-resident benchmark step uses this)."""

    def __init__(self, problem, dec, basis, interior_per_dim=None):
        _validate(problem, dec, basis)
        d = dec.dim
        masked = problem.mask_jets is not None
        counts = _lattice_counts(dec, basis, interior_per_dim, extra=1 if masked else 0)
        if not masked:
            axes = tuple(np.linspace(dec.domain.bounds[i, 0], dec.domain.bounds[i, 1], counts[i])
                         for i in range(d))
        else:
            # cell centres for hard-constrained problems (assembly.py:159-166)
            steps = dec.domain.widths / np.asarray(counts)
            axes = tuple(dec.domain.bounds[i, 0] + steps[i] * (np.arange(counts[i]) + 0.5)
                         for i in range(d))
        n_interior = int(np.prod(counts))
        _coverage(problem, dec, axes, n_interior)

        # right-hand side (assembly.py:179-192), host: user callables
        mesh = np.meshgrid(*axes, indexing="ij")
        interior = np.stack([m.ravel() for m in mesh], axis=1)
        iw = 1.0 / np.sqrt(n_interior)
        rhs_parts = [(np.asarray(problem.forcing(interior), dtype=float)
                      - _lift_values(problem, problem.operator, interior)) * iw]
        coef_rows = [[float(problem.operator.value_coef), iw, *problem.operator.first_coefs,
                      *problem.operator.second_coefs]]
        con_pts = []
        for con in problem.constraints:
            pts = np.atleast_2d(np.asarray(con.points, dtype=float))
            w = np.sqrt(con.weight / pts.shape[0])
            rhs_parts.append((np.asarray(con.targets, dtype=float)
                              - _lift_values(problem, con.operator, pts)) * w)
            op = con.operator
            coef_rows.append([float(op.value_coef), w, *op.first_coefs, *op.second_coefs])
            con_pts.append(pts)
        self.rhs = np.concatenate(rhs_parts)
        if len(problem.constraints) > 7:
            raise NotImplementedError("more than 7 constraint groups")

        K = basis.feature_count
        row_count, box, con_ptr, con_idx, con_grp, rows_per_block, self.layout = _cached_layout(
            problem, dec, axes, counts, K, con_pts)
        goff = np.cumsum([0] + [p.shape[0] for p in con_pts])
        con_idx = con_idx + goff[con_grp].astype(np.int32) if con_idx.size else con_idx
        self.rows_per_block = rows_per_block
        self.problem, self.dec, self.basis = problem, dec, basis
        self.axes, self.n_interior, self.row_count = axes, n_interior, row_count
        all_con = np.concatenate(con_pts) if con_pts else np.zeros((0, d))
        mask_int = mask_con = None
        if masked:  # per-point mask jets along every axis (assembly.py:111-112)
            mask_int = triples(problem.mask_jets, interior, d)
            mask_con = triples(problem.mask_jets, all_con, d) if all_con.shape[0] else None
        self.keep, self.desc = _make_desc(
            dec, basis, self.layout, axes, coef_rows, all_con, box, con_ptr, con_idx, con_grp,
            len(problem.constraints), mask_int, mask_con, counts)

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


# Row structure of the last few lattices (block runs, constraint membership,
# global row ids, BlockLayout with its device tables). It depends only on the
# decomposition's centres and half widths, the lattice axes and the
# constraint points, so it is keyed by a digest of exactly those arrays: a
# repeated assemble on the same geometry (e.g. a new basis or right-hand
# side) skips the host-side layout work; any change of geometry misses.
_LAYOUT_CACHE: dict = {}
_LAYOUT_CACHE_MAX = 2


def _cached_layout(problem, dec, axes, counts, K, con_pts):
    h = hashlib.blake2b(digest_size=20)
    h.update(repr((int(dec.dim), int(dec.count_per_dim), int(K), tuple(int(c) for c in counts),
                   len(con_pts))).encode())
    for a in (dec.centers, dec.half_widths, *axes, *con_pts):
        a = np.ascontiguousarray(a, dtype=np.float64)
        h.update(repr(a.shape).encode())
        h.update(a.tobytes())
    key = h.digest()
    hit = _LAYOUT_CACHE.get(key)
    if hit is None:
        row_count, box, con_ptr, con_idx, con_grp, rows_per_block = _layout_inputs(
            problem, dec, None, axes, counts)
        hit = (row_count, box, con_ptr, con_idx, con_grp, rows_per_block,
               D.BlockLayout(row_count, K, rows_per_block))
        while len(_LAYOUT_CACHE) >= _LAYOUT_CACHE_MAX:
            _LAYOUT_CACHE.pop(next(iter(_LAYOUT_CACHE)))
        _LAYOUT_CACHE[key] = hit
    return hit


def _validate(problem, dec, basis):
    if basis.decomposition is not dec and (
            basis.decomposition.count_per_dim != dec.count_per_dim
            or basis.decomposition.overlap_ratio != dec.overlap_ratio
            or not np.array_equal(basis.decomposition.domain.bounds, dec.domain.bounds)):
        raise InvalidInputError("basis was initialized on a different decomposition")
    if not np.array_equal(problem.domain.bounds, dec.domain.bounds):
        raise InvalidInputError("problem and decomposition domains differ")
    if basis.depth != 1:
        raise NotImplementedError("only depth-1 feature networks are on the accelerated path")
    if basis.activation not in ACTIVATIONS:
        raise InvalidInputError(f"unknown activation {basis.activation!r}")
    if dec.dim > 3:
        raise NotImplementedError("dimension > 3 is not on the accelerated path")


def _lattice_counts(dec, basis, interior_per_dim, extra=0):
    d = dec.dim
    if interior_per_dim is None:
        # masked problems get one extra point per subdomain and dimension (assembly.py:141-145)
        from .linalg import lattice_counts
        return (lattice_counts(dec.count_per_dim, basis.feature_count, d, extra),) * d
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


# ---------------------------------------------------------------------------
# prediction and testing (assembly.py:244-318): K1 evaluates the solution
# blocks at arbitrary points (value operator, unit weight, mask values)

class SolutionBlocks:
    """Device blocks P_j = mask * window_j * features_j at the points inside
    subdomain j (rows = point indices), plus the lift values: predictions are
    P a + lift (`assembly.py:244-272`)."""

    def __init__(self, problem, dec, basis, points):
        _validate(problem, dec, basis)
        pts = np.atleast_2d(np.asarray(points, dtype=float))
        n, d = pts.shape[0], dec.dim
        if d != pts.shape[1]:
            raise InvalidInputError(f"points must have {d} columns, got {pts.shape[1]}")
        J, K, S = dec.subdomain_count, basis.feature_count, dec.count_per_dim
        mem = _member(dec, pts)
        multi = np.array(np.unravel_index(np.arange(J), (S,) * d)).T
        rows = []
        for j in range(J):
            inside = mem[0, multi[j, 0]].copy()
            for i in range(1, d):
                inside &= mem[i, multi[j, i]]
            rows.append(np.nonzero(inside)[0])
        sizes = np.array([r.size for r in rows], dtype=np.int64)
        con_ptr = np.concatenate([[0], np.cumsum(sizes)]).astype(np.int64)
        con_idx = np.concatenate(rows).astype(np.int32) if J else np.zeros(0, np.int32)
        coef_rows = [[0.0] * (2 + 2 * d), [1.0, 1.0] + [0.0] * (2 * d)]
        mask_con = None
        if problem.mask_value is not None and n:
            mv = np.asarray(problem.mask_value(pts), dtype=float)
            mask_con = np.zeros((n, d, 3))
            mask_con[:, :, 0] = mv[:, None]
        self.layout = D.BlockLayout(n, K, rows)
        self.rows = rows
        self.points = pts
        self.column_count = basis.column_count
        self.lift = (np.asarray(problem.lift_value(pts), dtype=float) if problem.lift_value
                     else np.zeros(n))
        keep, desc = _make_desc(dec, basis, self.layout, (), coef_rows, pts,
                                np.zeros((J, d, 2), np.int32), con_ptr, con_idx,
                                np.zeros(con_idx.size, np.int32), 1, None, mask_con, (0,) * d)
        t = D.torch()
        vals = t.empty(max(self.layout.total, 1), dtype=t.float64, device=D.require_cuda())
        self.store = D.DeviceBlocks(self.layout, vals, np.full(J, K, np.int32),
                                    np.arange(J, dtype=np.int64) * K)
        if self.layout.J:
            _lib.check(_lib.lib().fl_assemble(C.byref(desc), C.byref(self.store.struct()),
                                              D.stream_ptr()), "fl_assemble")
        self._keep = keep
        self._csr = None

    def csr(self) -> scipy.sparse.csr_matrix:
        if self._csr is None:
            K = self.layout.K
            mats = self.store.all_blocks_host()
            r, c, v = [], [], []
            for j, (inside, mat) in enumerate(zip(self.rows, mats)):
                if inside.size == 0:
                    continue
                r.append(np.repeat(inside, K))
                c.append(np.tile(np.arange(j * K, (j + 1) * K), inside.size))
                v.append(mat.ravel())
            n = self.points.shape[0]
            if r:
                self._csr = scipy.sparse.coo_matrix(
                    (np.concatenate(v), (np.concatenate(r), np.concatenate(c))),
                    shape=(n, self.column_count)).tocsr()
            else:
                self._csr = scipy.sparse.csr_matrix((n, self.column_count))
        return self._csr

    def predict_device(self, coeffs_dev):
        """P a + lift on the device (n,)."""
        out = self.store.apply(coeffs_dev)[:self.points.shape[0]]
        return out + D.torch().from_numpy(self.lift).to(out.device)


def solution_blocks(problem, dec, basis, points) -> SolutionBlocks:
    return SolutionBlocks(problem, dec, basis, points)


def solution_matrix(problem, dec, basis, points):
    """(CSR P, lift) with predictions P a + lift (`assembly.py:244-272`);
    P's entries are evaluated on the device."""
    sb = SolutionBlocks(problem, dec, basis, points)
    return sb.csr(), sb.lift


def evaluate_solution(problem, dec, basis, coeffs, points) -> np.ndarray:
    """mask * sum_j window_j sum_k a_jk feature_jk + lift (`assembly.py:275-283`)."""
    coeffs = np.asarray(coeffs, dtype=float)
    if coeffs.shape != (basis.column_count,):
        raise InvalidInputError(f"coefficients must have shape ({basis.column_count},)")
    sb = SolutionBlocks(problem, dec, basis, points)
    if sb.points.shape[0] == 0:
        return np.zeros(0)
    return D.to_host(sb.predict_device(D.to_dev(coeffs)))


# featlsq's own test-lattice helpers (`assembly.py:286-318`)
TestSet = ref_assembly.TestSet
make_test_set = ref_assembly.make_test_set
l1_error = ref_assembly.l1_error
