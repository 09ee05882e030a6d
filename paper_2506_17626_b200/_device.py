"""Device-side plumbing: torch tensors own every device buffer; the C-ABI
only sees raw pointers (include/featlsq_b200.h `fl_blockop`).

A `BlockLayout` holds the row structure shared by the raw blocks A_j and the
orthonormal blocks Q_j: per-block row counts m_j, leading dimensions ld_j
(multiples of 16 doubles), element offsets, the global row id of every
block row and the fixed-order row-gather map. A `DeviceBlocks` couples a
layout with one values buffer and a column map (ncols_j, col_off_j) and
hands out the `fl_blockop` struct.
"""

from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib
from .errors import DeviceError

LD_ALIGN = 16

_torch = None


def torch():
    global _torch
    if _torch is None:
        import torch as t
        _torch = t
    return _torch


def require_cuda():
    t = torch()
    if not t.cuda.is_available():
        raise DeviceError("no CUDA device: the featlsq B200 path runs only on the GPU "
                          "(there is no CPU fallback)")
    _lib.lib()
    return t.device("cuda", t.cuda.current_device())


def stream_ptr() -> int:
    return torch().cuda.current_stream().cuda_stream


# host<->device traffic of the product path (bench.py reports it per step)
XFER = {"h2d": 0, "d2h": 0}


def to_dev(arr, dtype=None):
    t = torch()
    a = np.ascontiguousarray(arr if dtype is None else np.asarray(arr, dtype=dtype))
    if a.size == 0:
        a = np.zeros(1, dtype=a.dtype)
    XFER["h2d"] += a.nbytes
    return t.from_numpy(a).to(require_cuda(), non_blocking=False)


def to_host(tensor) -> np.ndarray:
    out = tensor.cpu().numpy()
    XFER["d2h"] += out.nbytes
    return out


def ptr(tensor) -> int:
    return tensor.data_ptr() if tensor is not None else 0


def round_up(x, a):
    return (x + a - 1) // a * a


def tile_table(extent, step) -> np.ndarray:
    """(n, 2) int32 rows (j, start) for start in range(0, extent[j], step)."""
    extent = np.asarray(extent, dtype=np.int64)
    per = (extent + step - 1) // step
    j = np.repeat(np.arange(extent.size, dtype=np.int64), per)
    first = np.repeat(np.cumsum(per) - per, per)
    start = (np.arange(j.size, dtype=np.int64) - first) * step
    return np.stack([j, start], axis=1).astype(np.int32).reshape(-1, 2)


def stable_argsort(keys: np.ndarray) -> np.ndarray:
    """Stable argsort as int32 (on the device when one is present)."""
    t = torch()
    if keys.size > 1 << 16 and t.cuda.is_available():
        k = t.from_numpy(np.ascontiguousarray(keys)).to(require_cuda())
        return t.sort(k, stable=True).indices.to(t.int32).cpu().numpy()
    return np.argsort(keys, kind="stable").astype(np.int32)


class BlockLayout:
    """Row structure of a block store (see module docstring)."""

    def __init__(self, nrows: int, K: int, rows_per_block: list):
        self.nrows = int(nrows)
        self.K = int(K)
        self.J = len(rows_per_block)
        self.m = np.array([r.size for r in rows_per_block], dtype=np.int32)
        self.ld = np.maximum(round_up(self.m.astype(np.int64), LD_ALIGN), LD_ALIGN).astype(np.int32)
        self.off = np.zeros(self.J, dtype=np.int64)
        if self.J:
            self.off[1:] = np.cumsum(self.ld.astype(np.int64) * K)[:-1]
        self.total = int(self.off[-1] + int(self.ld[-1]) * K) if self.J else 0
        self.row_off = np.zeros(self.J, dtype=np.int64)
        if self.J:
            self.row_off[1:] = np.cumsum(self.m.astype(np.int64))[:-1]
        self.partial_len = int(self.m.sum())
        self.rows = (np.concatenate(rows_per_block).astype(np.int32) if self.J
                     else np.zeros(0, np.int32))
        # gather map: sources of each global row in increasing partial index
        # (= increasing block index, as blocks are concatenated in order)
        self.gsrc = stable_argsort(self.rows)
        counts = np.bincount(self.rows, minlength=self.nrows) if self.rows.size else \
            np.zeros(self.nrows, np.int64)
        self.gptr = np.zeros(self.nrows + 1, dtype=np.int32)
        self.gptr[1:] = np.cumsum(counts)
        # forward (row) tiles: one CTA per FL_ROW_TILE rows of a block
        self.row_tiles = tile_table(self.m, _lib.FL_ROW_TILE)
        self.max_rows = int(self.m.max()) if self.J else 0
        self._dev = None

    def dev(self):
        if self._dev is None:
            t = torch()
            self._dev = dict(
                off=to_dev(self.off), ld=to_dev(self.ld), m=to_dev(self.m),
                row_off=to_dev(self.row_off), rows=to_dev(self.rows), gptr=to_dev(self.gptr),
                gsrc=to_dev(self.gsrc), row_tiles=to_dev(self.row_tiles),
                partial=t.empty(max(_lib.FL_LSQR_SPLIT_MAX * self.partial_len, 1), dtype=t.float64,
                                device=require_cuda()),
                counter=t.zeros(4, dtype=t.int32, device=require_cuda()),
            )
        return self._dev


def blocks_from_host(nrows: int, rows_list, mats_list) -> "DeviceBlocks":
    """Upload host blocks (row ids, (m_j, n_j) matrices) as a device block
    operator with y-space offsets = prefix sums of n_j."""
    ncols = np.array([m.shape[1] for m in mats_list], dtype=np.int32)
    K = int(ncols.max()) if len(ncols) else 1
    layout = BlockLayout(nrows, K, [np.asarray(r) for r in rows_list])
    buf = np.zeros(max(layout.total, 1))
    for j, mat in enumerate(mats_list):
        m, ld, off = int(layout.m[j]), int(layout.ld[j]), int(layout.off[j])
        blk = np.zeros((K, ld))
        blk[:mat.shape[1], :m] = np.asarray(mat, dtype=float).T
        buf[off:off + ld * K] = blk.ravel()
    col_off = np.concatenate([[0], np.cumsum(ncols)[:-1]]).astype(np.int64)
    return DeviceBlocks(layout, to_dev(buf), ncols, col_off)


class DeviceBlocks:
    """A values buffer over a layout plus a column map -> fl_blockop."""

    def __init__(self, layout: BlockLayout, vals, ncols: np.ndarray, col_off: np.ndarray):
        self.layout = layout
        self.vals = vals
        self.ncols = np.asarray(ncols, dtype=np.int32)
        self.col_off = np.asarray(col_off, dtype=np.int64)
        self.ncols_total = int((self.col_off + self.ncols).max()) if layout.J else 0
        self.col_tiles = tile_table(self.ncols, _lib.FL_COL_TILE)
        self._dev = None
        self._struct = None

    def dev(self):
        if self._dev is None:
            t = torch()
            L = self.layout
            n_scr = 2 * max(len(self.col_tiles), len(L.row_tiles), (L.nrows + 255) // 256,
                            _lib.FL_LSQR_SPLIT_MAX * L.J, 1) + 64
            # largest blocks first: the per-block LSQR CTAs then finish with a short tail
            work = L.m.astype(np.int64) * np.maximum(self.ncols.astype(np.int64), 1)
            order = np.argsort(-work, kind="stable").astype(np.int32)
            self._dev = dict(ncols=to_dev(self.ncols), col_off=to_dev(self.col_off),
                             col_tiles=to_dev(self.col_tiles), order=to_dev(order),
                             scratch=t.zeros(n_scr, dtype=t.float64, device=require_cuda()))
        return self._dev

    def struct(self) -> _lib.BlockOp:
        if self._struct is None:
            L, Ld, d = self.layout, self.layout.dev(), self.dev()
            self._struct = _lib.BlockOp(
                nblocks=L.J, nrows=L.nrows, ncols_total=self.ncols_total,
                partial_len=L.partial_len, max_rows=L.max_rows,
                max_ncols=int(self.ncols.max()) if L.J else 0,
                vals=ptr(self.vals), off=ptr(Ld["off"]), ld=ptr(Ld["ld"]), m=ptr(Ld["m"]),
                ncols=ptr(d["ncols"]), col_off=ptr(d["col_off"]), row_off=ptr(Ld["row_off"]),
                rows=ptr(Ld["rows"]), gptr=ptr(Ld["gptr"]), gsrc=ptr(Ld["gsrc"]),
                n_row_tiles=len(L.row_tiles), row_tiles=ptr(Ld["row_tiles"]),
                n_col_tiles=len(self.col_tiles), col_tiles=ptr(d["col_tiles"]),
                partial=ptr(Ld["partial"]), red_scratch=ptr(d["scratch"]),
                counter=ptr(Ld["counter"]), order=ptr(d["order"]))
        return self._struct

    # ---- products (stream ordered; results stay on device) ----
    def apply(self, x_dev, out_dev=None):
        t = torch()
        out = out_dev if out_dev is not None else t.empty(
            max(self.layout.nrows, 1), dtype=t.float64, device=x_dev.device)
        _lib.check(_lib.lib().fl_blockop_apply(C.byref(self.struct()), ptr(x_dev), ptr(out),
                                               stream_ptr()), "fl_blockop_apply")
        return out

    def apply_t(self, r_dev, out_dev=None):
        t = torch()
        out = out_dev if out_dev is not None else t.zeros(
            max(self.ncols_total, 1), dtype=t.float64, device=r_dev.device)
        _lib.check(_lib.lib().fl_blockop_apply_t(C.byref(self.struct()), ptr(r_dev), ptr(out),
                                                 stream_ptr()), "fl_blockop_apply_t")
        return out

    # ---- host views ----
    def block_host(self, j: int, ncols: int | None = None) -> np.ndarray:
        """Block j as a C-order (m_j, ncols) numpy array (D2H)."""
        L = self.layout
        nc = int(self.ncols[j]) if ncols is None else ncols
        m, ld, off = int(L.m[j]), int(L.ld[j]), int(L.off[j])
        if nc == 0 or m == 0:
            return np.zeros((m, nc))
        seg = self.vals[off:off + ld * nc].view(nc, ld)[:, :m]
        return np.ascontiguousarray(to_host(seg).T)

    def all_blocks_host(self, ncols=None):
        """All blocks in one D2H copy."""
        host = to_host(self.vals) if self.layout.J else np.zeros(0)
        L = self.layout
        out = []
        for j in range(L.J):
            nc = int(self.ncols[j]) if ncols is None else int(ncols[j])
            m, ld, off = int(L.m[j]), int(L.ld[j]), int(L.off[j])
            out.append(np.ascontiguousarray(host[off:off + ld * nc].reshape(nc, ld)[:, :m].T))
        return out

    def set_block(self, j: int, mat: np.ndarray) -> None:
        L = self.layout
        m, ld, off, K = int(L.m[j]), int(L.ld[j]), int(L.off[j]), int(self.ncols[j])
        buf = np.zeros((K, ld))
        buf[:, :m] = np.asarray(mat, dtype=float).T
        self.vals[off:off + ld * K].copy_(torch().from_numpy(buf.ravel()))
        XFER["h2d"] += buf.nbytes
