"""Drop-in `lsqr` with a device-resident Golub-Kahan loop (reference:
featlsq/solvers.py:24-145).

The recurrences run in CUDA (K4, csrc/qop.cu); the host enqueues the whole
iteration budget and reads back only scalars (and x / the monitor's best
iterate at the end). Operator polymorphism follows `as_operator`
(solvers.py:33-44):

- a `PreconditionedOperator` or a `GlobalSystem` already lives on the device
  as dense blocks and is streamed directly;
- a 2-D array is uploaded as one dense block;
- any other object with `matvec/rmatvec` (an `Operator`) or
  `apply/apply_transpose` is probed into a dense device block through its own
  products (`size cap` below) — the loop itself never runs on the host.

Monitor semantics (solvers.py:47-69): without an `error_fn` the device keeps
the best (lowest-residual) iterate itself and the records are rebuilt from
the device phibar trace; with a `monitor.DeviceL1Error` (the runner's
test-lattice error) the error of every recorded iterate is evaluated inside
the device loop (K6) and the best iterate is kept on the device; with any
other `error_fn` the loop is run in chunks of `stride` iterations and x is
copied back at each recorded iteration to call it. Keyword-only `atol`/`btol`/`conlim` add scipy's stopping rule (SURVEY.md
§0 F2); the default is the reference behaviour, a fixed budget.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _device as D
from . import _lib
from ._featlsq import ref_assembly, ref_solvers
from .errors import DivergenceError, InvalidInputError

PROBE_CAP = 50_000_000  # entries of a host-callback operator probed onto the device


Operator = ref_solvers.Operator                    # `solvers.py:24-30`
ConvergenceMonitor = ref_solvers.ConvergenceMonitor  # `solvers.py:47-69`


def as_operator(thing):
    """`solvers.py:33-44`, with a `GlobalSystem` (device-resident or featlsq's
    host one) applied through the device block products."""
    from .assembly import GlobalSystem, adopt_system, apply, apply_transpose
    if isinstance(thing, Operator):
        return thing
    if isinstance(thing, (GlobalSystem, ref_assembly.GlobalSystem)):
        system = adopt_system(thing)
        return Operator(lambda v: apply(system, v), lambda r: apply_transpose(system, r),
                        system.shape)
    if hasattr(thing, "apply") and hasattr(thing, "apply_transpose"):
        return Operator(thing.apply, thing.apply_transpose, thing.shape)
    try:
        arr = np.asarray(thing, dtype=float)
    except (TypeError, ValueError):
        arr = np.zeros(0)
    if arr.ndim != 2:
        raise InvalidInputError(f"cannot interpret {type(thing)} as an operator")
    return Operator(lambda v: arr @ v, lambda r: arr.T @ r, arr.shape)


@dataclass(frozen=True)
class SolveResult(ref_solvers.SolveResult):
    """featlsq's `SolveResult` (`solvers.py:72-84`) plus scipy's `istop` code
    when the keyword-only stopping rule is used (0 otherwise)."""

    istop: int = 0


def _dense_blocks(arr: np.ndarray) -> D.DeviceBlocks:
    """One dense block covering every row (rows 0..N-1, columns 0..n-1)."""
    n_rows, n_cols = arr.shape
    layout = D.BlockLayout(n_rows, n_cols, [np.arange(n_rows)])
    t = D.torch()
    buf = np.zeros((n_cols, int(layout.ld[0])))
    buf[:, :n_rows] = arr.T
    vals = t.from_numpy(buf.ravel()).to(D.require_cuda())
    return D.DeviceBlocks(layout, vals, np.array([n_cols], np.int32), np.array([0], np.int64))


def device_operator(operator):
    """Resolve anything `as_operator` accepts to device blocks + shape."""
    from .assembly import GlobalSystem, adopt_system
    from .filtering import PreconditionedOperator
    if isinstance(operator, PreconditionedOperator):
        return operator.device_blocks, operator.shape
    if isinstance(operator, GlobalSystem) or isinstance(operator, ref_assembly.GlobalSystem):
        operator = adopt_system(operator)
        operator.sync_device()
        return operator.store, operator.shape
    if isinstance(operator, D.DeviceBlocks):
        return operator, (operator.layout.nrows, operator.ncols_total)
    if isinstance(operator, Operator) or (hasattr(operator, "apply")
                                          and hasattr(operator, "apply_transpose")):
        op = as_operator(operator)
        m, n = (int(s) for s in op.shape)
        if m * n > PROBE_CAP:
            raise InvalidInputError(
                f"host-callback operator of shape {op.shape} exceeds the device probe cap")
        eye = np.eye(n)
        dense = np.stack([np.asarray(op.matvec(eye[:, c]), dtype=float) for c in range(n)], axis=1) \
            if n else np.zeros((m, 0))
        return _dense_blocks(dense), (m, n)
    arr = np.asarray(operator, dtype=float)
    if arr.ndim != 2:
        raise InvalidInputError(f"cannot interpret {type(operator)} as an operator")
    return _dense_blocks(arr), arr.shape


class DeviceLsqr:
    """Device buffers + state of one LSQR run over a `DeviceBlocks` operator.
    Reusable: `run()` re-initialises from a device rhs."""

    def __init__(self, blocks: D.DeviceBlocks, max_iters: int):
        t = D.torch()
        dev = D.require_cuda()
        self.blocks = blocks
        n_rows = blocks.layout.nrows
        n = max(blocks.ncols_total, 1)
        self.max_iters = int(max_iters)
        f64 = dict(dtype=t.float64, device=dev)
        self.u = t.empty(max(n_rows, 1), **f64)
        self.v, self.vp, self.w, self.x, self.xbest = (t.zeros(n, **f64) for _ in range(5))
        self.trace = t.zeros(self.max_iters + 2, **f64)
        # u at every block row (block-local order), for the fused kernel's contiguous reads
        self.ub = t.empty(max(blocks.layout.partial_len, 1), **f64)
        self.state = t.zeros(C.sizeof(_lib.LsqrState), dtype=t.uint8, device=dev)
        self.vecs = _lib.LsqrVecs(*(D.ptr(a) for a in (self.u, self.v, self.vp, self.w, self.x,
                                                          self.xbest, self.trace, self.ub)))

    def reset_state(self, stride: int, track_best: bool, atol=None, btol=None, conlim=1e8,
                    monitor: bool = False):
        st = _lib.LsqrState()
        st.best = np.inf if track_best else -np.inf
        st.best_it = -1
        st.stride = max(int(stride), 1)
        st.monitor = 1 if monitor else 0
        if atol is not None or btol is not None:
            st.use_rule = 1
            st.atol = float(atol or 0.0)
            st.btol = float(btol or 0.0)
            st.ctol = 1.0 / conlim if conlim > 0 else 0.0
        host = np.frombuffer(bytes(st), dtype=np.uint8).copy()
        self.state.copy_(D.torch().from_numpy(host))

    def read_state(self) -> _lib.LsqrState:
        raw = D.to_host(self.state).tobytes()
        return _lib.LsqrState.from_buffer_copy(raw)

    def init(self, rhs_dev):
        L = _lib.lib()
        _lib.check(L.fl_lsqr_init(C.byref(self.blocks.struct()), D.ptr(rhs_dev),
                                  C.byref(self.vecs), D.ptr(self.state), D.stream_ptr()),
                   "fl_lsqr_init")

    def iterate(self, first_it: int, count: int, monitor=None):
        """Enqueue iterations first_it..first_it+count-1; `monitor` = a
        `_lib.TestMonitor` evaluated after every recorded iteration (K6)."""
        if count <= 0:
            return
        L = _lib.lib()
        if monitor is None:
            _lib.check(L.fl_lsqr_iterate(C.byref(self.blocks.struct()), C.byref(self.vecs),
                                         D.ptr(self.state), int(first_it), int(count),
                                         D.stream_ptr()), "fl_lsqr_iterate")
            return
        _lib.check(L.fl_lsqr_iterate_monitored(C.byref(self.blocks.struct()), C.byref(self.vecs),
                                               D.ptr(self.state), int(first_it), int(count),
                                               C.byref(monitor), D.stream_ptr()),
                   "fl_lsqr_iterate_monitored")
        _lib.check(L.fl_lsqr_monitor_flush(C.byref(self.blocks.struct()), C.byref(self.vecs),
                                           D.ptr(self.state), D.stream_ptr()),
                   "fl_lsqr_monitor_flush")


def lsqr(operator, rhs: np.ndarray, max_iters: int,
         monitor: ConvergenceMonitor | None = None, *,
         atol: float | None = None, btol: float | None = None,
         conlim: float = 1e8) -> SolveResult:
    """Golub-Kahan LSQR from zero with a fixed budget (`solvers.py:87-145`)."""
    blocks, shape = device_operator(operator)
    rhs = np.asarray(rhs, dtype=float)
    if rhs.shape != (shape[0],):
        raise InvalidInputError(f"rhs shape {rhs.shape} != operator rows {shape[0]}")
    monitor = monitor or ConvergenceMonitor()
    max_iters = int(max_iters)
    n = int(shape[1])
    run = DeviceLsqr(blocks, max_iters)
    from .monitor import DeviceL1Error
    dev_error = isinstance(monitor.error_fn, DeviceL1Error)
    if dev_error and monitor.error_fn.n != n:
        raise InvalidInputError(f"error function expects iterates of length {monitor.error_fn.n}, "
                                f"operator has {n} columns")
    host_error = monitor.error_fn is not None and not dev_error
    run.reset_state(monitor.stride, track_best=not host_error, atol=atol, btol=btol,
                    conlim=conlim, monitor=dev_error)
    run.init(D.to_dev(rhs))
    st = run.read_state()
    x0 = np.zeros(n)
    if st.beta == 0.0:                              # solvers.py:104-106
        monitor.observe(0, x0, lambda: 0.0)
        return SolveResult(x0, 0, 0.0, monitor)
    if st.alpha == 0.0:                             # solvers.py:110-112
        monitor.observe(0, x0, lambda: st.beta)
        return SolveResult(x0, 0, st.beta, monitor, breakdown=True)

    if dev_error:
        err_trace = D.torch().full((max_iters + 2,), float("nan"), dtype=D.torch().float64,
                                   device=run.x.device)
        mon = monitor.error_fn.struct(err_trace)
        run.iterate(1, max_iters, mon)
        st = run.read_state()
    elif not host_error:
        run.iterate(1, max_iters)
        st = run.read_state()
    else:
        it = 0
        stride = max(monitor.stride, 1)
        while it < max_iters:
            count = min(stride - (it % stride), max_iters - it)
            run.iterate(it + 1, count)
            st = run.read_state()
            done_it = int(st.it)
            if st.diverged_at:
                break
            if done_it % stride == 0 and done_it > it:
                x_now = D.to_host(run.x)[:n]
                ph = float(run.trace[done_it].item())
                monitor.observe(done_it, x_now, lambda: ph)
            it = it + count
            if st.done:
                break
    if st.diverged_at:
        raise DivergenceError(f"non-finite iterate at iteration {int(st.diverged_at)}")
    iters = int(st.it)
    x = D.to_host(run.x)[:n]
    if not host_error:
        trace = D.to_host(run.trace)
        errs = D.to_host(err_trace) if dev_error else trace
        stride = max(monitor.stride, 1)
        for it in range(1, iters + 1):
            if stride > 1 and it % stride != 0:
                continue
            monitor.records.append((it, float(trace[it]), float(errs[it])))
        if st.best_it >= 1:
            monitor.best_error = float(st.best)
            monitor.best_iteration = int(st.best_it)
            monitor.best_iterate = D.to_host(run.xbest)[:n].copy()
    return SolveResult(x, iters, float(st.phibar), monitor, bool(st.breakdown), int(st.istop))


# ---------------------------------------------------------------------------
# N4 baselines: additive Schwarz and CG on the normal equations
# (solvers.py:150-239; the runner's "cg"/"as-cg" solvers, runner.py:296-305)

class AdditiveSchwarz:
    """Block-diagonal (pseudo-)inverse of the per-subdomain Gramians
    (`solvers.py:150-178`). Same fields as the reference; `apply` and the CG
    loop run the block products on the device (K: `fl_block_precond_apply`).
    Instances built by `as_preconditioner` keep their inverses on the device
    and materialise the host tuple on first access."""

    def __init__(self, column_count, block_ranges, block_inverses, degenerate_blocks,
                 _device=None):
        self.column_count = int(column_count)
        self.block_ranges = tuple(np.asarray(r) for r in block_ranges)
        self._inverses = None if block_inverses is None else tuple(
            np.asarray(b, dtype=float) for b in block_inverses)
        self.degenerate_blocks = tuple(int(j) for j in degenerate_blocks)
        self._dev = _device          # (vals tensor (sum s_b^2,), sizes)
        self._pre = None

    @property
    def block_inverses(self) -> tuple:
        if self._inverses is None:
            vals = D.to_host(self._dev)
            out, o = [], 0
            for r in self.block_ranges:
                s = r.size
                out.append(vals[o:o + s * s].reshape(s, s).copy())
                o += s * s
            self._inverses = tuple(out)
        return self._inverses

    def device_struct(self) -> _lib.BlockPrecond:
        if self._pre is None:
            sizes = np.array([r.size for r in self.block_ranges], dtype=np.int64)
            idx_off = np.concatenate([[0], np.cumsum(sizes)]).astype(np.int64)
            val_off = np.concatenate([[0], np.cumsum(sizes * sizes)[:-1]]).astype(np.int64)
            idx = (np.concatenate(self.block_ranges).astype(np.int32) if len(sizes)
                   else np.zeros(0, np.int32))
            if self._dev is None:
                self._dev = D.to_dev(np.concatenate([b.ravel() for b in self._inverses])
                                     if len(sizes) else np.zeros(1))
            keep = dict(idx_off=D.to_dev(idx_off), idx=D.to_dev(idx), val_off=D.to_dev(val_off))
            self._keep = keep
            self._pre = _lib.BlockPrecond(
                nblocks=len(sizes), max_size=int(sizes.max()) if len(sizes) else 0,
                idx_off=D.ptr(keep["idx_off"]), idx=D.ptr(keep["idx"]),
                val_off=D.ptr(keep["val_off"]), vals=D.ptr(self._dev))
        return self._pre

    def apply(self, vec: np.ndarray) -> np.ndarray:
        vec = np.asarray(vec, dtype=float)
        if vec.shape != (self.column_count,):
            raise InvalidInputError(f"expected shape ({self.column_count},), got {vec.shape}")
        t = D.torch()
        r = D.to_dev(vec)
        z = t.zeros(max(self.column_count, 1), dtype=t.float64, device=r.device)
        _lib.check(_lib.lib().fl_block_precond_apply(C.byref(self.device_struct()), D.ptr(r),
                                                     D.ptr(z), D.stream_ptr()),
                   "fl_block_precond_apply")
        return D.to_host(z)[:self.column_count]

    def materialize(self) -> np.ndarray:
        dense = np.zeros((self.column_count, self.column_count))
        for cols, inv in zip(self.block_ranges, self.block_inverses):
            dense[np.ix_(cols, cols)] = inv
        return dense


def as_preconditioner(system, cutoff: float = 1e-14) -> AdditiveSchwarz:
    """`solvers.py:178-192` on the device: per block the Gramian A_j^T A_j,
    its eigendecomposition and the pseudo-inverse over eigenvalues above
    cutoff * the largest. K <= 96 (every paper demo): one kernel
    (`fl_as_setup`, csrc/as_setup.cu: Gramian from the resident block,
    parallel cyclic Jacobi in shared memory). Wider blocks: a batched
    library eigensolver (cuBLAS Gramian + cuSOLVER syevd) — the baseline's
    one-off setup, not on the north-star path."""
    from .assembly import adopt_system
    t = D.torch()
    system = adopt_system(system)
    system.sync_device()
    st = system.store
    L = st.layout
    K = L.K
    J = L.J
    ranges = [np.arange(j * K, (j + 1) * K) for j in range(J)]
    if K <= _lib.FL_AS_MAX_K:
        inv = t.empty(max(J * K * K, 1), dtype=t.float64, device=st.vals.device)
        deg = t.zeros(max(J, 1), dtype=t.int32, device=st.vals.device)
        _lib.check(_lib.lib().fl_as_setup(C.byref(st.struct()), float(cutoff), D.ptr(inv), D.ptr(deg),
                                          D.stream_ptr()), "fl_as_setup")
        degenerate = np.nonzero(D.to_host(deg)[:J])[0]
        return AdditiveSchwarz(system.column_count, ranges, None, tuple(int(j) for j in degenerate),
                               _device=inv)
    grams = t.empty((max(J, 1), K, K), dtype=t.float64, device=st.vals.device)
    for ldv in np.unique(L.ld):
        js = np.nonzero(L.ld == ldv)[0]
        for c0 in range(0, js.size, 64):
            chunk = js[c0:c0 + 64]
            # each block's (K, ld) panel is a contiguous slice of the store
            # (padding rows are exact zeros, so they do not change A^T A)
            panels = t.stack([st.vals[int(L.off[j]):int(L.off[j]) + K * int(ldv)].view(K, int(ldv))
                              for j in chunk])
            grams[t.from_numpy(chunk).to(st.vals.device)] = t.bmm(panels, panels.transpose(1, 2))
    evals, evecs = t.linalg.eigh(grams[:J])
    top = evals[:, -1:]
    keep = (evals > cutoff * top) & (top > 0)
    inv_vals = t.where(keep, 1.0 / t.where(keep, evals, t.ones_like(evals)), t.zeros_like(evals))
    inv = t.bmm(evecs * inv_vals[:, None, :], evecs.transpose(1, 2))
    degenerate = np.nonzero(~D.to_host(keep.all(dim=1)))[0]
    return AdditiveSchwarz(system.column_count, ranges, None, tuple(int(j) for j in degenerate),
                           _device=inv.reshape(-1).contiguous())


def cg_normal(operator, rhs: np.ndarray, max_iters: int,
              monitor: ConvergenceMonitor | None = None,
              preconditioner: AdditiveSchwarz | None = None) -> SolveResult:
    """CG on the normal equations from zero (`solvers.py:195-239`), device loop."""
    blocks, shape = device_operator(operator)
    rhs = np.asarray(rhs, dtype=float)
    if rhs.shape != (shape[0],):
        raise InvalidInputError(f"rhs shape {rhs.shape} != operator rows {shape[0]}")
    monitor = monitor or ConvergenceMonitor()
    max_iters = int(max_iters)
    n, N = int(shape[1]), int(shape[0])
    t = D.torch()
    dev = D.require_cuda()
    f64 = dict(dtype=t.float64, device=dev)
    nn = max(blocks.ncols_total, 1)
    buf = {k: t.zeros(nn, **f64) for k in ("p", "q", "r", "x", "xbest")}
    buf["z"] = t.zeros(nn, **f64) if preconditioner is not None else buf["r"]
    buf["tmp"] = t.zeros(max(blocks.layout.nrows, 1), **f64)
    buf["res"] = t.full((max_iters + 2,), float("nan"), **f64)
    buf["rhs"] = D.to_dev(rhs)
    buf["scratch"] = t.zeros(2 * 592 + 64, **f64)
    buf["counter"] = t.zeros(4, dtype=t.int32, device=dev)
    buf["out"] = t.zeros(1, **f64)
    stride = max(int(monitor.stride), 1)
    vecs = _lib.CgVecs(tmp=D.ptr(buf["tmp"]), p=D.ptr(buf["p"]), q=D.ptr(buf["q"]),
                       r=D.ptr(buf["r"]), z=D.ptr(buf["z"]), x=D.ptr(buf["x"]),
                       xbest=D.ptr(buf["xbest"]), res_trace=D.ptr(buf["res"]),
                       rhs=D.ptr(buf["rhs"]), scratch=D.ptr(buf["scratch"]),
                       counter=D.ptr(buf["counter"]), stride=stride)
    from .monitor import DeviceL1Error
    dev_error = isinstance(monitor.error_fn, DeviceL1Error)
    if dev_error and monitor.error_fn.n != n:
        raise InvalidInputError(f"error function expects iterates of length {monitor.error_fn.n}, "
                                f"operator has {n} columns")
    host_error = monitor.error_fn is not None and not dev_error
    sst = _lib.LsqrState()
    sst.best = np.inf
    sst.best_it = -1
    sst.stride = stride
    sst.monitor = 1
    state = t.from_numpy(np.frombuffer(bytes(sst), dtype=np.uint8).copy()).to(dev)
    L = _lib.lib()
    op = C.byref(blocks.struct())
    if preconditioner is not None and not isinstance(preconditioner, AdditiveSchwarz):
        # featlsq's own AdditiveSchwarz (solvers.py:149-175): same fields
        preconditioner = AdditiveSchwarz(preconditioner.column_count, preconditioner.block_ranges,
                                         preconditioner.block_inverses,
                                         preconditioner.degenerate_blocks)
    pre = C.byref(preconditioner.device_struct()) if preconditioner is not None else None
    _lib.check(L.fl_cg_init(op, C.byref(vecs), pre, D.ptr(state), D.stream_ptr()), "fl_cg_init")
    err_trace = None
    mon = None
    if dev_error:
        err_trace = t.full((max_iters + 2,), float("nan"), **f64)
        mon = monitor.error_fn.struct(err_trace)

    def read():
        return _lib.LsqrState.from_buffer_copy(D.to_host(state).tobytes())

    if not host_error:
        _lib.check(L.fl_cg_iterate(op, C.byref(vecs), pre, D.ptr(state), 1, max_iters,
                                   C.byref(mon) if mon is not None else None, D.stream_ptr()),
                   "fl_cg_iterate")
        st = read()
    else:
        it = 0
        st = read()
        while it < max_iters:
            count = min(stride - (it % stride), max_iters - it)
            _lib.check(L.fl_cg_iterate(op, C.byref(vecs), pre, D.ptr(state), it + 1, count, None,
                                       D.stream_ptr()), "fl_cg_iterate")
            st = read()
            done_it = int(st.it)
            if st.diverged_at:
                break
            if done_it % stride == 0 and done_it > it:
                x_now = D.to_host(buf["x"])[:n]
                res = float(buf["res"][done_it].item())
                monitor.observe(done_it, x_now, lambda: res)
            it += count
            if st.done:
                break
    if st.diverged_at:
        raise DivergenceError(f"non-finite iterate at iteration {int(st.diverged_at)}")
    iters = int(st.it)
    if not host_error:
        lv = _lib.LsqrVecs(x=D.ptr(buf["x"]), xbest=D.ptr(buf["xbest"]))
        _lib.check(L.fl_lsqr_monitor_flush(op, C.byref(lv), D.ptr(state), D.stream_ptr()),
                   "fl_lsqr_monitor_flush")
    _lib.check(L.fl_cg_residual(op, C.byref(vecs), D.ptr(buf["out"]), D.stream_ptr()),
               "fl_cg_residual")
    final_res = float(D.to_host(buf["out"])[0])
    x = D.to_host(buf["x"])[:n]
    if not host_error:
        st = read()
        res = D.to_host(buf["res"])
        errs = D.to_host(err_trace) if dev_error else res
        for it in range(1, iters + 1):
            if stride > 1 and it % stride != 0:
                continue
            monitor.records.append((it, float(res[it]), float(errs[it])))
        if st.best_it >= 1:
            monitor.best_error = float(st.best)
            monitor.best_iteration = int(st.best_it)
            monitor.best_iterate = D.to_host(buf["xbest"])[:n].copy()
    return SolveResult(x, iters, final_res, monitor, bool(st.breakdown))
