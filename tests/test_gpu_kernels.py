"""Kernel-level checks of the internal building blocks against plain numpy
fp64 references of the same operation (gpu)."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def dev():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2506_17626_b200 import _device as D, _lib
    return torch, D, _lib


def _blocks(ms, ncols, ld_align=16, rng=None):
    lds = [max((m + ld_align - 1) // ld_align * ld_align, ld_align) for m in ms]
    offs = np.concatenate([[0], np.cumsum([ld * ncols for ld in lds])[:-1]]).astype(np.int64)
    buf = np.zeros(sum(ld * ncols for ld in lds))
    mats = []
    for m, ld, off in zip(ms, lds, offs):
        a = rng.standard_normal((m, ncols))
        blk = np.zeros((ncols, ld))
        blk[:, :m] = a.T
        buf[off:off + ld * ncols] = blk.ravel()
        mats.append(a)
    return buf, offs, np.array(lds, np.int32), mats


@pytest.mark.parametrize("NB", [32, 64])
@pytest.mark.parametrize("transT", [0, 1])
@pytest.mark.parametrize("row0", [0, 32])
def test_wy_apply_matches_numpy(dev, transT, row0, NB):
    torch, D, _lib = dev
    rng = np.random.default_rng(3 + transT + row0 + NB)
    ms = [row0 + NB + 8, row0 + 257, row0 + NB, row0 + 1000]
    ncol = 150
    vbuf, voff, vld, vmats = _blocks(ms, NB, rng=rng)
    cbuf, coff, cld, cmats = _blocks(ms, ncol, rng=rng)
    T = np.stack([np.triu(rng.standard_normal((NB, NB))) for _ in ms])
    tiles = np.array([(j, c0) for j in range(len(ms)) for c0 in range(0, ncol, 64)], np.int32)
    d = {k: D.to_dev(v) for k, v in dict(
        V=vbuf, voff=voff, vld=vld, C=cbuf, coff=coff, cld=cld, m=np.array(ms, np.int32),
        T=np.ascontiguousarray(T.transpose(0, 2, 1)).ravel(),   # column-major per block
        ncols=np.full(len(ms), ncol, np.int32), tiles=tiles.ravel()).items()}
    _lib.check(_lib.lib().fl_dev_wy_apply(
        D.ptr(d["V"]), D.ptr(d["voff"]), D.ptr(d["vld"]), D.ptr(d["C"]), D.ptr(d["coff"]),
        D.ptr(d["cld"]), D.ptr(d["m"]), D.ptr(d["T"]), NB * NB, NB, row0, transT, D.ptr(d["ncols"]),
        D.ptr(d["tiles"]), len(tiles), D.stream_ptr()), "wy")
    out = d["C"].cpu().numpy()
    for j, m in enumerate(ms):
        V = vmats[j][row0:].copy()
        V[:NB] = np.tril(V[:NB], -1) + np.eye(NB)
        Tj = T[j].T if transT else T[j]
        want = cmats[j].copy()
        want[row0:] -= V @ (Tj @ (V.T @ want[row0:]))
        got = out[coff[j]:coff[j] + cld[j] * ncol].reshape(ncol, cld[j])[:, :m].T
        assert np.abs(got - want).max() <= 1e-12 * max(1.0, np.abs(want).max()), j
        # padding rows untouched (zero)
        pad = out[coff[j]:coff[j] + cld[j] * ncol].reshape(ncol, cld[j])[:, m:]
        assert np.all(pad == 0.0)
