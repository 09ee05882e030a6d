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


@pytest.mark.parametrize("K", [128, 256])
def test_qform_fused_matches_numpy(dev, K):
    """K2c fused (qform.cu): C_j <- H_0 .. H_{K-1} [Q1_j; 0] as 64-wide compact-WY
    blocks in reverse, against numpy block by block (incl. m_j < K and
    partial ranks)."""
    torch, D, _lib = dev
    rng = np.random.default_rng(11 + K)
    ms = [K + 37, 3 * K, K, K - 20, 2 * K + 5]
    ranks = [K, K - 5, 70, K - 20, 1]
    nb = K // 64
    vbuf, voff, vld, vmats = _blocks(ms, K, rng=rng)
    # C = [Q1; 0]: rows >= K (and >= rank columns' rows past m) zero
    cbuf, coff, cld, cmats = _blocks(ms, K, rng=rng)
    for j, m in enumerate(ms):
        cmats[j][K:] = 0.0
        blk = cbuf[coff[j]:coff[j] + cld[j] * K].reshape(K, cld[j])
        blk[:, K:] = 0.0
    T = np.stack([np.stack([np.triu(rng.standard_normal((64, 64))) * 0.1 for _ in range(nb)]) for _ in ms])
    d = {k: D.to_dev(v) for k, v in dict(
        V=vbuf, voff=voff, vld=vld, C=cbuf, coff=coff, cld=cld, m=np.array(ms, np.int32),
        rank=np.array(ranks, np.int32),
        T=np.ascontiguousarray(T.transpose(0, 1, 3, 2)).ravel()).items()}   # column-major per block
    _lib.check(_lib.lib().fl_dev_qform(
        D.ptr(d["V"]), D.ptr(d["voff"]), D.ptr(d["vld"]), D.ptr(d["m"]), D.ptr(d["C"]),
        D.ptr(d["coff"]), D.ptr(d["cld"]), D.ptr(d["rank"]), D.ptr(d["T"]), K, len(ms),
        D.stream_ptr()), "qform")
    out = d["C"].cpu().numpy()
    for j, (m, r) in enumerate(zip(ms, ranks)):
        V = vmats[j].copy()
        for c in range(K):  # entries on and above the diagonal are not the reflector's
            V[:min(c, m), c] = 0.0
            if c < m:
                V[c, c] = 1.0
        want = cmats[j].copy()
        for b in range(nb - 1, -1, -1):
            r0 = 64 * b
            if r0 >= m:
                continue
            Vb = V[r0:, r0:r0 + 64]
            want[r0:, :r] -= Vb @ (T[j, b] @ (Vb.T @ want[r0:, :r]))
        got = out[coff[j]:coff[j] + cld[j] * K].reshape(K, cld[j])[:, :m].T
        scale = max(1.0, np.abs(want).max())
        assert np.abs(got[:, :r] - want[:, :r]).max() <= 1e-12 * scale, j
        # columns past the rank are left as they were
        assert np.array_equal(got[:, r:], cmats[j][:, r:]), j
