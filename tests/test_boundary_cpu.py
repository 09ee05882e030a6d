"""CPU-side checks of the drop-in boundary: the C-ABI library loads and
exports every symbol include/featlsq_b200.h declares, the ctypes structs
match the header layout, and the host logic (layouts, gather maps, row sets,
workloads) is right. No compute calls (there is no GPU here)."""

import ctypes as C
import os
import re

import numpy as np
import pytest

from paper_2506_17626_b200 import _lib, workloads
from paper_2506_17626_b200.domains import decompose, support_runs

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "featlsq_b200.h")


def _declared():
    src = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:int|int32_t|int64_t|const char\*)\s+(fl_\w+)\(", src, re.M)))


def test_library_exports_every_declared_symbol():
    if not os.path.exists(_lib.LIB_PATH):
        from paper_2506_17626_b200 import build
        build.build()
    L = _lib.lib()
    declared = _declared()
    assert set(declared) == set(_lib.EXPORTED)
    for name in declared:
        assert hasattr(L, name), name
    assert b"sm_100a" in L.fl_version()


def _struct_fields(name):
    src = open(HEADER).read()
    body = re.search(r"typedef struct %s \{(.*?)\} %s;" % (name, name), src, re.S).group(1)
    body = re.sub(r"/\*.*?\*/", "", body, flags=re.S)
    names = []
    for decl in body.split(";"):
        decl = decl.strip()
        if not decl:
            continue
        names += [re.sub(r"\[.*\]", "", piece.replace("*", " ").split()[-1])
                  for piece in decl.split(",")]
    return names


@pytest.mark.parametrize("cname,pyname", [("fl_blockop", "BlockOp"),
                                          ("fl_assembly_desc", "AssemblyDesc"),
                                          ("fl_lsqr_state", "LsqrState"),
                                          ("fl_lsqr_vecs", "LsqrVecs"),
                                          ("fl_test_monitor", "TestMonitor"),
                                          ("fl_cg_vecs", "CgVecs"),
                                          ("fl_block_precond", "BlockPrecond")])
def test_ctypes_structs_match_header(cname, pyname):
    py = getattr(_lib, pyname)
    assert [f[0] for f in py._fields_] == _struct_fields(cname)


def test_block_layout_gather_map():
    from paper_2506_17626_b200._device import BlockLayout
    rows = [np.array([0, 1, 2, 5]), np.array([2, 3, 5]), np.array([4, 5, 0])]
    L = BlockLayout(6, 3, rows)
    assert L.partial_len == 10
    assert np.all(L.ld % 16 == 0) and np.all(L.ld >= L.m)
    for g in range(6):
        srcs = L.gsrc[L.gptr[g]:L.gptr[g + 1]]
        assert np.all(L.rows[srcs] == g)
        assert np.all(np.diff(srcs) > 0)  # fixed increasing block order
    assert L.gptr[-1] == 10


def test_support_runs_match_strict_support():
    dec = decompose(workloads.build_small("cfg3").dec.domain, 5, 2.0)
    axes = (np.linspace(0, 1, 37), np.linspace(0, 1, 37))
    runs = support_runs(dec, axes)
    for i in range(2):
        for s in range(5):
            idx = np.nonzero(np.abs(axes[i] - dec.centers[i, s]) < dec.half_widths[i])[0]
            lo, cnt = runs[i, s]
            assert cnt == idx.size and (cnt == 0 or lo == idx[0])


@pytest.mark.parametrize("name", ["cfg1", "cfg2", "cfg3", "cfg4", "cfg5"])
def test_workloads_match_baseline_shapes(name):
    """Full-size shapes from SURVEY.md §8(d) (host arithmetic only)."""
    wl = workloads.build(name)
    dec, basis = wl.dec, wl.basis
    expect = {"cfg1": (2002, 1280), "cfg2": (40002, 25600), "cfg3": (161600, 65536),
              "cfg4": (643200, 524288), "cfg5": (282624, 262144)}[name]
    n_int = wl.interior_per_dim ** dec.dim
    n_con = sum(np.atleast_2d(c.points).shape[0] for c in wl.problem.constraints)
    assert (n_int + n_con, basis.column_count) == expect
    assert basis.weights[0].shape == (dec.subdomain_count, basis.feature_count, dec.dim)


def test_host_row_sets_match_oracle():
    """The host row-set construction used for the device layout equals the
    oracle's (reference assembly.py:199-231) on a small 2-D case."""
    from oracle import featlsq_oracle as O
    from paper_2506_17626_b200.assembly import _layout_inputs
    wl = workloads.build_small("cfg3")
    counts, axes = O.lattice_axes(wl.problem, wl.dec, wl.basis, wl.interior_per_dim)
    out = _layout_inputs(wl.problem, wl.dec, wl.basis, axes, counts)
    rows_per_block = out[-1]
    ref = O.assemble(wl.problem, wl.dec, wl.basis, wl.interior_per_dim)
    for got, (want, _) in zip(rows_per_block, ref["blocks"]):
        assert np.array_equal(got, want)


def test_product_path_refuses_without_gpu():
    torch = pytest.importorskip("torch")
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    import paper_2506_17626_b200 as fl
    wl = workloads.build("cfg1")
    with pytest.raises(fl.DeviceError):
        fl.assemble(wl.problem, wl.dec, wl.basis, interior_per_dim=wl.interior_per_dim)


def test_rrqr_route_respects_shared_memory_bounds():
    from paper_2506_17626_b200._device import BlockLayout
    from paper_2506_17626_b200.filtering import BLOCKED_MAX_K, BLOCKED_MAX_ROWS, rrqr_route

    def layout(K, m):
        return BlockLayout(m, K, [np.arange(m), np.arange(m)])
    assert rrqr_route(layout(512, 2700)) == "blocked"
    assert rrqr_route(layout(64, 300)) == "direct"                 # K < 128
    assert rrqr_route(layout(200, 900)) == "direct"                # K % 32 != 0
    assert rrqr_route(layout(512, 400)) == "direct"                # wide blocks
    assert rrqr_route(layout(BLOCKED_MAX_K + 32, 2000)) == "direct"
    # no row bound on route R (taller blocks: inner panels factored in place);
    # narrow blocks go there once the direct kernel's reflector no longer fits
    assert rrqr_route(layout(256, BLOCKED_MAX_ROWS + 16)) == "blocked"
    assert rrqr_route(layout(64, 20000)) == "direct"
    assert rrqr_route(layout(64, 40000)) == "blocked"
    assert rrqr_route(layout(72, 40000)) == "direct"               # neither route: CapExceededError
