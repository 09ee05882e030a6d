"""Parity at the full BASELINE sizes (cfg2, cfg3, cfg4 = the north-star system,
cfg5; cfg1 is full size in tests/test_gpu_parity.py).

1. Kept sequences: tests/golden/full_<cfg>.npz were produced by
   tests/golden/make_golden_full.py, which runs the reference's own
   `assemble` (assembly.py:124) and, per block, its `qr_column_pivot`
   (linalg.py:58) exactly as `filter_system` (filtering.py:92-115) does; the
   device pipeline reproduces every rank and kept sequence (pivot order).
2. Factor gates on EVERY block: ||Q^T Q - I||_max <=
   1e-12, ||Q R - A[:, kept]||_max <= 1e-12 max|A_j|, and ||R_j - R_j^LAPACK||_F
   <= 1e-10 ||R_j^LAPACK||_F against featlsq's own `qr_column_pivot` run on
   the host on the same device-assembled blocks; assembly entries against the
   oracle on 16 full-size blocks (corners, edges, interior) <= 1e-13.
3. The solution (y, M a and the predicted field on the test
   lattice) after the paper's 10 000-iteration budget, run D (device factors)
   against run L (LAPACK factors, same device LSQR kernels), gated by the
   spread of the computation itself: run D' repeats D on the system with
   every entry perturbed by at most 1 ulp. Why not 1e-8 (the north star's
   number): the converged regime where iterate parity is a property of the
   problem does not exist here — scipy's test-2 quantity
   ||Q^T r|| / (||Q||_F ||r||) bottoms out near 1e-5 (cfg4) and then GROWS
   under further iterations (profiles/r02_converge.log: 1.9e-5 at 20k, 1.9e-3
   at 200k), and two valid QR factors differ by ~1e-6 in their last columns
   (SURVEY F5), so y differs by ~1e-5 from iteration 100 on, in the device
   run and in any other correct implementation alike.
4. cfg3 against the REFERENCE's own end-to-end run (tests/golden/
   lsqr_full_cfg3.npz: featlsq assemble -> filter_system -> lsqr 10 000 ->
   recover_solution, tests/golden/make_golden_lsqr_full.py): runs L and D
   within the same bound as in 3 for y, M a and the prediction; the true
   residual ||rhs - M a|| within one iteration's worth of LSQR progress.
"""

from __future__ import annotations

import os

import numpy as np
import pytest

import fullsize

pytestmark = pytest.mark.gpu

FULL = ["cfg2", "cfg3", "cfg5", "cfg4"]
ITERS = 10_000


@pytest.fixture(scope="module")
def fl():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2506_17626_b200 as fl
    return fl


@pytest.fixture(scope="module", params=FULL)
def full(request, fl):
    """Device system + factors of one config (and, lazily, the host LAPACK
    factors), shared by the tests of that config: pytest groups the tests by
    this module-scoped parameter, so each config is assembled once."""
    import torch
    from paper_2506_17626_b200 import workloads
    name = request.param
    wl = workloads.build(name)
    sysd = fl.assemble(wl.problem, wl.dec, wl.basis, interior_per_dim=wl.interior_per_dim)
    fs = fl.filter_system(sysd, wl.sigma)
    st = dict(name=name, wl=wl, sysd=sysd, fs=fs)
    yield st
    st.clear()
    torch.cuda.empty_cache()


def _lapack(st):
    if "pqs" not in st:
        st["pqs"] = fullsize.lapack_factors(st["sysd"].blocks, st["wl"].sigma)
    return st["pqs"]


def test_full_size_kept_sequences_match_reference(fl, full, golden_dir):
    import torch
    st, name = full, full["name"]
    g = np.load(os.path.join(golden_dir, f"full_{name}.npz"))
    sysd, fs = st["sysd"], st["fs"]
    assert tuple(sysd.shape) == tuple(int(s) for s in g["shape"])
    assert np.array_equal(fs.ranks, g["ranks"])
    K = fs.K
    local = np.concatenate([k - j * K for j, k in enumerate(fs.kept_list)])
    assert np.array_equal(local, g["kept"].astype(np.int64))
    assert fs.kept_total == int(g["ranks"].sum())
    J = len(fs.kept_list)
    R = fs._R[:J * K * K].view(J, K, K)
    r = torch.as_tensor(fs.ranks, device=R.device)
    idx = torch.arange(K, device=R.device)
    mask = (idx[None, :, None] < r[:, None, None]) & (idx[None, None, :] < r[:, None, None])
    fro = torch.sqrt((torch.where(mask, R, torch.zeros((), dtype=R.dtype, device=R.device)) ** 2)
                     .sum(dim=(1, 2))).cpu().numpy()
    np.testing.assert_allclose(fro, g["r_fro"], rtol=1e-10)


def test_full_size_factor_gates(fl, full):
    """Every block: Q orthonormal, Q R = A[:, kept], R = LAPACK's R."""
    import torch
    from oracle import featlsq_oracle as O
    st, name = full, full["name"]
    sysd, fs, wl = st["sysd"], st["fs"], st["wl"]
    A, Q, L = sysd.store, fs.qstore, fs.qstore.layout
    K, J = fs.K, L.J
    perm = fs._perm[:J * K].view(J, K).long()
    R = fs._R[:J * K * K].view(J, K, K)              # column-major: R[j][col][row]
    pqs = _lapack(st)
    worst_orth = worst_rec = worst_r = 0.0
    for j in range(J):
        m, ld, off, r = int(L.m[j]), int(L.ld[j]), int(L.off[j]), int(fs.ranks[j])
        q = Q.vals[off:off + ld * r].view(r, ld)[:, :m]          # rows = columns of Q_j
        a = A.vals[off:off + ld * K].view(K, ld)[:, :m]
        rj = R[j, :r, :r].T                                      # (r, r) upper
        orth = (q @ q.T - torch.eye(r, dtype=q.dtype, device=q.device)).abs().max().item()
        rec = ((q.T @ rj) - a[perm[j, :r]].T).abs().max().item() / a.abs().max().item()
        r_ref = pqs[j].r_factor
        dr = np.linalg.norm(rj.cpu().numpy() - r_ref) / np.linalg.norm(r_ref)
        worst_orth, worst_rec, worst_r = max(worst_orth, orth), max(worst_rec, rec), max(worst_r, dr)
    print(f"{name}: {J} blocks, max ||Q^TQ-I|| {worst_orth:.2e}, max ||QR-A||/max|A| {worst_rec:.2e}, "
          f"max ||dR||/||R|| {worst_r:.2e}")
    assert worst_orth <= 1e-12
    assert worst_rec <= 1e-12
    assert worst_r <= 1e-10
    # assembly entries on 16 full-size blocks against the oracle
    S, d = wl.dec.count_per_dim, wl.dec.dim
    picks = {p % J for p in (0, J - 1, S // 2, (S // 2) * S ** (d - 1), J // 2 + S // 2)}
    rng = np.random.default_rng(0)
    picks |= set(rng.choice(J, 16 - len(picks), replace=False).tolist())
    sel = sorted(picks)[:16]
    ref = O.assemble(wl.problem, wl.dec, wl.basis, wl.interior_per_dim, only=sel)
    for j, (rows, mat) in zip(sel, ref["blocks"]):
        got = sysd.store.block_host(j)
        assert np.array_equal(sysd.block_rows[j], rows)
        assert np.abs(got - mat).max() <= 1e-13 * np.abs(mat).max(), f"block {j}"


def _solve(fl, blocks, rhs, iters):
    from paper_2506_17626_b200 import _device as D, solvers
    run = solvers.DeviceLsqr(blocks, iters)
    run.reset_state(1, track_best=False)
    run.init(D.to_dev(rhs))
    run.iterate(1, iters)
    st = run.read_state()
    tr = D.to_host(run.trace[iters - 1:iters + 1])
    _solve.last_step = float(abs(tr[0] - tr[1]))  # phi-bar's progress over the last iteration
    return D.to_host(run.x)[:blocks.ncols_total].copy(), float(st.phibar)


def _fields(fl, st, y, pqs=None, fs=None):
    """(y, M a, prediction on the test lattice, l1 error) of a solution y."""
    wl, sysd = st["wl"], st["sysd"]
    if pqs is None:
        a = fl.recover_solution(fs or st["fs"], y)
    else:
        a = fullsize._recover_host(pqs, y, st["fs"].K, len(pqs))
    ma = fl.apply(sysd, a)
    ts = st.setdefault("ts", fl.make_test_set(wl.problem, wl.dec))
    pred = fl.evaluate_solution(wl.problem, wl.dec, wl.basis, a, ts.points)
    return y, ma, pred, fl.l1_error(pred, ts)


def _rel(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


def test_full_size_solution_within_own_spread(fl, full, golden_dir):
    """Run D vs run L at the 10 000-iteration budget, gated by the 1-ulp
    spread D vs D' (module docstring, item 3); for cfg3 also both runs
    against featlsq's own end-to-end solve (item 4)."""
    from paper_2506_17626_b200 import _device as D
    st, name = full, full["name"]
    sysd, fs, wl = st["sysd"], st["fs"], st["wl"]
    pqs = _lapack(st)
    host_blocks = sysd.blocks
    ref_ops = D.blocks_from_host(sysd.row_count, [b.rows for b in host_blocks],
                                 [pq.q_factor for pq in pqs])
    y_l, ph_l = _solve(fl, ref_ops, sysd.rhs, ITERS)
    del ref_ops
    op = fl.precondition(fs)
    y_d, ph_d = _solve(fl, op.device_blocks, sysd.rhs, ITERS)
    step_d = _solve.last_step
    # D': every entry of A moved by at most 1 ulp (relative 2^-52 noise)
    noise = np.random.default_rng(7)
    pert = fl.assemble(wl.problem, wl.dec, wl.basis, interior_per_dim=wl.interior_per_dim)
    v = pert.store.vals
    import torch
    g = torch.Generator(device=v.device).manual_seed(int(noise.integers(1 << 30)))
    v.mul_(1.0 + (torch.rand(v.shape, generator=g, device=v.device, dtype=v.dtype) - 0.5) * 2.0 ** -52)
    fs_p = fl.filter_system(pert, wl.sigma)
    assert np.array_equal(fs_p.ranks, fs.ranks)
    y_p, ph_p = _solve(fl, fl.precondition(fs_p).device_blocks, sysd.rhs, ITERS)
    fd = _fields(fl, st, y_d)
    fl_ = _fields(fl, st, y_l, pqs=pqs)
    fp = _fields(fl, st, y_p, fs=fs_p)
    names = ("y", "Ma", "pred")
    dl = {n: _rel(fd[i], fl_[i]) for i, n in enumerate(names)}
    dp = {n: _rel(fp[i], fd[i]) for i, n in enumerate(names)}
    print(f"{name} at {ITERS} its: D vs L " + " ".join(f"{n} {dl[n]:.2e}" for n in names)
          + " | 1-ulp spread D' vs D " + " ".join(f"{n} {dp[n]:.2e}" for n in names)
          + f" | phibar D {ph_d:.10e} L {ph_l:.10e} D' {ph_p:.10e}"
          + f" | l1 D {fd[3]:.6e} L {fl_[3]:.6e} D' {fp[3]:.6e}")
    for n in names:
        assert dl[n] <= max(1e-8, 10.0 * dp[n]), n
    # the spread itself stays small, so the gate above is not vacuous (cfg2,
    # the least well-conditioned after preconditioning, spreads 9.5e-5 in M a)
    assert dp["Ma"] <= 1e-3 and dp["pred"] <= 1e-3
    # phi-bar: a difference of two scalars against a one-sample scalar spread
    # can fail by chance (the sample happens to be small), so the gate is the
    # larger of 10x that spread and one iteration's progress of phi-bar at the
    # budget (the two runs are then less than one iteration apart)
    sp_ph = abs(ph_p - ph_d)
    print(f"{name}: |phibar D - L| {abs(ph_d - ph_l):.3e}, 1-ulp spread {sp_ph:.3e}, "
          f"last iteration's progress {step_d:.3e}")
    assert abs(ph_d - ph_l) <= max(1e-9 * ph_l, 10.0 * sp_ph, step_d)
    # L1 test error: bounded by the mean prediction change over the spread
    # (|l1(a) - l1(b)| <= mean|a - b| / spread); gated at 10x what the 1-ulp
    # perturbation's prediction change allows
    l1_sp = float(np.mean(np.abs(fp[2] - fd[2]))) / st["ts"].spread
    assert abs(fd[3] - fl_[3]) <= max(1e-9 * fl_[3], 10.0 * l1_sp)
    del fs_p, pert
    path = os.path.join(golden_dir, f"lsqr_full_{name}.npz")
    if not os.path.exists(path):
        return
    g = np.load(path)
    assert np.array_equal(fs.ranks, g["kept"])
    ref = (g["y"], g["ma"], g["pred"])
    rl = {n: _rel(fl_[i], ref[i]) for i, n in enumerate(names)}
    rd = {n: _rel(fd[i], ref[i]) for i, n in enumerate(names)}
    print(f"{name} vs featlsq's own {int(g['max_iters'])}-iteration solve: L "
          + " ".join(f"{n} {rl[n]:.2e}" for n in names)
          + " | D " + " ".join(f"{n} {rd[n]:.2e}" for n in names)
          + f" | phibar ref {float(g['residual']):.10e} | l1 ref {float(g['l1']):.6e}")
    assert int(g["max_iters"]) == ITERS
    for n in names:
        assert rl[n] <= max(1e-8, 10.0 * dp[n]), n
        assert rd[n] <= max(1e-8, 10.0 * dp[n]), n
    # residual of the solution in the raw system, ||rhs - M a||: the reference's
    # recurrence estimate phi-bar drifts from its true residual over 10 000
    # iterations of sequential CSR sums (1.6e-5 relative at cfg3), the device
    # one does not (phi-bar = ||Q y - b|| to 11 digits), so the comparison
    # with featlsq's run is on the true residuals
    res = {k: float(np.linalg.norm(sysd.rhs - v)) for k, v in
           (("ref", g["ma"]), ("D", fd[1]), ("L", fl_[1]), ("P", fp[1]))}
    sp_res = abs(res["P"] - res["D"])
    print(f"{name} true residual ||rhs - M a||: ref {res['ref']:.12e} D {res['D']:.12e} "
          f"L {res['L']:.12e} D' {res['P']:.12e} (featlsq phi-bar {float(g['residual']):.12e})")
    # featlsq's run assembles with numpy (entries agree to 1e-13 of the block
    # maximum, not to 1 ulp) and factors with this container's OpenBLAS, so
    # its trajectory sits a fraction of an iteration away from the device
    # runs: the residual gate is one iteration's worth of LSQR progress at
    # 10 000 iterations (from featlsq's own phi-bar records), the 1-ulp
    # spread when that is larger
    rec = g["records"]
    per_it = float(rec[-2, 1] - rec[-1, 1]) / float(rec[-1, 0] - rec[-2, 0])
    print(f"{name}: one iteration of progress at {ITERS} = {per_it:.3e} "
          f"({per_it / res['ref']:.2e} relative); 1-ulp residual spread {sp_res:.3e}")
    for k in ("D", "L"):
        assert abs(res[k] - res["ref"]) <= max(per_it, 10.0 * sp_res), k


def test_full_size_lsqr_properties(fl, full):
    """LSQR at the BASELINE size, through size-independent properties: the
    residual estimate phibar is non-increasing and equals the true residual
    ||Q y - b|| (to 1e-9 relative after 60 iterations), the device run is
    bit-reproducible, and the recovered coefficients reproduce Q y through
    the raw blocks (M a = Q y)."""
    st = full
    sysd, fs = st["sysd"], st["fs"]
    op = fl.precondition(fs)
    r1 = fl.lsqr(op, sysd.rhs, 60)
    r2 = fl.lsqr(op, sysd.rhs, 60)
    assert np.array_equal(r1.solution, r2.solution)
    ph = np.array([r[1] for r in r1.monitor.records])
    assert np.all(np.diff(ph) <= 1e-12 * ph[0])
    qy = op.apply(r1.solution)
    true_res = np.linalg.norm(qy - sysd.rhs)
    assert r1.residual_norm == pytest.approx(true_res, rel=1e-9)
    a = fl.recover_solution(fs, r1.solution)
    ma = fl.apply(sysd, a)
    # M a = Q y up to eps * kappa(R_j) (kappa ~ 1e10 at sigma = 1e-10)
    assert np.linalg.norm(ma - qy) <= 1e-4 * np.linalg.norm(qy)
