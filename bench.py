"""Benchmark of the B200-native featlsq hot path (BASELINE.json metric:
"RRQR filter+precond sec & GFLOP/s; LSQR matvec GB/s vs HBM roofline; solve
sec").

One step = one full solve of the workload: K1 assembly -> K2 truncated RRQR
(filter + preconditioner factors) -> K4 device LSQR with a fixed budget of
--lsqr-iters iterations (the reference has no stopping rule) -> K5 recovery.
Default workload: cfg4, the north-star 2D 32x32-subdomain Helmholtz system
(643 200 x 524 288, M = 512), synthetic inputs per SURVEY.md §8(d).

`value` (solves/s, whole job) is timed with CUDA events on the launching
stream with the inputs already in HBM; `e2e` is the same metric through the
public Python API (`assemble` / `filter_system` / `precondition` / `lsqr` /
`recover_solution`) with host inputs and host outputs, copies included
(warm: the lattice layout cache is hit; `e2e.cold_ms` is one call with it
empty). `per_config` times one solve of every BASELINE config (cfg1..cfg5)
per stage; `paper_protocol` is one cfg4 solve at the paper's 10 000 LSQR
iterations.

`--impl reference` times featlsq itself (the reference package, installed
into baseline/_ref) on the host cores: its real `assemble`, `filter_system`,
`precondition`, `lsqr` and `recover_solution` on a stratified sample of the
workload's blocks (corner / edge / interior strata; the global lattice,
coverage check and right-hand side are built in full), extrapolated per
stratum with a work model (assembly ~ m_j, RRQR ~ m_j K^2, LSQR and CSR
build ~ nnz(Q)); each step draws a new sample, and the spread of the steps'
estimates is reported as the sampling error.

Multi-GPU: replicas (each rank solves its own seed of the workload; the
north star pins one GPU per solve), timed as the
max over ranks.
"""

from __future__ import annotations

import argparse
import json
import os
import platform
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "RRQR filter+precond sec & GFLOP/s; LSQR matvec GB/s vs HBM roofline; solve sec"
UNIT = "solves/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="product", choices=["product", "reference"])
    ap.add_argument("--config", default="cfg4")
    ap.add_argument("--lsqr-iters", type=int, default=1000)
    ap.add_argument("--e2e-steps", type=int, default=2)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-configs", action="store_true", help="skip the per-config table")
    ap.add_argument("--no-paper", action="store_true", help="skip the 10 000-iteration solve")
    ap.add_argument("--cpu-per-stratum", type=int, default=4,
                    help="reference sample: blocks per corner/edge/interior stratum")
    return ap.parse_args()


# ---------------------------------------------------------------- helpers
def peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        with open(path) as fh:
            p = json.load(fh)
        return float(p["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


class Clocks:
    """nvidia-smi sampler during the timed region (B200_PROFILING.md recipe)."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.path = None

    def start(self):
        try:
            fd, self.path = tempfile.mkstemp(suffix=".csv")
            os.close(fd)
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except Exception:  # noqa: BLE001
            self.proc = None

    def stop(self):
        if self.proc is None:
            return None
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:  # noqa: BLE001
            self.proc.kill()
        rows = []
        for line in open(self.path):
            parts = [x.strip() for x in line.split(",")]
            if len(parts) >= 9:
                rows.append(parts)
        os.unlink(self.path)
        if not rows:
            return None
        sm = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({n for r in rows for n, v in zip(names, r[5:9]) if v == "Active"})
        loaded = sorted(sm)[len(sm) // 2:] if sm else []
        return {"sm_mhz": float(np.median(loaded)) if loaded else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(rows)}


def fp64_peak(torch, D, _lib):
    """Measured FP64 peak (TFLOP/s): DFMA and DMMA probes, best of 3."""
    out = torch.zeros(1, dtype=torch.float64, device="cuda")
    res = {}
    grid, iters = 148 * 8, 4096
    for mode, name in ((0, "dfma"), (1, "dmma")):
        best = 0.0
        for _ in range(4):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            _lib.check(_lib.lib().fl_probe_fp64(mode, grid, iters, D.ptr(out), D.stream_ptr()),
                       "probe")
            e1.record()
            torch.cuda.synchronize()
            flops = grid * 256 * iters * 16 if mode == 0 else grid * 8 * iters * 4 * 512
            best = max(best, flops / (e0.elapsed_time(e1) * 1e-3) / 1e12)
        res[name] = round(best, 2)
    return res


def read_peak(torch, D, _lib):
    """Measured HBM streaming-read ceiling (GB/s), 4 GiB buffer, best of 5."""
    n = 1 << 29
    buf = torch.zeros(n, dtype=torch.float64, device="cuda")
    out = torch.zeros(1, dtype=torch.float64, device="cuda")
    best = 0.0
    for _ in range(6):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        _lib.check(_lib.lib().fl_probe_read(D.ptr(buf), n, D.ptr(out), D.stream_ptr()), "probe")
        e1.record()
        torch.cuda.synchronize()
        best = max(best, 8.0 * n / (e0.elapsed_time(e1) * 1e-3) / 1e9)
    del buf
    return round(best, 1)


# ---------------------------------------------------------------- work counts
def launches_per_step(fs, iters):
    """Kernels of this library launched per solve (rrqr_blocked.cu / qop.cu /
    lsqr_fused.cu launch sequences)."""
    from paper_2506_17626_b200.filtering import rrqr_route
    K = fs.K
    if rrqr_route(fs.qstore.layout) == "blocked":
        npan = K // 32
        if K % 64 == 0:
            q = K // 64
            k2a = 4 * q + (q - 1)            # panel, wy32, panel, combine_t, wy64
            k2c = 1                          # qform.cu: one fused sweep
        else:
            k2a = npan + (npan - 1)
            k2c = npan
        # zero_pad, K2a, extract, qrcp, clamp, build_t, init_q1_r, Q1, init_qhat, K2c, mark_nonfinite
        rrqr = 1 + k2a + 5 + npan + 1 + k2c + 1
    else:
        rrqr = 1
    return 1 + rrqr + 2 + 2 * iters + 1      # assemble, rrqr, lsqr init, iterations, recover


def rrqr_flops(m, K, r):
    """F_alg (truncated QRCP + thin Q + initial norms) and
    F_ref (full dgeqp3 + dorgqr, what the reference executes), plus F_exec,
    what route R executes (DESIGN.md §3 K2): unpivoted QR of A_j, truncated
    QRCP of R0 (gemv + block updates), Q1 formation, Q0 [Q1; 0]."""
    m, r = m.astype(np.float64), r.astype(np.float64)
    f_alg = (4 * m * K * r - 2 * (m + K) * r ** 2 + (4 / 3) * r ** 3
             + 2 * m * r ** 2 - (2 / 3) * r ** 3 + 2 * m * K)
    kk = np.minimum(m, K)
    f_ref = 4 * m * K * kk - (4 / 3) * kk ** 3
    f_exec = ((2 * m * K ** 2 - (2 / 3) * K ** 3)                   # K2a
              + (4 / 3) * (K ** 3 - (K - r) ** 3)                    # K2b
              + (2 * K * r ** 2 - (2 / 3) * r ** 3)                  # Q1
              + 4 * r * (m * K - K ** 2 / 2))                        # K2c
    return float(f_alg.sum()), float(f_ref.sum()), float(f_exec.sum())


# ---------------------------------------------------------------- product arm
class Pipeline:
    """The device-resident solve of one workload (host preparation outside
    the timed region): K1 -> K2 -> K4 (iters) -> K5, with CUDA events
    between the stages."""

    def __init__(self, wl, iters):
        import paper_2506_17626_b200 as fl
        from paper_2506_17626_b200 import _device as D
        from paper_2506_17626_b200.assembly import AssemblyPlan
        self.fl, self.wl, self.iters = fl, wl, iters
        self.plan = AssemblyPlan(wl.problem, wl.dec, wl.basis, wl.interior_per_dim)
        self.rhs_dev = D.to_dev(self.plan.rhs)
        self.store = self.plan.new_store()
        self.system = self.plan.system(self.store)
        self.run = None
        self.fs = None

    def step(self, ev):
        from paper_2506_17626_b200.filtering import recover_solution_device
        from paper_2506_17626_b200.solvers import DeviceLsqr
        ev[0].record()
        self.plan.launch(self.store)
        ev[1].record()
        fs = self.fl.filter_system(self.system, self.wl.sigma)
        ev[2].record()
        op = self.fl.precondition(fs)
        if self.run is None or self.run.blocks is not op.device_blocks:
            self.run = DeviceLsqr(op.device_blocks, self.iters)
        self.run.reset_state(1, track_best=True)
        self.run.init(self.rhs_dev)
        ev[3].record()
        self.run.iterate(1, self.iters)
        ev[4].record()
        coeffs, _ = recover_solution_device(fs, self.run.x)
        ev[5].record()
        self.fs = fs
        return coeffs

    @staticmethod
    def events():
        import torch
        return [torch.cuda.Event(enable_timing=True) for _ in range(6)]

    def work(self):
        """Algorithmic work of one solve."""
        fs = self.fs
        L = fs.qstore.layout
        m = L.m.astype(np.int64)
        nnz_q = int(np.sum(m * fs.ranks))
        nnz_a = int(m.sum()) * L.K
        f_alg, f_ref, f_exec = rrqr_flops(m, L.K, fs.ranks)
        # compulsory bytes of one fused iteration: Q read once (the kernel reuses
        # each staged column tile for Q^T u and Q v'), u/partials, 6 y-space vectors
        bytes_it = 8.0 * (nnz_q + 2 * L.partial_len + 2 * L.nrows + 6 * fs.kept_total)
        # SURVEY.md §8(d) per-iteration bytes assume two passes over Q (Q v, Q^T u)
        bytes_survey = 8.0 * (2 * nnz_q + 2 * L.nrows + 6 * fs.kept_total)
        return dict(L=L, nnz_q=nnz_q, nnz_a=nnz_a, f_alg=f_alg, f_ref=f_ref, f_exec=f_exec,
                    bytes_it=bytes_it, bytes_survey=bytes_survey)


def stage_times(evs):
    def avg(a, b):
        return float(np.mean([e[a].elapsed_time(e[b]) for e in evs])) / 1e3
    return dict(assemble=avg(0, 1), rrqr=avg(1, 2), init=avg(2, 3), lsqr=avg(3, 4),
                recover=avg(4, 5))


def stage_table(w, t, iters, hbm, fp64_tf, latency_bound=False):
    """Per-stage time, throughput and roofline fractions of one config."""
    t_it = t["lsqr"] / iters
    solve = t["assemble"] + t["rrqr"] + t["init"] + t["lsqr"] + t["recover"]
    out = {"assemble_ms": round(t["assemble"] * 1e3, 3), "rrqr_ms": round(t["rrqr"] * 1e3, 3),
           "lsqr_ms_per_iter": round(t_it * 1e3, 4), "recover_ms": round(t["recover"] * 1e3, 3),
           "solve_s": round(solve, 4), "rows": w["L"].nrows, "cols": int(w["L"].J * w["L"].K)}
    if latency_bound:
        out["note"] = "latency-bound (blocks and Q fit in L2): time only"
        return out
    gbs_a = 8 * w["nnz_a"] / t["assemble"] / 1e9
    gbs_q = w["bytes_it"] / t_it / 1e9
    gf = w["f_alg"] / t["rrqr"] / 1e9
    out.update({
        "assemble_GB/s": round(gbs_a, 1), "assemble_frac_hbm": round(gbs_a / hbm, 4),
        "rrqr_GFLOP/s_alg": round(gf, 1), "rrqr_frac_fp64": round(gf / 1e3 / fp64_tf, 4),
        "rrqr_F_alg_TF": round(w["f_alg"] / 1e12, 4),
        "lsqr_GB/s": round(gbs_q, 1), "lsqr_frac_hbm": round(gbs_q / hbm, 4)})
    return out


def product(args, rank, world, local_rank):
    import torch
    import paper_2506_17626_b200 as fl
    from paper_2506_17626_b200 import _device as D, _lib, assembly, workloads
    from paper_2506_17626_b200.replicas import (barrier, max_over_ranks, replica_seed,
                                                 whole_job_rate)
    torch.cuda.set_device(local_rank)
    wl = workloads.build(args.config, seed=replica_seed(rank))
    iters = args.lsqr_iters
    pipe = Pipeline(wl, iters)

    for _ in range(args.warmup):
        pipe.step(pipe.events())
    torch.cuda.synchronize()
    barrier()
    clocks = Clocks(local_rank)
    clocks.start()
    torch.cuda.synchronize()
    t_start, t_end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    evs = [pipe.events() for _ in range(args.steps)]
    t_start.record()
    for k in range(args.steps):
        pipe.step(evs[k])
    t_end.record()
    torch.cuda.synchronize()
    clk = clocks.stop()
    elapsed = max_over_ranks(t_start.elapsed_time(t_end) / 1e3)
    barrier()

    t = stage_times(evs)
    t_asm, t_rrqr, t_init, t_lsqr, t_rec = t["assemble"], t["rrqr"], t["init"], t["lsqr"], t["recover"]
    fs = pipe.fs
    w = pipe.work()
    L, nnz_q, nnz_a = w["L"], w["nnz_q"], w["nnz_a"]
    f_alg, f_ref, f_exec = w["f_alg"], w["f_ref"], w["f_exec"]
    bytes_it, bytes_survey = w["bytes_it"], w["bytes_survey"]
    t_it = t_lsqr / iters
    hbm, hbm_src = peaks()
    fp64 = fp64_peak(torch, D, _lib)
    read_gbs = read_peak(torch, D, _lib)
    fp64_peak_tf = max(fp64.values())
    st = pipe.run.read_state()
    stage_t = {"assemble": t_asm, "rrqr": t_rrqr, "lsqr": t_lsqr + t_init, "recover": t_rec}
    dominant = max(stage_t, key=stage_t.get)
    step_s = elapsed / args.steps
    traffic = asm_flops = None
    tpath = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tpath):
        tj = json.load(open(tpath)).get(args.config, {})
        traffic = tj.get("lsqr_bytes_per_iter")
        asm_flops = tj.get("assemble_fp64_flops")
    out = {
        "metric": METRIC, "value": round(whole_job_rate(world, 1, step_s), 6), "unit": UNIT,
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(step_s * 1e3, 3), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (SURVEY.md §8(d) inputs, seeded)",
        "config": config_of(args, wl, iters, world, int(L.nrows)),
        "workload_stats": {"kept": int(fs.kept_total), "Q_GB": round(nnz_q * 8 / 1e9, 2),
                           "A_store_GB": round(nnz_a * 8 / 1e9, 2)},
        "roofline": {"bound": "hbm", "kernel": "LSQR iteration (fused_kernel + row_kernel)",
                     "achieved": round(bytes_it / t_it / 1e9, 1), "peak": hbm, "unit": "GB/s",
                     "frac": round(bytes_it / t_it / 1e9 / hbm, 4),
                     "traffic": traffic, "peak_source": hbm_src,
                     # the kernel is read-dominated; the copy peak counts read + write
                     "read_peak_measured": read_gbs,
                     "frac_of_read_peak": round(bytes_it / t_it / 1e9 / read_gbs, 4),
                     "algorithmic_bytes_per_launch": bytes_it, "dominant_stage": dominant},
        "stages": {
            "assemble": {"ms": round(t_asm * 1e3, 3), "GB/s": round(8 * nnz_a / t_asm / 1e9, 1),
                         "frac_hbm": round(8 * nnz_a / t_asm / 1e9 / hbm, 4),
                         **({"TF/s_fp64": round(asm_flops / t_asm / 1e12, 2),
                             "frac_fp64_dfma_peak": round(asm_flops / t_asm / 1e12 / fp64["dfma"], 4),
                             "fp64_flops_source": "ncu SASS counts, profiles/traffic.json"}
                            if asm_flops else {})},
            "rrqr_filter_precond": {"ms": round(t_rrqr * 1e3, 3),
                                    "GFLOP/s_alg": round(f_alg / t_rrqr / 1e9, 1),
                                    "GFLOP/s_ref": round(f_ref / t_rrqr / 1e9, 1),
                                    "F_alg_TF": round(f_alg / 1e12, 4),
                                    "frac_fp64_peak": round(f_alg / t_rrqr / 1e12 / fp64_peak_tf, 4),
                                    "F_exec_TF": round(f_exec / 1e12, 4),
                                    "GFLOP/s_exec": round(f_exec / t_rrqr / 1e9, 1),
                                    "frac_fp64_peak_exec": round(f_exec / t_rrqr / 1e12 / fp64_peak_tf, 4),
                                    "fp64_peak_TF_measured": fp64},
            "lsqr": {"ms_per_iter": round(t_it * 1e3, 4), "GB/s": round(bytes_it / t_it / 1e9, 1),
                     "frac_hbm": round(bytes_it / t_it / 1e9 / hbm, 4),
                     "GB/s_survey_two_pass_bytes": round(bytes_survey / t_it / 1e9, 1),
                     "init_ms": round(t_init * 1e3, 3),
                     "phibar": st.phibar, "iterations": int(st.it)},
            "recover": {"ms": round(t_rec * 1e3, 3)},
            "solve_s": round(step_s, 4),
        },
        "clocks": clk,
        "gpu_launches": args.steps * launches_per_step(fs, iters),
    }

    # ---- the paper's protocol: one solve at 10 000 LSQR iterations
    if not args.no_paper:
        paper = Pipeline(wl, 10_000)
        paper.plan, paper.store, paper.system = pipe.plan, pipe.store, pipe.system
        ev = paper.events()
        paper.step(ev)
        torch.cuda.synchronize()
        tp = stage_times([ev])
        out["paper_protocol"] = {
            "lsqr_iters": 10_000, "solve_s": round(ev[0].elapsed_time(ev[5]) / 1e3, 4),
            "lsqr_ms_per_iter": round(tp["lsqr"] / 10_000 * 1e3, 4),
            "phibar": paper.run.read_state().phibar}
        del paper

    # ---- end to end through the public API, host buffers
    if not args.no_e2e:
        fl_steps = max(args.e2e_steps, 1)

        def e2e_step():
            system_h = fl.assemble(wl.problem, wl.dec, wl.basis, interior_per_dim=wl.interior_per_dim)
            fs_h = fl.filter_system(system_h, wl.sigma)
            res = fl.lsqr(fl.precondition(fs_h), system_h.rhs, iters)
            return fl.recover_solution(fs_h, res.solution)
        # cold: the lattice row-structure cache empty (first call on a geometry)
        assembly._LAYOUT_CACHE.clear()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        e2e_step()
        torch.cuda.synchronize()
        cold = time.perf_counter() - t0
        barrier()
        x0 = dict(D.XFER)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(fl_steps):
            e2e_step()
        e1.record()
        torch.cuda.synchronize()
        t_e2e = max_over_ranks(e0.elapsed_time(e1) / 1e3)
        out["e2e"] = {"value": round(whole_job_rate(world, fl_steps, t_e2e), 6), "unit": UNIT,
                      "h2d_bytes_per_step": int((D.XFER["h2d"] - x0["h2d"]) / fl_steps),
                      "d2h_bytes_per_step": int((D.XFER["d2h"] - x0["d2h"]) / fl_steps),
                      "ms_per_step": round(t_e2e / fl_steps * 1e3, 2),
                      "cold_ms": round(cold * 1e3, 2),
                      "cold_note": "first public-API solve on a new geometry (layout cache empty)"}

    # ---- every BASELINE config, one solve each (rank 0, N = 1)
    if rank == 0 and world == 1 and not args.no_configs:
        table = {}
        main_tab = stage_table(w, t, iters, hbm, fp64_peak_tf)
        main_tab["kept"] = int(fs.kept_total)
        del pipe
        torch.cuda.empty_cache()
        for name in ("cfg1", "cfg2", "cfg3", "cfg4", "cfg5"):
            if name == args.config:
                table[name] = main_tab
                continue
            p2 = Pipeline(workloads.build(name), iters)
            p2.step(p2.events())
            # three timed solves, per-stage median (a single solve's RRQR stage
            # varied by up to 2x between runs at cfg3 / cfg5)
            evs = [p2.events() for _ in range(3)]
            for ev in evs:
                p2.step(ev)
            torch.cuda.synchronize()
            per = [stage_times([ev]) for ev in evs]
            med = {k: float(np.median([q[k] for q in per])) for k in per[0]}
            tab = stage_table(p2.work(), med, iters, hbm, fp64_peak_tf,
                              latency_bound=name in ("cfg1", "cfg2"))
            tab["rrqr_ms_runs"] = [round(q["rrqr"] * 1e3, 2) for q in per]
            tab["kept"] = int(p2.fs.kept_total)
            table[name] = tab
            del p2
            torch.cuda.empty_cache()
        out["per_config"] = table
    if rank == 0 and world == 1 and not args.no_cpu:
        out["cpu_baseline"] = ref_sample(wl, iters, args.cpu_per_stratum, seed=1)
    return out


# ---------------------------------------------------------------- CPU: featlsq itself
class SampledDecomposition:
    """A featlsq `Decomposition` whose per-block loops see only the blocks in
    `sel` (block i of the view is block sel[i] of the full grid). Everything
    else — centres, half widths, count_per_dim, the coverage check
    (`domains.py:187-196` walks count_per_dim, not subdomain_count) — is the
    full decomposition's, so featlsq's `assemble` builds the full lattice,
    coverage check and right-hand side and only the sampled blocks."""

    def __init__(self, dec, sel):
        self._dec, self._sel = dec, list(sel)

    def __getattr__(self, name):
        return getattr(self._dec, name)

    @property
    def subdomain_count(self):
        return len(self._sel)

    def multi_index(self, j):
        return self._dec.multi_index(self._sel[j])


def _block_rows(wl):
    """m_j of every block (interior box + constraint points in support),
    for the work model only."""
    dec, prob = wl.dec, wl.problem
    d, S = dec.dim, dec.count_per_dim
    n = wl.interior_per_dim
    per = [[int(np.sum(np.abs(np.linspace(dec.domain.bounds[i, 0], dec.domain.bounds[i, 1], n)
                              - dec.centers[i, s]) < dec.half_widths[i])) for s in range(S)]
           for i in range(d)]
    multi = np.array(np.unravel_index(np.arange(S ** d), (S,) * d)).T
    m = np.ones(S ** d, dtype=np.int64)
    for i in range(d):
        m *= np.array(per[i])[multi[:, i]]
    for con in prob.constraints:
        pts = np.atleast_2d(con.points)
        inside = np.ones((S ** d, pts.shape[0]), dtype=bool)
        for i in range(d):
            mem = np.abs(pts[None, :, i] - dec.centers[i][:, None]) < dec.half_widths[i]
            inside &= mem[multi[:, i]]
        m += inside.sum(axis=1)
    return m, multi


def config_of(args, wl, iters, world, rows):
    """The workload description both arms print (same keys and values: the
    driver compares them). Sizes from the host-side block row counts."""
    m, _ = _block_rows(wl)
    K = wl.basis.feature_count
    return {"workload": f"{args.config}: {wl.description}", "lsqr_iters_per_solve": iters,
            "sigma": wl.sigma, "rows": rows, "cols": int(m.size * K),
            "l2": f"inputs larger than L2 (A {float(m.sum()) * K * 8 / 1e9:.2f} GB of block entries, "
                  f"Q of the same order)",
            "parallelism": f"replicas x{world}"}


def ref_sample(wl, iters, per_stratum, seed):
    """featlsq's own stage functions on a stratified block sample of the
    workload, extrapolated to the full solve (module docstring)."""
    import time as _t
    from paper_2506_17626_b200._featlsq import featlsq
    from featlsq import assembly as RA, filtering as RF, solvers as RS
    dec, basis, prob = wl.dec, wl.basis, wl.problem
    d, S, K = dec.dim, dec.count_per_dim, basis.feature_count
    J = S ** d
    m, multi = _block_rows(wl)
    faces = ((multi == 0) | (multi == S - 1)).sum(axis=1)
    rng = np.random.default_rng(seed)
    strata = {}
    for f in np.unique(faces):
        members = np.nonzero(faces == f)[0]
        pick = rng.choice(members, min(per_stratum, members.size), replace=False)
        strata[int(f)] = (members, np.sort(pick))
    sel = np.concatenate([p for _, p in strata.values()])

    def sampled(s):
        sd = SampledDecomposition(dec, s)
        sb = featlsq.FeatureBasis(sd, K, basis.depth, basis.activation,
                                  tuple(w[s] for w in basis.weights),
                                  tuple(None if b is None else b[s] for b in basis.biases))
        return sd, sb

    # global part of assemble (lattice, coverage, rhs): a zero-block view
    sd0, sb0 = sampled(np.zeros(0, dtype=int))
    t0 = _t.perf_counter()
    RA.assemble(prob, sd0, sb0, interior_per_dim=wl.interior_per_dim)
    t_glob = _t.perf_counter() - t0
    # per-block assembly and RRQR, one block at a time (featlsq's own loops)
    t_asm, t_qr, blocks, fblocks = {}, {}, [], []
    for j in sel:
        sd, sb = sampled(np.array([j]))
        t0 = _t.perf_counter()
        sysj = RA.assemble(prob, sd, sb, interior_per_dim=wl.interior_per_dim)
        t1 = _t.perf_counter()
        fsj = RF.filter_system(sysj, wl.sigma)
        t2 = _t.perf_counter()
        t_asm[int(j)] = max(t1 - t0 - t_glob, 0.0)
        t_qr[int(j)] = t2 - t1
        blocks.append(sysj.blocks[0])
        fblocks.append(fsj.blocks[0])
    # LSQR on the sampled blocks' preconditioned operator (featlsq's CSR)
    sd, sb = sampled(sel)
    sys_s = featlsq.GlobalSystem(prob, sd, sb, [RA.SubdomainBlock(i, b.rows, sb.column_range(i), b.matrix)
                                                for i, b in enumerate(blocks)],
                                 sysj.rhs, sysj.interior_count, sysj.row_count, sb.column_count,
                                 sysj.lattice_axes)
    kept = np.array([fb.kept_count for fb in fblocks])
    # each block was filtered as block 0 of a one-block view: shift to slot i
    fbl = [RF.FilteredBlock(i, fb.rows, fb.kept_columns + i * K, fb.dropped_columns + i * K,
                            fb.q_factor, fb.r_factor)
           for i, fb in enumerate(fblocks)]
    offsets = np.concatenate([[0], np.cumsum(kept)])
    fs_s = RF.FilteredSystem(sys_s, wl.sigma, fbl, offsets)
    op = RF.precondition(fs_s)
    t0 = _t.perf_counter()
    op.csr()
    t1 = _t.perf_counter()
    n_it = 5
    res = RS.lsqr(op, sys_s.rhs, n_it)
    t2 = _t.perf_counter()
    RF.recover_solution(fs_s, res.solution)
    t3 = _t.perf_counter()
    # extrapolation: per stratum, assembly ~ m_j, RRQR ~ m_j K^2; Q nonzeros
    # ~ m_j * (stratum mean kept fraction)
    asm_full = qr_full = nnz_full = 0.0
    for f, (members, pick) in strata.items():
        msum_p = float(m[pick].sum())
        asm_full += sum(t_asm[int(j)] for j in pick) / msum_p * float(m[members].sum())
        qr_full += sum(t_qr[int(j)] for j in pick) / msum_p * float(m[members].sum())
        kfrac = float(np.mean([fblocks[list(sel).index(j)].kept_count for j in pick])) / K
        nnz_full += float(m[members].sum()) * K * kfrac
    nnz_s = float(sum(b.rows.size * fb.kept_count for b, fb in zip(blocks, fblocks)))
    scale_q = nnz_full / nnz_s
    t_it = (t2 - t1) / n_it * scale_q
    solve = (t_glob + asm_full + qr_full + (t1 - t0) * scale_q + iters * t_it
             + (t3 - t2) * J / len(sel))
    return {"value": round(1.0 / solve, 8), "unit": UNIT, "cores": os.cpu_count(),
            "kind": "reference", "rows": int(sysj.row_count),
            "sample": (f"featlsq (baseline/_ref) assemble / filter_system / precondition / lsqr / "
                       f"recover_solution on {len(sel)} of {J} blocks ({per_stratum} per "
                       f"corner/edge/interior stratum, seed {seed}) plus the full lattice, "
                       f"coverage check and rhs; {n_it} LSQR iterations; extrapolated per "
                       f"stratum (assembly ~ m_j, RRQR ~ m_j K^2, LSQR/CSR ~ nnz(Q), factor "
                       f"{J / len(sel):.0f}x blocks, {scale_q:.0f}x nonzeros) to the full "
                       f"{iters}-iteration solve; OpenBLAS threads = all {os.cpu_count()} cores, "
                       f"CSR SpMV single-threaded; host {platform.processor() or platform.machine()}"),
            "stages": {"solve_s": round(solve, 2), "assemble_s": round(t_glob + asm_full, 2),
                       "assemble_global_s": round(t_glob, 3), "rrqr_s": round(qr_full, 2),
                       "csr_build_s": round((t1 - t0) * scale_q, 2),
                       "lsqr_ms_per_iter": round(t_it * 1e3, 2),
                       "recover_s": round((t3 - t2) * J / len(sel), 4),
                       "sample_blocks": [int(j) for j in sel]}}


def reference(args, rank, world):
    from paper_2506_17626_b200 import workloads
    wl = workloads.build(args.config, seed=0)
    iters = args.lsqr_iters
    if args.warmup > 0:  # first scipy.linalg.qr call pays LAPACK start-up
        ref_sample(wl, iters, 1, seed=1000)
    vals = []
    t0 = time.perf_counter()
    for k in range(args.steps):
        vals.append(ref_sample(wl, iters, args.cpu_per_stratum, seed=k + 1))
    wall = time.perf_counter() - t0
    est = np.array([v["stages"]["solve_s"] for v in vals])
    mid = vals[int(np.argsort(est)[len(est) // 2])]
    return {"impl": "reference", "metric": METRIC, "value": mid["value"], "unit": UNIT,
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round(1e3 / mid["value"], 1), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (SURVEY.md §8(d) inputs, seeded)",
            "config": config_of(args, wl, iters, world, int(mid["rows"])),
            "cpu_baseline": {"value": mid["value"], "unit": UNIT, "cores": mid["cores"],
                             "kind": mid["kind"], "sample": mid["sample"]},
            "e2e": {"value": mid["value"], "unit": UNIT, "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0},
            "sampling_error": {"solve_s_per_step": [round(float(x), 1) for x in est],
                               "rel_spread": round(float((est.max() - est.min()) / np.median(est)), 4),
                               "note": "each step draws a new stratified sample; value = median step"},
            "stages": mid["stages"], "wall_s": round(wall, 2)}


def main():
    args = parse()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        if rank != 0:
            return
        print(json.dumps(reference(args, rank, world)), flush=True)
        return
    if world > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local_rank)
        dist.init_process_group("nccl")
    out = product(args, rank, world, local_rank)
    if rank == 0:
        print(json.dumps(out), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
