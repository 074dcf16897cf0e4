#!/usr/bin/env python
"""Benchmark of the B200 S_N hot path (repo BASELINE.json metric).

Workload (N=1): BASELINE configs[1] = C2, 2048 instances x 2000 cells x S32, parametric
sinusoidal Sigma_t, vacuum, source iteration to rel-Linf < 1e-8 from a zero guess. One "step"
= one batched solve of all 2048 instances by the fused source-iteration kernel (K1).

  value      cell.angle.group sweep updates/s (sum over instances of iterations x N x Nc),
             inputs resident in HBM, device time (CUDA events on the solver stream).
  e2e        same metric through the public host API (numpy arrays in pinned host memory, in and out;
             H2D of the inputs + D2H of flux/iterations inside the timed region).
  roofline   algorithmic bytes per launch (40 B per cell per source iteration)
             / average launch time, vs the measured HBM copy bandwidth.
  cpu_baseline / --impl reference
             the CPU oracle (restated reference solver; the reference's own solver sources are
             absent) on the host cores, bounded sample of the same workload.

Multi-GPU (torchrun): instances are independent -> each rank solves its own
2048-instance batch (seed offset by rank, weak scaling), no data-path collective; the step time
is the max over ranks.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import tempfile
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "cell_angle_group_sweep_updates_per_sec"
UNIT = "updates/s"
BYTES_PER_CELL_ITER = 40  # read St, Ss0, q_ext, phi_old; write phi_new


def peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d.get("hbm_gbs", 6650.0)), "measured"
    return 6650.0, "fallback"


def fno_flops_per_sample(n, width=64, modes=16, layers=4, hidden=128):
    """Algorithmic FLOPs of one FNO forward per sample: lift 2 -> C, per layer the
    truncated forward DFT (2 n 2M C), the complex mixing (M C C x 8), the inverse DFT and the W
    path (2 n C C), projection C -> hidden -> 1."""
    lift = 2 * n * 2 * width
    layer = 2 * n * 2 * modes * width * 2 + modes * width * width * 8 + 2 * n * width * width
    proj = 2 * n * (width * hidden + hidden)
    return lift + layers * layer + proj


def timed_device(ctx, stream, fn, reps=2):
    """min device time (s) of fn() over reps runs, CUDA events on the solver stream, after one
    untimed run; returns the last result too."""
    import torch
    out = fn()
    ts = []
    for _ in range(reps):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        out = fn()
        e1.record(stream)
        ctx.synchronize()
        ts.append(e0.elapsed_time(e1) / 1e3)
    return out, float(np.min(ts))


def warm_stats(r, t, batch, it_cold_mean):
    """One MD-PNOP arm (precondition_fixed_source) as a bench record."""
    pit, ref = r.precond_iterations.to(torch_int64()), r.refine_iterations.to(torch_int64())
    return {"ms": 1e3 * t, "solves_per_sec": batch / t,
            "recast_iterations_mean": float(pit.float().mean().item()), "recast_iterations_max": int(pit.max().item()),
            "recast_status_counts": [int((r.recast_status == k).sum().item()) for k in range(3)],
            "refine_iterations_mean": float(ref.float().mean().item()), "refine_iterations_max": int(ref.max().item()),
            "refine_iteration_ratio_vs_zero_guess": float(ref.float().mean().item()) / it_cold_mean}


def torch_int64():
    import torch
    return torch.int64


def c5_arm(snop, ctx, stream, args):
    """BASELINE configs[4] (C5): the MD-PNOP warm start on 4096 x 1024-cell S16 instances
    (SURVEY §9 #11): zero guess; the random-init FNO (4 layers, width 64, 16 modes, lift 2->64,
    proj 64->128->1, GELU) single shot (Eq. 9) and as the full recast fixed point (tol 1e-4, max
    50); the exact operator (the model-based solve at p*) single shot and full fixed
    point - the arm that shows the mechanism, since no trained weights ship; and Delta p = 0 with
    the exact operator (refine <= 2 iterations). Device-resident inputs, CUDA events."""
    import torch
    from paper_2509_01416_b200 import operators as OPS, workloads as W
    p = W.config5()
    g = snop.Grid1D(p.length, p.n_cells)
    cfg = snop.SolverConfig(tolerance=p.tolerance)
    st, ss, src = (torch.from_numpy(a).cuda() for a in (p.sigma_t, p.sigma_s0, p.source))
    fno = snop.SolutionOperator.fno(g, OPS.fno_init(64, 16, 4, 128, OPS.GELU), p.ref_params, ctx=ctx)
    exact = snop.SolutionOperator.exact(g, p.order, p.ref_params, snop.SolverConfig(tolerance=p.tolerance), ctx=ctx)

    cold, t_cold = timed_device(ctx, stream, lambda: snop.source_iteration(g, p.order, st, ss, src, cfg, ctx=ctx,
                                                                           sync=False))
    _, t_op = timed_device(ctx, stream, lambda: fno.predict(src, sync=False), reps=3)
    it_cold = cold.iterations.to(torch.int64)
    it_mean = float(it_cold.float().mean().item())
    upd = int(it_cold.sum().item()) * p.n_cells * p.order
    alg = int(it_cold.sum().item()) * p.n_cells * BYTES_PER_CELL_ITER / t_cold / 1e9
    flops = fno_flops_per_sample(p.n_cells) * p.batch
    tf32 = tf32_peak()
    arms = {}
    for name, op, rmax in (("fno_single_shot", fno, 1), ("fno_recast_fixed_point", fno, 50),
                           ("exact_single_shot", exact, 1), ("exact_recast_fixed_point", exact, 50)):
        r, t = timed_device(ctx, stream, lambda: snop.precondition_fixed_source(
            op, p.order, st, ss, src, cfg, recast_tolerance=1e-4, recast_max_iterations=rmax))
        arms[name] = warm_stats(r, t, p.batch, it_mean)
    one = torch.ones_like(st)
    r, t = timed_device(ctx, stream, lambda: snop.precondition_fixed_source(exact, p.order, one, 0.8 * one, src, cfg))
    arms["exact_delta_p0"] = warm_stats(r, t, p.batch, it_mean)
    arms["exact_delta_p0"]["note"] = "instances at p* (Sigma_t = 1, Sigma_s = 0.8): SPEC.md:421 refine <= 2"
    out = {"workload": "C5 4096x1024 S16, p*=(1.0,0.8), tol 1e-8; FNO random-init (seeded), fp32 on tcgen05 (3xTF32)",
           "zero_guess_ms": 1e3 * t_cold, "solves_per_sec_zero_guess": p.batch / t_cold,
           "zero_guess_updates_per_sec": upd / t_cold, "iterations_mean_zero_guess": it_mean,
           "zero_guess_roofline": {"bound": "hbm", "achieved": alg, "peak": peaks()[0], "unit": "GB/s",
                                   "frac": alg / peaks()[0],
                                   "note": "K1 at S16: 40 B per cell per iteration = 2.5 B per update"},
           "operator_ms": 1e3 * t_op,
           "operator_roofline": None,
           "warm_start": arms,
           # the fixed-point arm is the warm start SURVEY §9 #11 names; single shot beside it
           "warm_start_ms": arms["fno_recast_fixed_point"]["ms"],
           "solves_per_sec_warm_start": arms["fno_recast_fixed_point"]["solves_per_sec"],
           "iterations_mean_warm_start": arms["fno_recast_fixed_point"]["refine_iterations_mean"]}
    if tf32:
        out["operator_roofline"] = {
            "bound": "tensor", "achieved": flops / t_op / 1e12, "peak": tf32, "unit": "TFLOP/s",
            "frac": flops / t_op / 1e12 / tf32, "flops_per_forward": flops,
            "frac_3xtf32_issued": 3 * flops / t_op / 1e12 / tf32,
            "note": "algorithmic FNO FLOPs (SURVEY §8d) / forward time vs the measured tcgen05 TF32 burst peak "
                    "(profiles/tf32_peak.json); the GEMMs issue 3 TF32 products per fp32 product (3xTF32)"}
    return out


def tf32_peak():
    p = ROOT / "profiles" / "tf32_peak.json"
    if not p.exists():
        return None
    return float(json.loads(p.read_text())["tf32_tflops"])


def eigen_arms(snop, ctx, stream, args):
    """BASELINE configs[2] (C3: 512 x 4096 S32 single-group, reflective-left / vacuum-right) and
    configs[3] (C4: 128 x 2000 S16, G = 7 with upscatter, Gauss-Seidel over groups): one batched
    power iteration (fused K2) per step, device-resident inputs, CUDA-event timing; beside it the
    CPU oracle on a bounded sample of the same instances (all host threads), and the k parity of
    that sample."""
    import torch
    from paper_2509_01416_b200 import workloads as W
    from tests import oracle_lib as O
    th = O.hardware_threads()
    out = {}
    for name, p, n_cpu in (("c3_eigen", W.config3(), args.cpu_eigen_sample), ("c4_multigroup", W.config4(),
                                                                               args.cpu_eigen_sample)):
        g = snop.Grid1D(p.length, p.n_cells)
        cfg = snop.SolverConfig(tolerance=p.tolerance_inner, tolerance_k=p.tolerance_k, tolerance_phi=p.tolerance_phi,
                                boundary_left=p.bc_left, boundary_right=p.bc_right)
        dev = [torch.from_numpy(a).cuda() for a in (p.sigma_t, p.sigma_s0, p.nu_sigma_f, p.chi)]
        r = snop.power_iteration(g, p.order, *dev, cfg, ctx=ctx)
        ts = []
        for _ in range(2):
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            r = snop.power_iteration(g, p.order, *dev, cfg, ctx=ctx, sync=False)
            e1.record(stream)
            ctx.synchronize()
            ts.append(e0.elapsed_time(e1) / 1e3)
        t = float(np.min(ts))
        inner = r.total_inner_iterations.to(torch.int64)
        outer = r.outer_iterations.to(torch.int64)
        upd = int(inner.sum().item()) * p.n_cells * p.order
        k_gpu = r.k.cpu().numpy()
        q = p.subset(np.arange(n_cpu))
        t0 = time.perf_counter()
        o = O.power_iteration(q.length, q.n_cells, q.order, q.n_groups, q.sigma_t, q.sigma_s0, q.nu_sigma_f, q.chi,
                              cfg.c(), n_threads=th)
        tc = time.perf_counter() - t0
        upd_cpu = int(o["inner"].astype(np.int64).sum()) * q.n_cells * q.order
        out[name] = {
            "workload": f"{p.name} {p.batch}x{p.n_cells} S{p.order} G={p.n_groups}, power iteration tol_k "
                        f"{p.tolerance_k:g} tol_phi {p.tolerance_phi:g}",
            "ms_per_solve_batch": 1e3 * t, "solves_per_sec": p.batch / t, "updates_per_sec": upd / t,
            "outer_mean": float(outer.float().mean().item()), "outer_max": int(outer.max().item()),
            "inner_sweeps_total": int(inner.sum().item()),
            "cpu_baseline": {"solves_per_sec": n_cpu / tc, "updates_per_sec": upd_cpu / tc, "cores": th,
                             "kind": "port", "sample": f"first {n_cpu} of the {p.batch} instances, full solve, "
                                                       f"{tc:.1f} s"},
            "k_parity_vs_oracle_sample": float(np.max(np.abs(k_gpu[:n_cpu] - o["k"]) / np.abs(o["k"]))),
        }
    return out


def sweep_arm(snop, ctx, stream, args):
    """The standalone transport sweep (snop_sweep_batched) at the C2 and C5 sizes:
    one diamond-difference sweep of all directions with a per-direction emission, psi materialised.
    This is the HBM-bound form of the sweep kernel (16 B per cell.angle update + 8 B per cell of
    Sigma_t); inputs and outputs (1.1-2.1 GB) are far larger than L2. Device-resident inputs, R
    back-to-back calls between CUDA events; the CPU oracle's sweep on a sample, all host threads."""
    import torch
    from tests import oracle_lib as O
    th = O.hardware_threads()
    peak, peak_kind = peaks()
    prof = {}
    pj = ROOT / "profiles" / "r2_sweep_dram_bytes.json"
    if pj.exists():
        prof = json.loads(pj.read_text())
    out = {}
    for name, B, Nc, N in (("c2", 2048, 2000, 32), ("c5", 4096, 1024, 16)):
        gen = torch.Generator(device="cuda").manual_seed(1234)
        st = torch.rand((B, Nc), generator=gen, device="cuda", dtype=torch.float64) * 1.8 + 0.2
        em = torch.rand((B, Nc, N), generator=gen, device="cuda", dtype=torch.float64)
        g = snop.Grid1D(10.0, Nc)
        R = 8
        snop.sweep(g, N, st, em, ctx=ctx)
        ts = []
        for _ in range(3):
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            snop.sweep(g, N, st, em, ctx=ctx, sync=False)  # (the device is busy while the host enqueues the rest)
            e0.record(stream)
            for _ in range(R):
                psi, ol, orr = snop.sweep(g, N, st, em, ctx=ctx, sync=False)
            e1.record(stream)
            ctx.synchronize()
            ts.append(e0.elapsed_time(e1) / 1e3 / R)
        t = float(np.min(ts))
        alg = B * Nc * (16.0 * N + 8.0)
        n_cpu = max(th, 16)
        idx = np.arange(n_cpu)
        hs, he = st[idx].cpu().numpy(), em[idx].cpu().numpy()
        t0 = time.perf_counter()
        reps = 0
        while time.perf_counter() - t0 < 2.0:
            o_psi, _, _ = O.sweep(10.0, Nc, N, hs, he, n_threads=th)
            reps += 1
        tc = (time.perf_counter() - t0) / reps
        err = float(np.max(np.abs(psi[idx].cpu().numpy() - o_psi)) / np.max(np.abs(o_psi)))
        pr = prof.get(name, {})
        out[name] = {
            "workload": f"{B} x {Nc} cells x S{N}, vacuum faces, emission [B][Nc][N] -> psi_avg [B][N][Nc]",
            "ms_per_sweep": 1e3 * t, "updates_per_sec": B * Nc * N / t,
            "roofline": {"bound": "hbm", "achieved": alg / t / 1e9, "peak": peak, "unit": "GB/s",
                         "frac": alg / t / 1e9 / peak, "peak_source": peak_kind,
                         "traffic": (pr.get("dram_bytes_read", 0) + pr.get("dram_bytes_write", 0)) or None,
                         "traffic_source": "profile-derived (profiles/r2_sweep_dram_bytes.json), not measured here",
                         "note": "algorithmic bytes = 16 B per update (q in, psi out) + 8 B per cell (Sigma_t)"},
            "cpu_baseline": {"updates_per_sec": n_cpu * Nc * N / tc, "cores": th, "kind": "port",
                             "sample": f"oracle sweep of the first {n_cpu} instances, {reps} repetitions"},
            "psi_parity_vs_oracle_sample": err,
        }
        del st, em, psi
    return out


def hybrid_arms(snop, ctx, stream, args):
    """SP / CP hybrid eigen solves (paper Eqs. A5-A8) on the first
    args.hybrid_batch instances of C3 (512 x 4096 x S32 single-group eigen): stage 1 = power
    iteration whose within-group solve is the operator's recast fixed point (SP) or the operator
    prediction refined by a model-based solve (CP), stage 2 = model-based power iteration from
    (k_NO, phi_NO); against the cold model-based power iteration of the same instances. Operators:
    the exact operator at p* = (1.0, 0.5) (the model-based solve) and the random-init
    FNO. Stage 1's outer loop runs on the device (nested CUDA-graph loops)."""
    import torch
    from paper_2509_01416_b200 import operators as OPS, workloads as W
    p = W.config3().subset(np.arange(args.hybrid_batch))
    g = snop.Grid1D(p.length, p.n_cells)
    cfg = snop.SolverConfig(tolerance=p.tolerance_inner, tolerance_k=p.tolerance_k, tolerance_phi=p.tolerance_phi,
                            boundary_left=p.bc_left, boundary_right=p.bc_right)
    dev = [torch.from_numpy(a).cuda() for a in (p.sigma_t, p.sigma_s0, p.nu_sigma_f, p.chi)]
    cold, t_cold = timed_device(ctx, stream, lambda: snop.power_iteration(g, p.order, *dev, cfg, ctx=ctx, sync=False))
    inner_cold = int(cold.total_inner_iterations.sum().item())
    ops = {"exact": snop.SolutionOperator.exact(g, p.order, (1.0, 0.5), snop.SolverConfig(
               tolerance=p.tolerance_inner, boundary_left=p.bc_left, boundary_right=p.bc_right), ctx=ctx),
           "fno": snop.SolutionOperator.fno(g, OPS.fno_init(64, 16, 4, 128, OPS.GELU), (1.0, 0.5), ctx=ctx)}
    out = {"workload": f"C3 first {p.batch} instances x 4096 cells x S32, reflective-left, tol_k 1e-8 tol_phi 1e-7",
           "cold": {"ms": 1e3 * t_cold, "solves_per_sec": p.batch / t_cold,
                    "outer_mean": float(cold.outer_iterations.float().mean().item()), "inner_total": inner_cold}}
    # (SP with the exact operator is left to tools/md_pnop_probe.py: its stage 1 takes ~500 outers
    # of exact-operator fixed points, ~110 s for 32 instances - profiles/r2_md_pnop_c3_hybrid_probe.txt)
    for opname, alg in (("exact", "cp"), ("fno", "sp"), ("fno", "cp")):
        op = ops[opname]
        fn = getattr(snop, f"{alg}_eigen")
        r, t = timed_device(ctx, stream, lambda: fn(op, p.order, *dev, cfg), reps=1)
        out[f"{alg}_{opname}"] = {
            "ms": 1e3 * t, "solves_per_sec": p.batch / t,
            "stage1_outer_mean": float(r.stage1_outer.float().mean().item()),
            "stage2_outer_mean": float(r.stage2_outer.float().mean().item()),
            "stage2_inner_total": int(r.stage2_inner.sum().item()),
            "stage2_inner_ratio_vs_cold": int(r.stage2_inner.sum().item()) / max(inner_cold, 1),
            "fallback_count": int(r.fallback.sum().item()),
            "k_max_rel_diff_vs_cold": float(((r.k - cold.k).abs() / cold.k).max().item())}
    return out


def fp64_peak():
    p = ROOT / "profiles" / "fp64_peak.json"
    if not p.exists():
        return None
    d = json.loads(p.read_text())
    return float(d["dfma_per_clk_per_sm"]), float(d["k1_fp64_thread_ops_per_update"])


def dist_env():
    from paper_2509_01416_b200.distributed import env
    return env()


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.idx = gpu_index
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        self.p = None

    def __enter__(self):
        try:
            self.p = subprocess.Popen(["nvidia-smi", f"--id={self.idx}", f"--query-gpu={self.Q}",
                                       "--format=csv,noheader,nounits", "-lms", "50"],
                                      stdout=self.f, stderr=subprocess.DEVNULL)
        except FileNotFoundError:
            self.p = None
        # nvidia-smi takes a few hundred ms to start: wait for its first row so the whole (short)
        # timed region is sampled
        t0 = time.perf_counter()
        while self.p is not None and time.perf_counter() - t0 < 10.0:
            self.f.flush()
            if Path(self.f.name).read_text().strip():
                break
            time.sleep(0.02)
        self.n0 = len([r for r in Path(self.f.name).read_text().splitlines() if r.strip()])
        return self

    def __exit__(self, *a):
        if self.p is not None:
            self.p.terminate()
            try:
                self.p.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.p.kill()

    def summary(self):
        self.f.flush()
        rows = [r.split(",") for r in Path(self.f.name).read_text().splitlines() if r.strip()]
        rows = rows[getattr(self, "n0", 0):]  # rows taken before the timed region started
        os.unlink(self.f.name)
        sm = [float(r[1]) for r in rows if len(r) >= 9 and r[1].strip().replace(".", "").isdigit()]
        mx = [float(r[2]) for r in rows if len(r) >= 9 and r[2].strip().replace(".", "").isdigit()]
        reasons = set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in rows:
            if len(r) >= 9:
                for n, v in zip(names, r[5:9]):
                    if v.strip().lower() in ("active", "1"):
                        reasons.add(n)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "samples": len(sm), "reasons": sorted(reasons)}


def traffic_from_profiles():
    """dram bytes per launch of K1 from the committed ncu summary (profiles/), if present."""
    p = ROOT / "profiles" / "k1_dram_bytes.json"
    if p.exists():
        try:
            d = json.loads(p.read_text())
            return d.get("dram_bytes_per_launch_scaled_to_bench"), d
        except Exception:
            return None, None
    return None, None


def cpu_baseline(problem, n_inst: int, threads: int):
    """The CPU oracle (restated reference solver) on a bounded sample of the workload."""
    from tests import oracle_lib as O
    sub = problem.subset(np.arange(n_inst))
    cfg = O.make_config(sub.tolerance)
    t0 = time.perf_counter()
    r = O.source_iteration(sub.length, sub.n_cells, sub.order, sub.sigma_t, sub.sigma_s0, sub.source, cfg,
                           n_threads=threads)
    dt = time.perf_counter() - t0
    upd = int(r["iterations"].astype(np.int64).sum()) * sub.n_cells * sub.order
    return upd / dt, dt, upd, r


def bench_config(batch, world):
    """The workload both arms report (identical dicts; the reference arm's per-step CPU sample is
    described in its cpu_baseline.sample)."""
    return {"workload": "C2 fixed-source 2048x2000 S32, zero guess, tol 1e-8", "instances_per_gpu": batch,
            "n_cells": 2000, "order": 32, "l2": "GPU arm: flushed between timed steps (256 MB write)",
            "parallelism": f"instance-sharded x{world}" if world > 1 else "single GPU"}


def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return 0
    from paper_2509_01416_b200 import workloads as W
    from tests import oracle_lib as O
    threads = O.hardware_threads()
    p = W.config2(batch=args.batch, n_cells=2000)
    n_inst = args.cpu_sample
    for _ in range(args.warmup):
        cpu_baseline(p, max(1, n_inst // 8), threads)
    vals, times = [], []
    for s in range(args.steps):
        v, dt, upd, _ = cpu_baseline(p, n_inst, threads)
        vals.append(v)
        times.append(dt)
    value = float(np.sum([v * t for v, t in zip(vals, times)]) / np.sum(times))
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1e3 * float(np.mean(times)), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded, BASELINE C2)",
        "config": bench_config(args.batch, world),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "port",
                         "sample": f"{n_inst} of the 2048 C2 instances per step (same seeds), full solve"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))
    return 0


def run_gpu(args):
    import torch
    import torch.distributed as dist
    from paper_2509_01416_b200 import snop, workloads as W

    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    ctx = snop.Context(local)
    stream = torch.cuda.ExternalStream(ctx.stream_ptr, device=torch.device("cuda", local))
    from paper_2509_01416_b200.distributed import rank_seed, reduce_max, reduce_sum
    p = W.config2(batch=args.batch, n_cells=2000, seed=rank_seed(rank))
    g = snop.Grid1D(p.length, p.n_cells)
    cfg = snop.SolverConfig(tolerance=p.tolerance)
    dev = torch.device("cuda", local)
    st, ss, src = (torch.from_numpy(a).to(dev) for a in (p.sigma_t, p.sigma_s0, p.source))
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)  # > 126 MB L2

    def step(sync=True):
        return snop.source_iteration(g, p.order, st, ss, src, cfg, ctx=ctx, sync=sync)

    for _ in range(max(3, args.warmup)):
        r = step()
    iters = r.iterations.to(torch.int64)
    updates_per_step = int(iters.sum().item()) * p.n_cells * p.order
    bytes_per_step = int(iters.sum().item()) * p.n_cells * BYTES_PER_CELL_ITER

    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    launches0 = ctx.launch_count
    times = []
    with ClockSampler(local) as clk:
        for _ in range(args.steps):
            flush.zero_()  # L2 flush between timed steps (not timed)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            r = step(sync=False)
            e1.record(stream)
            ctx.synchronize()
            times.append(e0.elapsed_time(e1) / 1e3)
    launches = ctx.launch_count - launches0
    torch.cuda.synchronize()
    t_local = float(np.sum(times))
    t_max = reduce_max(t_local, dev)                      # device time, max over ranks
    total_updates = reduce_sum(updates_per_step, dev) * args.steps
    value = total_updates / t_max
    ms_per_step = 1e3 * t_max / args.steps
    solves_per_s = p.batch * world * args.steps / t_max

    # e2e through the public host API: pinned host arrays, H2D + D2H inside the timed region
    pin = [torch.from_numpy(a).pin_memory() for a in (p.sigma_t, p.sigma_s0, p.source)]
    host = [x.numpy() for x in pin]
    outs = (torch.empty((p.batch, p.n_cells), dtype=torch.float64).pin_memory().numpy(),
            torch.empty(p.batch, dtype=torch.int32).pin_memory().numpy(),
            torch.empty(p.batch, dtype=torch.uint8).pin_memory().numpy())
    snop.source_iteration(g, p.order, *host, cfg, ctx=ctx, out=outs)  # warm the staging buffers
    e2e_times = []
    for _ in range(args.steps):
        flush.zero_()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        rh = snop.source_iteration(g, p.order, *host, cfg, ctx=ctx, out=outs)
        e2e_times.append(time.perf_counter() - t0)
    upd_h = int(np.asarray(rh.iterations, dtype=np.int64).sum()) * p.n_cells * p.order
    e2e_t = reduce_max(float(np.sum(e2e_times)), dev)
    e2e_value = reduce_sum(upd_h, dev) * args.steps / e2e_t
    h2d = 3 * p.batch * p.n_cells * 8
    d2h = p.batch * p.n_cells * 8 + p.batch * 4 + p.batch

    # MD-PNOP warm-start arm (BASELINE C2): random-init DeepONet (branch 2000->128x4, trunk 1->128x4,
    # tanh) on the recast source, then the model-based solve from phi_NO: single
    # shot (Eq. 9) and the full recast fixed point (tol 1e-4, max 50).
    warm = None
    if not args.no_warm_start:
        from paper_2509_01416_b200 import operators as OPS
        don = snop.SolutionOperator.deeponet(g, OPS.deeponet_init(p.n_cells), p.ref_params, ctx=ctx)
        it_mean = float(iters.float().mean().item())
        arms = {}
        for name, rmax in (("single_shot", 1), ("recast_fixed_point", 50)):
            rw, tw = timed_device(ctx, stream, lambda: snop.precondition_fixed_source(
                don, p.order, st, ss, src, cfg, recast_tolerance=1e-4, recast_max_iterations=rmax), reps=3)
            arms[name] = warm_stats(rw, tw, p.batch, it_mean)
        _, t_op = timed_device(ctx, stream, lambda: don.predict(src, sync=False), reps=3)
        warm = {"operator": "DeepONet 2000->128x4 / 1->128x4, p=128, tanh, random-init (seeded Xavier), fp32 "
                            "on tcgen05 (3xTF32)",
                "operator_ms": 1e3 * t_op, "zero_guess_iterations_mean": it_mean, "arms": arms,
                "timing": "min of 3 device-timed solves (CUDA events on the solver stream)",
                "note": "random-init operator: the warm start does not reduce iterations (DESIGN.md §5); "
                        "the exact-operator arms of c5_fno_warm_start show the mechanism"}

    c5 = None if (args.no_c5 or world > 1) else c5_arm(snop, ctx, stream, args)
    eig = None if (args.no_eigen or world > 1) else eigen_arms(snop, ctx, stream, args)
    hyb = None if (args.no_hybrid or world > 1) else hybrid_arms(snop, ctx, stream, args)
    swp = None if (args.no_sweep or world > 1) else sweep_arm(snop, ctx, stream, args)

    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return 0

    peak, peak_kind = peaks()
    avg_launch = t_local / args.steps
    achieved = bytes_per_step / avg_launch / 1e9
    traffic, _ = traffic_from_profiles()
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": max(3, args.warmup), "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded, BASELINE C2)",
        "config": bench_config(p.batch, world),
        "solves_per_sec": solves_per_s,
        "iterations": {"mean": float(iters.float().mean().item()), "max": int(iters.max().item()),
                       "min": int(iters.min().item())},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                     "traffic": traffic, "peak_source": peak_kind,
                     "traffic_source": "profile-derived: ncu dram__bytes_read.sum + dram__bytes_write.sum of one "
                                       "launch of this workload (profiles/k1_dram_bytes.json), not measured here",
                     "note": "algorithmic bytes = 40 B per cell per source iteration; the kernel keeps instance "
                             "state on-chip, so DRAM traffic is far below this; fp64-issue bound (DESIGN.md)"},
        "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h},
        "gpu_launches": int(launches),
        "clocks": clk.summary(),
    }
    fp = fp64_peak()
    if fp is not None:  # the kernel's binding ceiling (report both, name the binding one)
        per_sm_clk, ops_per_update = fp
        sm_mhz = (line["clocks"] or {}).get("sm_mhz") or 1965.0
        peak_ops = per_sm_clk * torch.cuda.get_device_properties(dev).multi_processor_count * sm_mhz * 1e6
        ach = value / world * ops_per_update
        line["roofline_fp64"] = {"bound": "fp64-issue", "achieved": ach / 1e12, "peak": peak_ops / 1e12,
                                 "unit": "T fp64-ops/s", "frac": ach / peak_ops,
                                 "note": "fp64 pipe instructions per update from ncu (profiles/fp64_peak.json); "
                                         "peak = measured DFMA rate per SM x SMs x sampled SM clock"}
    if warm is not None:
        line["warm_start"] = warm
    if c5 is not None:
        line["c5_fno_warm_start"] = c5
    if eig is not None:
        line.update(eig)
    if hyb is not None:
        line["c3_hybrid_eigen"] = hyb
    if swp is not None:
        line["sweep_standalone"] = swp
    if not args.no_cpu_baseline and world == 1:
        from tests import oracle_lib as O
        th = O.hardware_threads()
        v, dt, _, _ = cpu_baseline(p, args.cpu_sample, th)
        line["cpu_baseline"] = {"value": v, "unit": UNIT, "cores": th, "kind": "port",
                                "sample": f"{args.cpu_sample} of the 2048 C2 instances (same seeds), full solve, "
                                          f"{dt:.1f} s"}
    print(json.dumps(line))
    if world > 1:
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--batch", type=int, default=2048)
    ap.add_argument("--cpu-sample", type=int, default=2048)
    ap.add_argument("--cpu-eigen-sample", type=int, default=16)
    ap.add_argument("--no-eigen", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-warm-start", action="store_true")
    ap.add_argument("--no-c5", action="store_true", help="skip the C5 FNO warm-start arm")
    ap.add_argument("--no-hybrid", action="store_true", help="skip the C3 SP/CP hybrid eigen arm")
    ap.add_argument("--no-sweep", action="store_true", help="skip the standalone sweep arm")
    ap.add_argument("--hybrid-batch", type=int, default=32)
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)
    return run_gpu(args)


if __name__ == "__main__":
    sys.exit(main())
