#!/usr/bin/env python
"""Benchmark of the reduced-hybrid FDTD hot path (BASELINE.json metric:
Mcell-updates/s of the coarse grid + reduced blocks on one B200).

A bench "step" is one full run of the workload: config 2 of BASELINE.json
(2-D 1024x1024 coarse cells, one 64x64-cell box refined 8x reduced to q = 256,
20,000 time steps, fp32) from the current state, inputs resident in HBM.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

N > 1 (torchrun): N independent replicas (weak scaling); time =
max over ranks.  Rank 0 prints one JSON line.  --impl reference times the CPU
oracle (the reference arm of this tier) on a bounded sample of the workload.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
for p in (ROOT, os.path.join(ROOT, "tests")):
    if p not in sys.path:
        sys.path.insert(0, p)

import numpy as np  # noqa: E402

WORKLOADS = {
    2: "config2: 2-D Ez/Hx/Hy PEC cavity 1024x1024 cells of 0.5 mm, 32 dielectric inclusions, "
       "64x64-cell box refined 8x -> reduced block q=256 (recipe B), dt = 4x fine CFL, 20000 steps, fp32",
    3: "config3: 3-D PEC cavity 256^3 cells of 1 mm, random initial E, dt = 0.99 CFL, 1000 steps",
    5: "config5: 3-D microstrip-shaped 400x200x40 cells of 0.25 mm, eps_r 3.38 substrate, PEC strips with "
       "64 stubs, 64 z-refined (r=10) stub-tip regions reduced to q=128 in 2 shared models (32 instances "
       "each), dt = 6x fine CFL, 50000 steps, fp32",
    4: "config4: 3-D PEC rectangular waveguide 512x128x128 cells of 0.5 mm, 2-cell iris slab refined 10x in x "
       "-> one reduced block q=1024 (65,024 interface rows), B=16 modulated-Gaussian TE10 port excitations, "
       "dt = 8x fine CFL, 10000 steps, fp32",
}


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index=0):
        self.index = index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), "--query-gpu=" + self.FIELDS,
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.th = threading.Thread(target=self._read, daemon=True)
            self.th.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if not self.proc:
            return None
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, mx, reasons = [], 0.0, set()
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        for ln in self.lines:
            parts = [x.strip() for x in ln.split(",")]
            if len(parts) < 8:
                continue
            try:
                sm.append(float(parts[0]))
                mx = max(mx, float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[4:8]):
                if v.lower() == "active":
                    reasons.add(nm)
        if not sm:
            return None
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


def build_workload(config, precision, rank=0):
    from synth import scenario
    from paper_1406_7042_b200 import prep
    scn = scenario(config, precision=precision)
    prob, info = prep.build_problem(scn, precision=precision)
    if rank and prob.get("sources"):
        from paper_1406_7042_b200.dist import replica_scale
        prob = dict(prob)
        prob["sources"] = dict(prob["sources"])
        prob["sources"]["wave"] = np.asarray(prob["sources"]["wave"]) * replica_scale(rank)
    return scn, prob, info


def cells_of(prob):
    n = prob["n"]
    return int(n[0] * n[1] * (n[2] if prob["dim"] == 3 else 1))


def algorithmic_bytes_per_cell(prob, precision):
    w = 4 if precision == 32 else 8
    words = 12 if prob["dim"] == 3 else 6
    mat = 1 if prob.get("mat_id") is not None else 0
    return words * w + mat


def run_oracle_sample(prob, seconds=15.0, max_steps=800):
    """Time the CPU oracle (oracle.problem_step, single-threaded SciPy SpMV) on a
    bounded number of steps of the same workload."""
    try:
        from threadpoolctl import threadpool_limits
        lim = threadpool_limits(limits=1)
    except Exception:
        lim = None
    from oracle import problem_step as ps
    from oracle.matrix_form import step_leapfrog
    rec = ps.build(prob)
    E, H = ps.initial_state(rec, prob, 0)
    PE, PH = ps.probe_matrices(rec)
    done, t0 = 0, time.perf_counter()
    while done < max_steps:
        su = None
        if len(rec.src_row) and done < rec.wave.shape[0]:
            su = np.zeros(len(E))
            np.add.at(su, rec.src_row, -rec.src_coef * rec.wave[done, rec.src_col, 0])
        E, H = step_leapfrog(E, H, rec.GE, rec.GH, rec.KE, rec.KH, su_E=su)
        _ = PE @ E + PH @ H
        done += 1
        if time.perf_counter() - t0 > seconds:
            break
    el = time.perf_counter() - t0
    if lim is not None:
        lim.unregister() if hasattr(lim, "unregister") else None
    return done, el


def bench_reference(args):
    from paper_1406_7042_b200.dist import init
    rank, world, _ = init(backend="gloo")
    if rank != 0:
        return 0
    scn, prob, info = build_workload(args.config, args.precision)
    cells = cells_of(prob)
    per = max(1, args.ref_steps)
    tot_steps, tot_t = 0, 0.0
    for i in range(args.warmup + args.steps):
        n, el = run_oracle_sample(prob, seconds=1e9, max_steps=per)
        if i >= args.warmup:
            tot_steps += n
            tot_t += el
    val = cells * tot_steps / tot_t / 1e6
    sample = f"{per} oracle time steps per bench step of {WORKLOADS[args.config].split(':')[0]}"
    out = {"impl": "reference", "metric": METRIC, "value": val, "unit": "Mcell-updates/s",
           "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
           "ms_per_step": 1e3 * tot_t / args.steps, "higher_is_better": True, "scaling": "weak",
           "vs_baseline": None, "dtype": "f64", "data": "synthetic",
           "config": {"workload": WORKLOADS[args.config], "oracle_steps_per_step": per},
           "cpu_baseline": {"value": val, "unit": "Mcell-updates/s", "cores": 1, "kind": "oracle",
                            "sample": sample},
           "e2e": {"value": val, "unit": "Mcell-updates/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)
    return 0


METRIC = "Mcell-updates/s (coarse grid + reduced blocks) at 1 B200"


def bench_ours(args):
    import torch
    from paper_1406_7042_b200 import build as B
    from paper_1406_7042_b200.dist import barrier, finalize, init, reduce_max, reduce_sum
    from paper_1406_7042_b200.fdtd import PHASES, Sim
    B.build()
    rank, world, local = init()
    prec = args.precision
    scn, prob, info = build_workload(args.config, prec, rank)
    n_steps = int(args.time_steps or scn["n_steps"])
    cells = cells_of(prob) * int(prob.get("batch", 1))
    stream = torch.cuda.current_stream()
    sim = Sim(prob, precision=prec, probe_capacity=(args.warmup + args.steps + 2) * n_steps + 16,
              graph_steps=args.graph_steps)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
    # warm-up (W full runs)
    for _ in range(args.warmup):
        sim.step(n_steps)
    sim.sync()
    _ = sim.probe()
    torch.cuda.synchronize()
    barrier()
    torch.cuda.synchronize()
    clocks = ClockSampler(local)
    clocks.start()
    evs = []
    l0 = sim.launch_count()
    for _ in range(args.steps):
        flush.zero_()                                  # L2 flush between timed iterations
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        sim.step(n_steps)
        e1.record(stream)
        evs.append((e0, e1))
    torch.cuda.synchronize()
    barrier()
    torch.cuda.synchronize()
    clk = clocks.stop()
    launches = sim.launch_count() - l0
    ms = sum(a.elapsed_time(b) for a, b in evs)
    ms_max = reduce_max(ms)
    units = reduce_sum(float(cells) * n_steps * args.steps)
    value = units / (ms_max / 1e3) / 1e6
    sim.sync()
    _ = sim.probe()
    # per-kernel device times (eager launches with CUDA events on the same stream)
    prof_steps = min(n_steps, args.profile_steps)
    sim.profile(True)
    sim.step(prof_steps)
    sim.sync()
    ph = sim.phase_times()
    sim.profile(False)
    _ = sim.probe()
    stencil_ms = ph["stencil"] / max(ph["steps"], 1)
    grid_ms = ph["reduced_grid"] / max(ph["steps"], 1)
    step_ms_prof = sum(ph[p] for p in PHASES) / max(ph["steps"], 1)
    peak, peak_kind = _peaks()
    bpc = algorithmic_bytes_per_cell(prob, prec)
    alg_bytes = bpc * cells_of(prob) * int(prob.get("batch", 1))
    achieved = alg_bytes / (stencil_ms * 1e-3) / 1e9
    paths = sim.path()
    persistent = "persistent2d" in paths
    # leap-frog reduced blocks (config 4): the HBM-streamed matrices per step
    # (K~' and K~'^T once each, S_E twice: y = S_E h~ and S_E^T G) + the states
    w = 4 if prec == 32 else 8
    grid_bytes = 0
    red_flops = 0.0
    for b in prob.get("blocks") or []:
        qe = int(b.get("qe", b.get("q"))); qh = int(b.get("qh", b.get("q")))
        nif = int(np.asarray(b["S_E"]).size // qh)
        Nb = int(b["n_inst"]) * int(prob.get("batch", 1))
        grid_bytes += w * (2 * qe * qh + 2 * nif * qh + 4 * (qe + qh + nif) * Nb)
        # 4 (q_e q_h + n_if q_h) flops per column per step (each
        # of K~', S_E applied twice, multiply + add)
        red_flops += 4.0 * (qe * qh + nif * qh) * Nb
    grid_kernel = None
    if grid_ms > 0:
        kname = ("reduced leap-frog products (a4+a6): split-K TN GEMMs for K~' h~, K~'^T e~, S_E^T G; "
                 "y = S_E h~ on tcgen05 (3xTF32)" if "tc_gemm" in sim.path() else
                 "reduced leap-frog products (a4+a6): GEMV / SIMT GEMM kernels")
        ach = grid_bytes / (grid_ms * 1e-3) / 1e9
        grid_kernel = {"kernel": kname, "bound": "hbm", "algorithmic_bytes_per_step": grid_bytes, "avg_ms": grid_ms,
                       "achieved": ach, "peak": peak, "frac": ach / peak,
                       "gflops": red_flops / (grid_ms * 1e-3) / 1e9,
                       "note": "eager per-step launches with CUDA events (includes launch gaps)"}
    traffic = None
    tf = os.path.join(ROOT, "profiles", "stencil_traffic.json")
    if os.path.exists(tf):
        try:
            with open(tf) as f:
                tj = json.load(f)
            traffic = tj.get(f"config{args.config}_fp{prec}" + ("_persistent" if persistent else ""))
        except Exception:
            traffic = None
    # end to end through the public API with host buffers
    e2e = None
    if not args.no_e2e:
        comps = (0, 1, 2, 3, 4, 5) if prob["dim"] == 3 else (2, 3, 4)
        host_state = {c: np.zeros((sim.B, sim.S)) for c in comps}
        wsize = 4 if prec == 32 else 8
        h2d = len(comps) * sim.S * sim.B * wsize
        e2e_ms = 0.0
        d2h = 0
        # one untimed end-to-end warm-up (first-use allocations of the upload path)
        for c in comps:
            sim.set_state(c, host_state[c])
        sim.step(min(n_steps, 32))
        _ = sim.probe()
        for _ in range(max(1, args.e2e_steps)):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            for c in comps:
                sim.set_state(c, host_state[c])
            sim.step(n_steps)
            series = sim.probe()
            t1 = time.perf_counter()
            e2e_ms += (t1 - t0) * 1e3
            d2h = series.size * wsize
        e2e_ms /= max(1, args.e2e_steps)
        e2e_ms = reduce_max(e2e_ms)
        e2e = {"value": float(cells) * n_steps * world / (e2e_ms / 1e3) / 1e6, "unit": "Mcell-updates/s",
               "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h), "ms_per_step": e2e_ms}
    sim.close()
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu and args.config == 4:
        cpu = {"value": None, "unit": "Mcell-updates/s", "cores": 1, "kind": "oracle",
               "sample": "unavailable: the oracle's matrix form of config 4 (8.5 M cells + a 65,024 x 1,024 "
                         "coupling block) exceeds host memory; parity uses oracle.problem_step."
                         "sampled_hybrid_step"}
    elif rank == 0 and world == 1 and not args.no_cpu:
        ns, el = run_oracle_sample(prob, seconds=args.cpu_seconds)
        cpu = {"value": cells_of(prob) * ns / el / 1e6, "unit": "Mcell-updates/s", "cores": 1,
               "kind": "oracle",
               "sample": f"{ns} time steps of the same workload in {el:.1f} s (SciPy CSR SpMV, 1 thread)"}
    red_ms = ph["reduced"] / max(ph["steps"], 1)
    reduced_fused = None
    if red_ms > 0 and grid_ms == 0 and red_flops > 0:
        # fused blocks: the whole reduced update of a step (one GEMV / GEMM phase)
        reduced_fused = {"kernel": "fused reduced update (reduced_fused_kernel / reduced_gemm_kernel)",
                         "algorithmic_gflop_per_step": red_flops / 1e9, "avg_ms": red_ms,
                         "gflops": red_flops / (red_ms * 1e-3) / 1e9,
                         "note": "eager per-step launch with CUDA events; FMA roofline: SIMT fp32"}
    per_step = {"phase_ms_per_step": {p: ph[p] / max(ph["steps"], 1) for p in PHASES}, "reduced_grid": grid_kernel,
                "reduced_fused": reduced_fused}
    if persistent:
        # the timed path is ONE persistent launch per bench step (n_steps time
        # steps, state resident in shared memory): algorithmic bytes = what a
        # streaming step moves (state read + write) x n_steps; DRAM traffic of
        # the launch (ncu) is ~ the state once in and once out
        launch_ms = ms_max / args.steps
        alg_launch = alg_bytes * n_steps
        ach = alg_launch / (launch_ms * 1e-3) / 1e9
        roof = {"bound": "hbm", "achieved": ach, "peak": peak, "unit": "GB/s", "frac": ach / peak,
                "traffic": traffic, "kernel": "persist2d (tiles resident in shared memory, whole run per launch)",
                "algorithmic_bytes_per_launch": alg_launch, "avg_launch_ms": launch_ms, "share_of_step": 1.0,
                "peak_kind": peak_kind, "paths": paths,
                "per_step_kernels_eager_profile": dict(per_step, stencil_achieved_gbs=achieved)}
    else:
        roof = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                "frac": achieved / peak, "traffic": traffic,
                "kernel": "stencil2d (fused E->H)" if prob["dim"] == 2 else "stencil3d (fused E->H)",
                "algorithmic_bytes_per_launch": alg_bytes, "avg_launch_ms": stencil_ms,
                "share_of_step": stencil_ms / step_ms_prof if step_ms_prof else None,
                "peak_kind": peak_kind, "paths": paths, **per_step}
    if rank == 0:
        out = {"metric": METRIC, "value": value, "unit": "Mcell-updates/s", "n_gpus": world,
               "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_max / args.steps,
               "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
               "dtype": "f32" if prec == 32 else "f64",
               "data": "synthetic (seeded, SURVEY §8(d) recipe)",
               "config": {"workload": WORKLOADS[args.config], "time_steps_per_step": n_steps,
                          "cells": cells_of(prob), "q": [b["q"] for b in prob.get("blocks") or []],
                          "parallelism": f"replicas x{world}",
                          "l2": ("flushed (256 MB write) between timed steps; state resident in shared "
                                 "memory for the whole launch" if persistent else
                                 "flushed (256 MB write) between timed steps; the state is L2-resident "
                                 "within a step when it fits (126 MB L2)")},
               "roofline": roof,
               "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": int(launches), "clocks": clk,
               "prep": {k: v for k, v in info.items() if k in ("n_if", "alpha", "coarse_sigma", "coarse_limit")}}
        print(json.dumps(out), flush=True)
    finalize()
    return 0


def main(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=("ours", "reference"))
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--precision", type=int, default=None)
    ap.add_argument("--graph-steps", type=int, default=32)
    ap.add_argument("--profile-steps", type=int, default=2000)
    ap.add_argument("--e2e-steps", type=int, default=2)
    ap.add_argument("--cpu-seconds", type=float, default=15.0)
    ap.add_argument("--ref-steps", type=int, default=20)
    ap.add_argument("--time-steps", type=int, default=0, help="override the workload's time steps per bench step")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    args = ap.parse_args(argv)
    if args.precision is None:
        args.precision = 32 if args.config in (2, 3, 4, 5) else 64
    if args.impl == "reference":
        return bench_reference(args)
    return bench_ours(args)


if __name__ == "__main__":
    sys.exit(main())
