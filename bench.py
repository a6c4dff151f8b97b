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
    "lossy256": "lossy256 (SURVEY NEXT-2): config 3's 256^3 grid with 5-cell 4th-order matched absorbers on the x and y "
                "ends and a lossy dielectric slab (eps_r 2.5, 0.02 S/m), Ez point source, dt = 0.95 CFL, 1000 steps, fp32",
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


class OracleStepper:
    """The CPU oracle (oracle.problem_step: SciPy CSR SpMV, single-threaded)
    stepping batch member 0 of a workload; assembly once, then timed steps."""

    def __init__(self, prob):
        from oracle import problem_step as ps
        t0 = time.perf_counter()
        self.rec = ps.build(prob)
        self.t_build = time.perf_counter() - t0
        self.E, self.H = ps.initial_state(self.rec, prob, 0)
        self.PE, self.PH = ps.probe_matrices(self.rec)
        self.step_no = 0

    def run(self, max_steps, seconds=1e9):
        from oracle.matrix_form import step_leapfrog
        try:
            from threadpoolctl import threadpool_limits
            lim = threadpool_limits(limits=1)
        except Exception:
            lim = None
        rec = self.rec
        done, t0 = 0, time.perf_counter()
        while done < max_steps:
            su = None
            if len(rec.src_row) and self.step_no < rec.wave.shape[0]:
                su = np.zeros(len(self.E))
                np.add.at(su, rec.src_row, -rec.src_coef * rec.wave[self.step_no, rec.src_col, 0])
            self.E, self.H = step_leapfrog(self.E, self.H, rec.GE, rec.GH, rec.KE, rec.KH, su_E=su)
            _ = self.PE @ self.E + self.PH @ self.H
            done += 1
            self.step_no += 1
            if time.perf_counter() - t0 > seconds:
                break
        el = time.perf_counter() - t0
        if lim is not None and hasattr(lim, "unregister"):
            lim.unregister()
        return done, el


def run_oracle_sample(prob, seconds=15.0, max_steps=800, member_cells=None):
    """Time the oracle on a bounded number of steps of the same workload.
    Returns (steps, seconds, assembly seconds)."""
    st = OracleStepper(prob)
    st.run(2)                                   # warm-up (first-touch of the matrices)
    done, el = st.run(max_steps, seconds)
    return done, el, st.t_build


def bench_reference(args):
    from paper_1406_7042_b200.dist import init
    rank, world, _ = init(backend="gloo")
    if rank != 0:
        return 0
    scn, prob, info = build_workload(args.config, args.precision)
    cells = cells_of(prob)
    per = max(1, args.ref_steps)
    st = OracleStepper(prob)
    tot_steps, tot_t = 0, 0.0
    for i in range(args.warmup + args.steps):
        n, el = st.run(per)
        if i >= args.warmup:
            tot_steps += n
            tot_t += el
    val = cells * tot_steps / tot_t / 1e6
    sample = (f"{per} oracle time steps (batch member 0) per bench step of {WORKLOADS[args.config].split(':')[0]}; "
              f"matrix assembly {st.t_build:.0f} s not timed")
    out = {"impl": "reference", "metric": METRIC, "value": val, "unit": "Mcell-updates/s",
           "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
           "ms_per_step": 1e3 * tot_t / args.steps, "higher_is_better": True, "scaling": "weak",
           "vs_baseline": None, "dtype": "f64", "data": "synthetic",
           "config": {"workload": WORKLOADS[args.config], "oracle_steps_per_step": per},
           "cpu_baseline": {"value": val, "unit": "Mcell-updates/s", "cores": 1, "kind": "oracle",
                            "sample": sample, **cpu_info()},
           "e2e": {"value": val, "unit": "Mcell-updates/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)
    return 0


METRIC = "Mcell-updates/s (coarse grid + reduced blocks) at 1 B200"


def _fp32_peak_gflops():
    """SIMT FP32 FMA peak: SMs x 128 lanes x 2 flop x max SM clock."""
    import torch
    pr = torch.cuda.get_device_properties(0)
    mhz = 1965.0
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            mhz = float(json.load(f).get("sm_max_mhz", mhz))
    except Exception:
        pass
    return pr.multi_processor_count * 128 * 2 * mhz * 1e-3


def _tf32_peak_gflops():
    """Dense TF32 tensor peak: the measured bf16 figure x the nominal tf32/bf16
    ratio 1/2 (B200_PROFILING.md)."""
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["bf16_tflops"]) * 1e3 / 2
    except Exception:
        return 2250e3 / 2


def cpu_info():
    model = None
    try:
        with open("/proc/cpuinfo") as f:
            for ln in f:
                if ln.startswith("model name"):
                    model = ln.split(":", 1)[1].strip()
                    break
    except Exception:
        pass
    pools = None
    try:
        from threadpoolctl import threadpool_info
        pools = [{k: d.get(k) for k in ("internal_api", "num_threads")} for d in threadpool_info()]
    except Exception:
        pass
    return {"cpu_model": model, "os_cpu_count": os.cpu_count(), "threadpools": pools}


def measure(config, prec, steps, warmup, args, rank=0, world=1, local=0, headline=False):
    """One configuration: W warm-up runs, K timed runs of the whole workload
    (``n_steps`` time steps each, inputs resident in HBM), then the per-kernel
    profile, the end-to-end run with host buffers and the CPU oracle sample."""
    import torch
    from paper_1406_7042_b200.dist import barrier, reduce_max, reduce_sum
    from paper_1406_7042_b200.fdtd import PHASES, Sim
    scn, prob, info = build_workload(config, prec, rank)
    n_steps = int(args.time_steps or scn["n_steps"])
    cells = cells_of(prob) * int(prob.get("batch", 1))
    stream = torch.cuda.current_stream()
    sim = Sim(prob, precision=prec, probe_capacity=(warmup + steps + 2) * n_steps + 16,
              graph_steps=args.graph_steps)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
    for _ in range(warmup):
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
    for _ in range(steps):
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
    units = reduce_sum(float(cells) * n_steps * steps)
    value = units / (ms_max / 1e3) / 1e6
    sim.sync()
    _ = sim.probe()
    # per-kernel device times: eager launches with CUDA events on the launching
    # stream (the same kernels the graphs replay)
    prof_steps = min(n_steps, args.profile_steps)
    sim.profile(True)
    sim.step(prof_steps)
    sim.sync()
    ph = sim.phase_times()
    sim.profile(False)
    _ = sim.probe()
    nph = max(ph["steps"], 1)
    stencil_ms = ph["stencil"] / nph
    grid_ms = ph["reduced_grid"] / nph
    red_ms = ph["reduced"] / nph
    step_ms_prof = sum(ph[p] for p in PHASES) / nph
    peak, peak_kind = _peaks()
    bpc = algorithmic_bytes_per_cell(prob, prec)
    alg_bytes = bpc * cells
    paths = sim.path()
    persistent = "persistent2d" in paths
    w = 4 if prec == 32 else 8
    # reduced blocks: algorithmic bytes (K~' and S_E each read twice) and flops
    # (4 (q_e q_h + n_if q_h) per column per step)
    red_bytes, red_flops = 0, 0.0
    for b in prob.get("blocks") or []:
        qe = int(b.get("qe", b.get("q"))); qh = int(b.get("qh", b.get("q")))
        nif = int(np.asarray(b["S_E"]).size // qh)
        Nb = int(b["n_inst"]) * int(prob.get("batch", 1))
        red_bytes += w * (2 * qe * qh + 2 * nif * qh + 4 * (qe + qh + nif) * Nb)
        red_flops += 4.0 * (qe * qh + nif * qh) * Nb
    fp32_peak = _fp32_peak_gflops()
    reduced = None
    if red_flops > 0:
        step_ms = ms_max / steps / n_steps
        if persistent:
            # the reduced CTAs of the persistent kernel: their rows of M stay in
            # shared memory for the whole launch; their throughput is the
            # step's (they run beside the tiles), bounded by the exchange chain
            gf = red_flops / (step_ms * 1e-3) / 1e9
            reduced = {"kernel": "persist2d reduced CTAs (fused M rows resident in shared memory)",
                       "bound": "latency (G -> reduced CTAs -> y chain per step)", "gflops": gf,
                       "roofline_gflops": fp32_peak, "frac": gf / fp32_peak,
                       "algorithmic_gflop_per_step": red_flops / 1e9,
                       "note": "flops per time step / measured ms per time step of the timed launch"}
        elif grid_ms > 0:
            # leap-frog blocks streamed from HBM (config 4): AI = 8 flop/B
            ai = red_flops / red_bytes
            roof = min(ai * peak, _tf32_peak_gflops() if "tc_gemm" in paths else fp32_peak)
            gf = red_flops / (grid_ms * 1e-3) / 1e9
            ach = red_bytes / (grid_ms * 1e-3) / 1e9
            reduced = {"kernel": ("leap-frog reduced products (a4+a6): split-K TN GEMMs K~' h~, K~'^T e~, "
                                  "S_E^T G; y = S_E h~ on tcgen05 (3xTF32)" if "tc_gemm" in paths else
                                  "leap-frog reduced products (a4+a6): GEMV / SIMT GEMM kernels"),
                       "bound": "hbm", "avg_ms": grid_ms, "algorithmic_bytes_per_step": red_bytes,
                       "achieved_gbs": ach, "hbm_frac": ach / peak, "gflops": gf,
                       "roofline_gflops": roof, "frac": gf / roof,
                       "note": "eager launches on a busy stream, CUDA events around each kernel group read back every 64 steps"}
        elif red_ms > 0:
            gf = red_flops / (red_ms * 1e-3) / 1e9
            reduced = {"kernel": "fused reduced update (reduced_fused_kernel / reduced_gemm_kernel)",
                       "bound": "latency (L2-resident M, one GEMM phase per step)", "avg_ms": red_ms,
                       "gflops": gf, "roofline_gflops": fp32_peak, "frac": gf / fp32_peak,
                       "algorithmic_gflop_per_step": red_flops / 1e9,
                       "note": "eager launches on a busy stream, CUDA events read back every 64 steps; SIMT fp32 FMA roofline"}
    traffic = None
    tf = os.path.join(ROOT, "profiles", "stencil_traffic.json")
    if os.path.exists(tf):
        try:
            with open(tf) as f:
                tj = json.load(f)
            traffic = tj.get(f"config{config}_fp{prec}" + ("_persistent" if persistent else ""))
        except Exception:
            traffic = None
    e2e = None
    if not args.no_e2e:
        comps = (0, 1, 2, 3, 4, 5) if prob["dim"] == 3 else (2, 3, 4)
        host_state = {c: np.zeros((sim.B, sim.S)) for c in comps}
        # fdtd_set_state takes fp64 host arrays (fdtd.h): those are the bytes copied
        h2d = sum(host_state[c].nbytes for c in comps)
        e2e_ms, d2h = 0.0, 0
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
            d2h = series.nbytes
        e2e_ms /= max(1, args.e2e_steps)
        e2e_ms = reduce_max(e2e_ms)
        e2e = {"value": float(cells) * n_steps * world / (e2e_ms / 1e3) / 1e6, "unit": "Mcell-updates/s",
               "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h), "ms_per_step": e2e_ms,
               "note": "fdtd_set_state of every coarse component from fp64 host arrays, fdtd_step, "
                       "fdtd_probe (fp64 series) per bench step"}
    sim.close()
    del flush
    torch.cuda.empty_cache()
    cpu = None          # filled in by bench_ours from the oracle worker processes
    per_step = {"phase_ms_per_step": {p: ph[p] / nph for p in PHASES}}
    if persistent:
        # ONE persistent launch per bench step (n_steps time steps, state
        # resident in shared memory): algorithmic bytes = what a streaming step
        # moves (state read + write) x n_steps; the launch's DRAM traffic is
        # ~ the state once in and once out
        launch_ms = ms_max / steps
        alg_launch = alg_bytes * n_steps
        ach = alg_launch / (launch_ms * 1e-3) / 1e9
        roof = {"bound": "hbm", "achieved": ach, "peak": peak, "unit": "GB/s", "frac": ach / peak,
                "traffic": traffic, "kernel": "persist2d_kernel (tiles resident in shared memory, whole run "
                                              "per launch; HBM-equivalent effective bandwidth, SURVEY §8(d))",
                "algorithmic_bytes_per_launch": alg_launch, "avg_launch_ms": launch_ms, "share_of_step": 1.0,
                "peak_kind": peak_kind, "paths": paths,
                "per_step_kernels_eager_profile": dict(per_step, stencil_achieved_gbs=alg_bytes / (stencil_ms * 1e-3) / 1e9)}
    else:
        achieved = alg_bytes / (stencil_ms * 1e-3) / 1e9
        roof = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                "frac": achieved / peak, "traffic": traffic,
                "kernel": "stencil2d (fused E->H)" if prob["dim"] == 2 else "stencil3d_tile_kernel (fused E->H)",
                "algorithmic_bytes_per_launch": alg_bytes, "avg_launch_ms": stencil_ms,
                "share_of_step": stencil_ms / step_ms_prof if step_ms_prof else None,
                "peak_kind": peak_kind, "paths": paths, **per_step}
    out = {"value": value, "ms_per_step": ms_max / steps, "steps": steps, "warmup": warmup,
           "dtype": "f32" if prec == 32 else "f64",
           "config": {"workload": WORKLOADS[config], "time_steps_per_step": n_steps, "cells": cells_of(prob),
                      "batch": int(prob.get("batch", 1)), "q": [b["q"] for b in prob.get("blocks") or []],
                      "l2": ("flushed (256 MB write) between timed steps; state resident in shared memory for "
                             "the whole launch" if persistent else
                             "flushed (256 MB write) between timed steps")},
           "roofline": roof, "reduced_block": reduced, "cpu_baseline": cpu, "e2e": e2e,
           "gpu_launches": int(launches), "clocks": clk,
           "prep": {k: v for k, v in info.items() if k in ("n_if", "alpha", "coarse_sigma", "coarse_limit")}}
    return out


METRIC_CONFIGS = {"config2_fp32": (2, 32), "config3_fp32": (3, 32), "config3_fp64": (3, 64),
                  "config5_fp32": (5, 32), "lossy256_fp32": ("lossy256", 32)}


def measure_rom(args, batch, steps=5, warmup=3, cpu=True, dmma_peak=None):
    """the paper's 2-D cavity reduced to order 80 (Table I),
    stepped for the physical time of its 10,000 steps at s = 4.95, batched over
    ``batch`` excitation waveforms (rom_* calls, csrc/rom.cu).  Reported beside the
    hybrid configurations: column-steps/s, GFLOP/s of the two dense products
    against the measured fp64 tensor-core peak, the oracle timed on the host."""
    import torch
    from paper_1406_7042_b200 import rom as R
    from paper_1406_7042_b200.prep import rom as prom
    from synth import scenario
    scn = scenario("rom2d", batch=batch)
    t0 = time.time()
    model, info = prom.build_rom(scn)
    t_prep = time.time() - t0
    n = int(scn["n_steps"])
    q = int(model["q_e"])
    sim = R.Rom(model, model["amp"], model["wave"])
    geo = sim.info()
    for _ in range(max(3, warmup)):
        sim.step(n); sim.probe()
    ms = []
    for _ in range(steps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); sim.step(n); e1.record(); torch.cuda.synchronize()
        ms.append(e0.elapsed_time(e1))
        sim.probe()
    t = sum(ms) / len(ms)
    colsteps = batch * n / (t * 1e-3)
    gflops = 4.0 * q * q * batch * n / (t * 1e-3) / 1e9
    peak = dmma_peak if dmma_peak is not None else R.dmma_peak_tflops()
    # end to end: create (uploads K~', B~, the waveforms), all steps, the probe series back on the host
    te = []
    for _ in range(2):
        torch.cuda.synchronize(); w0 = time.perf_counter()
        s2 = R.Rom(model, model["amp"], model["wave"]); s2.step(n); pr = s2.probe(); s2.close()
        te.append(time.perf_counter() - w0)
    e2e_t = min(te)
    out = {"value": colsteps, "unit": "reduced-model column-steps/s", "ms_per_step": t, "steps": steps, "dtype": "f64",
           "config": {"workload": (f"rom2d: whole-domain reduced model of the 2-D PEC cavity of Table I (101 x 101 cells of "
                                   f"1 cm, N = {info['Ne'] + info['Nh']}), order q = {q}, 5 expansion points, s = "
                                   f"{scn['s_factor']} ({info['clipped']} singular values clipped), {batch} excitation "
                                   f"waveforms, {n} time steps per bench step"),
                      "time_steps_per_step": n, "batch": batch, "q": [q], "launch": geo, "prep_s": round(t_prep, 1),
                      "l2": "state and K~' resident on chip for the whole launch (no HBM traffic in steady state)"},
           "roofline": {"bound": "tensor", "achieved": gflops / 1e3, "peak": peak, "unit": "TFLOP/s",
                        "frac": gflops / 1e3 / peak if peak and peak > 0 else None, "traffic": None,
                        "kernel": "rom_persist_kernel (mma.sync m8n8k4 f64, K~' in registers)",
                        "algorithmic_flops_per_launch": 4.0 * q * q * batch * n,
                        "peak_kind": "measured here: register-only mma.sync m8n8k4 f64 loop on every SM "
                                     "(rom_dmma_peak_tflops; fp64 is not in MEASURED_PEAKS.json)"},
           "us_per_time_step": t * 1e3 / n,
           "e2e": {"value": batch * n / e2e_t, "unit": "reduced-model column-steps/s",
                   "h2d_bytes_per_step": int(8 * (model["wave"].size + model["amp"].size + 3 * q * q)),
                   "d2h_bytes_per_step": int(pr.size * 8), "ms_per_step": e2e_t * 1e3,
                   "note": "rom_create (uploads), rom_step, rom_probe (fp64 series to the host) per bench step"},
           "gpu_launches": steps}
    sim.close()
    if cpu:
        from oracle import rom as orom
        nb = min(batch, 64)
        w0 = time.perf_counter()
        orom.run(model, model["amp"][:, :nb], model["wave"][:, :nb], n)
        el = time.perf_counter() - w0
        out["cpu_baseline"] = {"value": nb * n / el, "unit": "reduced-model column-steps/s", "cores": 1, "kind": "oracle",
                               "sample": f"oracle.rom.run: {n} steps x {nb} columns of the same model in {el:.1f} s "
                                         f"(NumPy/LAPACK Cholesky solves and matmuls)", **cpu_info()}
    return out


def measure_mor(args, config=2):
    """the Krylov basis of one refined region of ``config`` on
    the device (mor_* calls, csrc/mor.cu: block Schur + batched CGS at the
    paper's 1e-4, block Gram-Schmidt), timed through the public binding with
    host buffers (uploads and the basis download included).  The host
    preprocessing's time for the same basis is in profiles/r02/mor_bench.txt
    (tools/mor_bench.py --host; too long for the default bench)."""
    import torch
    sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "tools"))
    from mor_bench import region_system
    from paper_1406_7042_b200 import mor as M
    from synth import scenario
    scn = scenario(config)
    part, Bm, pts, q = region_system(scn)
    Ne, Nh = part.Kff.shape
    m = M.Mor(part.De_f, part.Dm_f, part.Kff, scn["dt"])
    ts = []
    for _ in range(3):
        torch.cuda.synchronize(); w0 = time.perf_counter()
        V1, V2, st = m.krylov_basis(Bm, np.arange(Ne), np.arange(Nh), q, pts, solve_tol=1e-4)
        ts.append(time.perf_counter() - w0)
    launches = m.launch_count() // 3
    m.close()
    t = min(ts[1:])
    # algorithmic traffic of one CGS iteration and column (complex fp64 unless the point is real): two Schur
    # applications (K^T: read x, write t; K: read t, x, write v) and the recursion's vector updates and dots
    cplx = sum(1 for z in pts if complex(z).imag != 0)
    el = 16.0 * cplx / len(pts) + 8.0 * (len(pts) - cplx) / len(pts)
    # (CSR values and indices once per iteration of the whole block of columns)
    per_it = el * (2 * (2 * Nh + 3 * Ne) + 17 * Ne)
    csr = 2 * (2 * 12.0 * part.Kff.nnz + 8.0 * (Ne + Nh))
    bytes_cgs = per_it * st["cgs_iterations"] + csr * st["cgs_iterations"] / Bm.shape[1]
    hbm, hbm_kind = _peaks()
    return {"value": t, "unit": "s per reduction (Krylov basis of the region, host buffers in / basis out)",
            "higher_is_better": False, "dtype": "f64",
            "config": {"workload": (f"config{config} region: K_ff {Ne} x {Nh} ({part.Kff.nnz} entries), {len(pts)} expansion "
                                    f"points, block of {Bm.shape[1]}, q = {q}, CGS to 1e-4 (P:371)")},
            "stats": st, "gpu_launches": launches,
            "roofline": {"bound": "hbm", "achieved": bytes_cgs / st["t_solve"] / 1e9 if st["t_solve"] > 0 else None,
                         "peak": hbm, "peak_kind": hbm_kind, "unit": "GB/s",
                         "frac": (bytes_cgs / st["t_solve"] / 1e9 / hbm) if st["t_solve"] > 0 else None,
                         "traffic": None, "kernel": "batched CGS (spmm_kernel, cgs_v*, dot_partial_kernel)",
                         "note": "13 kernels per CGS iteration of the column block, 4 iterations replayed as one "
                                 f"CUDA graph; the solves' share of the reduction: {st['t_solve']:.2f} s of {t:.2f} s"},
            "orth_err": [float(np.abs(V1.T @ V1 - np.eye(q)).max()), float(np.abs(V2.T @ V2 - np.eye(q)).max())]}


def oracle_sample_worker(config, prec, seconds):
    """CPU-oracle timing of one workload in its own process (single-threaded
    SciPy), run beside the GPU measurements so the bench stays within minutes.
    Returns the cpu_baseline dict."""
    try:
        from threadpoolctl import threadpool_limits
        threadpool_limits(limits=1)
    except Exception:
        pass
    try:
        _, prob, _ = build_workload(config, prec)
        ns, el, t_build = run_oracle_sample(prob, seconds=seconds)
        return {"value": cells_of(prob) * ns / el / 1e6, "unit": "Mcell-updates/s", "cores": 1, "kind": "oracle",
                "sample": (f"{ns} time steps of batch member 0 of the same workload in {el:.1f} s "
                           f"(oracle.problem_step, SciPy CSR SpMV, 1 thread, in a worker process beside the GPU "
                           f"run; matrix assembly {t_build:.0f} s not timed)" +
                           ("; per-member rate (the batch's members are independent)"
                            if int(prob.get("batch", 1)) > 1 else "")),
                **cpu_info()}
    except MemoryError as ex:
        return {"value": None, "unit": "Mcell-updates/s", "cores": 1, "kind": "oracle",
                "sample": f"unavailable: {ex}", **cpu_info()}


def bench_ours(args):
    from paper_1406_7042_b200 import build as B
    from paper_1406_7042_b200.dist import finalize, init
    B.build()
    rank, world, local = init()
    futs, pool = {}, None
    if rank == 0 and world == 1 and not args.no_cpu:
        # the oracle samples in worker processes (spawned before CUDA work),
        # one per distinct oracle problem (config 3's fp32 and fp64 lines share
        # the fp64 oracle run of the same problem)
        import concurrent.futures as cf
        import multiprocessing as mp
        jobs = {args.config: (args.config, args.precision)}
        if args.per_config:
            for name, (c, p) in METRIC_CONFIGS.items():
                jobs.setdefault(c, (c, p))
        pool = cf.ProcessPoolExecutor(max_workers=len(jobs), mp_context=mp.get_context("spawn"))
        futs = {c: pool.submit(oracle_sample_worker, c, p, args.cpu_seconds) for c, (c_, p) in jobs.items()}
    head = measure(args.config, args.precision, args.steps, args.warmup, args, rank, world, local, headline=True)
    per = {}
    if args.per_config and world == 1:
        for name, (c, p) in METRIC_CONFIGS.items():
            if c == args.config and p == args.precision:
                continue
            try:
                per[name] = measure(c, p, args.per_config_steps, max(3, args.per_config_warmup), args,
                                    rank, world, local)
            except Exception as ex:       # report, never hide: the headline line still prints
                per[name] = {"error": f"{type(ex).__name__}: {ex}"}
    if args.per_config and world == 1 and rank == 0:
        try:
            from paper_1406_7042_b200 import rom as R
            pk = R.dmma_peak_tflops()
            per["rom2d_fp64_b64"] = measure_rom(args, 64, cpu=not args.no_cpu, dmma_peak=pk)
            per["rom2d_fp64_b9472"] = measure_rom(args, 9472, cpu=False, dmma_peak=pk)
        except Exception as ex:
            per["rom2d_fp64_b64"] = {"error": f"{type(ex).__name__}: {ex}"}
        try:
            per["mor_config2_region"] = measure_mor(args, 2)
        except Exception as ex:
            per["mor_config2_region"] = {"error": f"{type(ex).__name__}: {ex}"}
    if futs:
        for c, f in futs.items():
            try:
                res = f.result(timeout=1800)
            except Exception as ex:
                res = {"value": None, "kind": "oracle", "cores": 1, "sample": f"failed: {type(ex).__name__}: {ex}"}
            if c == args.config:
                head["cpu_baseline"] = res
            for name, v in per.items():
                if isinstance(v, dict) and name in METRIC_CONFIGS and METRIC_CONFIGS[name][0] == c:
                    v["cpu_baseline"] = res
        pool.shutdown()
    if rank == 0:
        cfg = dict(head["config"])
        cfg.update(parallelism=f"replicas x{world}")
        out = {"metric": METRIC, "value": head["value"], "unit": "Mcell-updates/s", "n_gpus": world,
               "steps": args.steps, "warmup": args.warmup, "ms_per_step": head["ms_per_step"],
               "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
               "dtype": head["dtype"], "data": "synthetic (seeded, SURVEY §8(d) recipe)",
               "config": cfg, "roofline": head["roofline"], "reduced_block": head["reduced_block"],
               "cpu_baseline": head["cpu_baseline"], "e2e": head["e2e"], "gpu_launches": head["gpu_launches"],
               "clocks": head["clocks"], "prep": head["prep"]}
        if per:
            out["per_config"] = per
        print(json.dumps(out), flush=True)
    finalize()
    return 0


def main(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=("ours", "reference"))
    ap.add_argument("--config", type=int, default=4)
    ap.add_argument("--precision", type=int, default=None)
    ap.add_argument("--graph-steps", type=int, default=32)
    ap.add_argument("--profile-steps", type=int, default=2000)
    ap.add_argument("--e2e-steps", type=int, default=2)
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    ap.add_argument("--ref-steps", type=int, default=20)
    ap.add_argument("--time-steps", type=int, default=0, help="override the workload's time steps per bench step")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-per-config", dest="per_config", action="store_false",
                    help="only the headline configuration (default: also configs 2, 3 fp32/fp64, 5)")
    ap.add_argument("--per-config-steps", type=int, default=3)
    ap.add_argument("--per-config-warmup", type=int, default=3)
    ap.add_argument("--rom-only", action="store_true", help="only the NEXT-3 reduced-model lines (development)")
    args = ap.parse_args(argv)
    if args.precision is None:
        args.precision = 32 if args.config in (2, 3, 4, 5) else 64
    if args.impl == "reference":
        return bench_reference(args)
    if args.rom_only:
        from paper_1406_7042_b200 import build as B
        B.build()
        for b in (64, 1184, 9472):
            print(json.dumps({f"rom2d_fp64_b{b}": measure_rom(args, b, cpu=(b == 64))}), flush=True)
        return 0
    return bench_ours(args)


if __name__ == "__main__":
    sys.exit(main())
