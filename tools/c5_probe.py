#!/usr/bin/env python
"""Where does config 5's step go?  Times fdtd_step on variants of the config-5
domain (400 x 200 x 40 cells, fp32) through the C ABI, one variant per process
(the environment selects the kernel shape):

  vac     the same domain as a vacuum cavity (uniform coefficients, no blocks)
  tab     config 5's material table and PEC plates, no reduced blocks / rows
  full    config 5 as benchmarked

    python tools/c5_probe.py                # the sweep (spawns itself)
    python tools/c5_probe.py --one full     # one variant in this process
"""
import json
import os
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def one(kind, steps=2000):
    import numpy as np
    import torch
    from paper_1406_7042_b200 import fdtd, prep
    from synth import scenario
    if os.environ.get("FDTD_LIB"):
        fdtd.load_library(os.path.join(ROOT, "paper_1406_7042_b200", os.environ["FDTD_LIB"]))
    from synth.scenarios import cavity3d_random
    if kind in ("vac", "vactab", "vaczero"):
        scn = cavity3d_random("c5vac", 55, 400, 200, 40, 0.25e-3, 0.6, 100, 32)
        prob, _ = prep.build_problem(scn, precision=32, cache=False)
        if kind == "vactab":       # the same vacuum problem through the material-table kernel
            S = 401 * 201 * 41
            prob = dict(prob, mat_id=np.zeros(S, np.uint8), mat_coef=np.asarray(prob["uniform_coef"], float)[None, :],
                        mat_ifmask=np.zeros(1, np.uint8))
        if kind == "vaczero":
            prob = dict(prob, init={})
    else:
        prob, _ = prep.build_problem(scenario(5), precision=32)
        if kind == "tab":
            prob = dict(prob)
            prob["blocks"] = []
            prob["interface"] = None
            prob["mat_ifmask"] = np.zeros_like(np.asarray(prob["mat_ifmask"]))
            prob["probes"] = [p for p in prob["probes"] if int(p["kind"]) == 0]
        if kind == "tabrand":      # config 5's tables, no blocks, random initial field
            prob = dict(prob)
            prob["blocks"] = []
            prob["interface"] = None
            prob["mat_ifmask"] = np.zeros_like(np.asarray(prob["mat_ifmask"]))
            prob["probes"] = [p for p in prob["probes"] if int(p["kind"]) == 0]
            rng = np.random.default_rng(3)
            prob["init"] = {c: rng.uniform(-1, 1, (1, 401 * 201 * 41)) for c in range(3)}
    sim = fdtd.Sim(prob, precision=32, check_every=0)
    sim.step(256); sim.sync()
    best = 1e9
    for _ in range(3):
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(); sim.step(steps); e1.record(); torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1) / steps * 1e3)
    sim.profile(True); sim.step(64); sim.sync(); ph = sim.phase_times(); sim.profile(False)
    cells = 400 * 200 * 40
    print(json.dumps(dict(kind=kind, us_per_step=round(best, 2), gcell=round(cells / best / 1e3, 1),
                          hbm_frac=round(cells * 49 / (best * 1e-6) / 6456.8e9, 3), path=sim.path(),
                          phase_us={k: round(1e3 * v / max(1, ph['steps']), 2) for k, v in ph.items() if k != 'steps'},
                          env={k: v for k, v in os.environ.items() if k.startswith("FDTD_")})), flush=True)


def main():
    if "--one" in sys.argv:
        one(sys.argv[sys.argv.index("--one") + 1])
        return
    envs = [{}]
    for spec in sys.argv[1:]:
        envs.append(dict(kv.split("=") for kv in spec.split(";") if kv))
    for env in envs:
        for kind in (os.environ.get("C5_KINDS") or "vac,tab,full").split(","):
            e = dict(os.environ); e.update(env)
            t = time.time()
            r = subprocess.run([sys.executable, __file__, "--one", kind], env=e, capture_output=True, text=True,
                               timeout=600)
            line = [l for l in r.stdout.splitlines() if l.startswith("{")]
            print(line[-1] if line else f"FAILED {kind} {env}: {r.stderr[-400:]}", flush=True)


if __name__ == "__main__":
    main()
