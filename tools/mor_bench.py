"""Offline reduction on the device (include/fdtd_mor.h) at the
sizes of the BASELINE configurations: the Krylov basis of one refined region
(recipe B: block Arnoldi on the fine-region system started at K_cf^T Omega) by
``mor.Mor.krylov_basis`` (block Schur + batched CGS at the paper's 1e-4, or the
z = 0 back substitution) against the host preprocessing
(``prep.reduce.krylov_basis``: SciPy sparse LU + NumPy Gram-Schmidt).

    python tools/mor_bench.py --config 2 [--host] [--tol 1e-4]

Prints one JSON line per run.  The host leg of config 4 takes ~25 min; without
--host the time recorded in the prep cache (info["blocks"][0]["t_basis"]) is
quoted instead when the cache holds it.
"""
import argparse
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_1406_7042_b200 import mor, prep  # noqa: E402
from paper_1406_7042_b200.prep import fit, reduce  # noqa: E402
from synth import scenario  # noqa: E402


def region_system(scn, box=0):
    dim, n, d = scn["dim"], tuple(scn["n"]), scn["delta"]
    P = fit.assemble(dim, n, d, scn["eps_r"], scn["boxes"], scn["eps0"], scn["mu0"], pec_extra=prep._pec_extra(scn))
    part = P.boxes[box]
    bas = scn.get("basis") or {}
    rng = np.random.default_rng(int(bas.get("seed", 0)) + box)
    p = int(bas.get("p", 4))
    Om = rng.standard_normal((part.Kcf.shape[0], p))
    Ne, Nh = part.Kff.shape
    B = np.vstack([np.zeros((Ne, p)), np.asarray(part.Kcf.T @ Om)])
    if bas.get("points") == "zero":
        pts = [0.0]
    else:
        pts = reduce.expansion_points(bas.get("M", 1.1), bas.get("L", 2), bas.get("fmax", 30e9), scn["dt"])
    return part, B, pts, int(scn["boxes"][box]["q"])


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="2")
    ap.add_argument("--host", action="store_true")
    ap.add_argument("--tol", type=float, default=1e-4)
    ap.add_argument("--window", type=float, default=120e9)
    ap.add_argument("--pipeline", action="store_true",
                    help="the whole preprocessing of the configuration with the device reducer "
                         "(prep.build_problem(reducer='gpu')), then a short stepped run of the result")
    a = ap.parse_args()
    cfg = int(a.config) if a.config.isdigit() else a.config
    scn = scenario(cfg)
    if a.pipeline:
        from paper_1406_7042_b200.fdtd import Sim
        t0 = time.time()
        prob, info = prep.build_problem(scn, cache=False, reducer="gpu", reducer_opts=dict(solve_tol=a.tol, window_bytes=a.window))
        t_total = time.time() - t0
        sim = Sim(prob)
        for c, arr in (prob.get("init") or {}).items():
            sim.set_state(int(c), arr)
        sim.step(1000)
        sim.sync()
        pr = sim.probe()
        sim.close()
        print(json.dumps(dict(config=cfg, pipeline="gpu reducer", t_total_s=round(t_total, 1), t_assemble_s=round(info["t_assemble"], 1),
                              blocks=[{k: (round(v, 3) if isinstance(v, float) else v) for k, v in b.items()} for b in info["blocks"]],
                              mor_stats=info.get("mor_stats"), limit=2.0 / scn["dt"],
                              probe_max_after_1000_steps=float(np.abs(pr).max()), finite=bool(np.all(np.isfinite(pr))))), flush=True)
        return
    t0 = time.time()
    part, B, pts, q = region_system(scn)
    t_asm = time.time() - t0
    Ne, Nh = part.Kff.shape
    out = dict(config=cfg, n_e=Ne, n_h=Nh, nnz=int(part.Kff.nnz), q=q, n_b=B.shape[1],
               points=[[z.real, z.imag] for z in map(complex, pts)], t_assemble_s=round(t_asm, 2))
    import torch
    torch.cuda.init()
    m = mor.Mor(part.De_f, part.Dm_f, part.Kff, scn["dt"])
    for rep in range(2):                 # the second run is the timed one (first: allocator, module load)
        torch.cuda.synchronize()
        t0 = time.time()
        V1, V2, st = m.krylov_basis(B, np.arange(Ne), np.arange(Nh), q, pts, solve_tol=a.tol, window_bytes=a.window)
        t_gpu = time.time() - t0
    out.update(gpu_s=round(t_gpu, 3), gpu_stats=st, launches=m.launch_count(),
               orth_err=[float(np.abs(V1.T @ V1 - np.eye(q)).max()), float(np.abs(V2.T @ V2 - np.eye(q)).max())])
    m.close()
    if a.host:
        t0 = time.time()
        H1, H2 = reduce.krylov_basis(part.De_f, part.Dm_f, part.Kff, scn["dt"], B, np.arange(Ne), np.arange(Nh), q, pts)
        out["host_s"] = round(time.time() - t0, 2)
        # direct solves on the host, CGS at --tol on the device: the leading part of the two Krylov spaces coincides,
        # the later blocks inherit the solver tolerance (columns of the host space reproduced to cos > 0.999)
        s1 = np.linalg.svd(H1.T @ V1, compute_uv=False)
        s2 = np.linalg.svd(H2.T @ V2, compute_uv=False)
        out["principal_cosines_above_0.999"] = [int(np.sum(s1 > 0.999)), int(np.sum(s2 > 0.999))]
        out["speedup"] = round(out["host_s"] / t_gpu, 1)
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
