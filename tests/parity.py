"""Parity helpers shared by the GPU tests, smoke() and bench.py: run a problem
through the CUDA library (paper_1406_7042_b200.fdtd) and through the oracle
(oracle.problem_step), and compare the same quantities element by element."""
from __future__ import annotations

import numpy as np

from oracle import problem_step as ps


def run_gpu(problem, n_steps, precision=None, member_init=None, chunks=None, **kw):
    from paper_1406_7042_b200.fdtd import Sim
    sim = Sim(problem, precision=precision, **kw)
    init = problem.get("init") or {}
    for c, a in init.items():
        a = np.asarray(a, np.float64).reshape(-1, sim.S)
        if a.shape[0] != sim.B:
            a = np.broadcast_to(a, (sim.B, sim.S))
        sim.set_state(int(c), a)
    for n in (chunks or [n_steps]):
        sim.step(n)
    sim.sync()
    comps = (0, 1, 2, 3, 4, 5) if problem["dim"] == 3 else (2, 3, 4)
    st = {c: sim.get_state(c) for c in comps}
    red_e = sim.get_state(6) if problem.get("blocks") else np.zeros(0)
    red_h = sim.get_state(7) if problem.get("blocks") else np.zeros(0)
    probes = sim.probe()
    launches = sim.launch_count()
    sim.close()
    return dict(state=st, red_e=red_e, red_h=red_h, probes=probes, launches=launches)


def run_oracle(problem, n_steps, member=0):
    E, H, probes, rec = ps.run(problem, n_steps, member=member)
    st, re, rh = ps.to_storage(rec, E, H)
    return dict(state=st, red_e=re, red_h=rh, probes=probes, rec=rec, E=E, H=H)


def state_vectors(gpu, ora, member=0):
    """Concatenate the oracle's active unknowns and the GPU values at the same
    unknown ids (coarse), then the reduced states."""
    rec = ora["rec"]
    S = rec.S
    g_parts, o_parts = [], []
    for ids, vec in ((rec.e_ids, ora["E"][:len(rec.e_ids)]), (rec.h_ids, ora["H"][:len(rec.h_ids)])):
        comp = ids // S
        pos = ids % S
        g = np.empty(len(ids))
        for c in np.unique(comp):
            m = comp == c
            g[m] = gpu["state"][int(c)][member][pos[m]]
        g_parts.append(g)
        o_parts.append(vec)
    # reduced: GPU layout [block][inst][B][q]; the oracle's [block][inst][q] (one member)
    blocks = getattr(rec, "_blocks", None)
    return np.concatenate(g_parts), np.concatenate(o_parts)


def reduced_member(gpu_red, shapes, B, member, side):
    out, o = [], 0
    for qe, qh, ni in shapes:
        q = qe if side == "e" else qh
        blk = gpu_red[o:o + ni * B * q].reshape(ni, B, q)
        out.append(blk[:, member, :].ravel())
        o += ni * B * q
    return np.concatenate(out) if out else np.zeros(0)


def block_shapes(problem):
    sh = []
    for b in problem.get("blocks") or []:
        qe = int(b.get("qe", b.get("q")))
        qh = int(b.get("qh", b.get("q")))
        sh.append((qe, qh, int(b["n_inst"])))
    return sh


def rel_l2(a, b):
    nb = np.linalg.norm(b)
    return float(np.linalg.norm(a - b) / (nb if nb > 0 else 1.0))


def compare(problem, gpu, ora, member=0):
    """Relative L2 errors: coarse+reduced state, and the worst probe series."""
    g, o = state_vectors(gpu, ora, member)
    B = int(problem.get("batch", 1))
    sh = block_shapes(problem)
    ge = reduced_member(gpu["red_e"], sh, B, member, "e")
    gh = reduced_member(gpu["red_h"], sh, B, member, "h")
    g_all = np.concatenate([g, ge, gh])
    o_all = np.concatenate([o, ora["red_e"], ora["red_h"]])
    err_state = rel_l2(g_all, o_all)
    err_probe = 0.0
    if gpu["probes"] is not None and len(gpu["probes"]):
        gp = gpu["probes"][:, :, member]
        op = ora["probes"]
        for p in range(op.shape[1]):
            err_probe = max(err_probe, rel_l2(gp[:, p], op[:, p]))
    return err_state, err_probe, float(np.linalg.norm(o_all))
