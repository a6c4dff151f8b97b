"""Parity helpers shared by the GPU tests, smoke() and bench.py: run a problem
through the CUDA library (paper_1406_7042_b200.fdtd) and through the oracle
(oracle.problem_step), and compare the same quantities element by element."""
from __future__ import annotations

import numpy as np

from oracle import problem_step as ps


def gpu_reduced_order(vec_by_member, problem):
    """[B][q_total] per-member reduced vectors -> the binding's set_state order
    [block][inst][B][q]."""
    out, o = [], 0
    for b in problem["blocks"]:
        q = int(b.get("qe", b.get("q")))
        for i in range(int(b["n_inst"])):
            out.append(vec_by_member[:, o:o + q].ravel())
            o += q
    return np.concatenate(out)


def run_gpu(problem, n_steps, precision=None, member_init=None, chunks=None, start=None, **kw):
    """``start``: optional dict(arrays={comp: [B][S]}, red_e=[B][q], red_h=[B][q],
    step=int) -- a (random) starting state instead of the problem's init."""
    from paper_1406_7042_b200.fdtd import Sim
    sim = Sim(problem, precision=precision, **kw)
    init = problem.get("init") or {}
    for c, a in init.items():
        a = np.asarray(a, np.float64).reshape(-1, sim.S)
        if a.shape[0] != sim.B:
            a = np.broadcast_to(a, (sim.B, sim.S))
        sim.set_state(int(c), a)
    if start is not None:
        for c, a in start["arrays"].items():
            sim.set_state(int(c), a)
        if problem.get("blocks"):
            sim.set_state(6, gpu_reduced_order(start["red_e"], problem))
            sim.set_state(7, gpu_reduced_order(start["red_h"], problem))
        sim.set_state(8, [float(start.get("step", 0))])
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


def run_oracle(problem, n_steps, member=0, start=None):
    """``start``: the run_gpu start dict (random state + source step)."""
    if start is not None:
        from sampled_state import oracle_vectors
        rec = ps.build(problem)
        B = int(problem.get("batch", 1))
        re_ = start.get("red_e", np.zeros((B, 0)))
        rh_ = start.get("red_h", np.zeros((B, 0)))
        state = oracle_vectors(rec, start["arrays"], re_, rh_, member)
        E, H, probes, rec = ps.run(problem, n_steps, member=member, state=state,
                                   start_step=int(start.get("step", 0)), rec=rec)
        st, re, rh = ps.to_storage(rec, E, H)
        return dict(state=st, red_e=re, red_h=rh, probes=probes, rec=rec, E=E, H=H)
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


class VacuousReference(AssertionError):
    """A parity subset whose reference is identically zero proves nothing."""


def rel_l2(a, b, name="subset", allow_zero=False):
    """||a - b|| / ||b||; a non-empty subset with ||b|| == 0 fails (a vacuous
    comparison) unless ``allow_zero``."""
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    nb = np.linalg.norm(b)
    if nb == 0:
        if b.size and not allow_zero:
            raise VacuousReference(f"{name}: the reference is identically zero ({b.size} values)")
        return float(np.linalg.norm(a))
    return float(np.linalg.norm(a - b) / nb)


def max_abs(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    if not b.size:
        return 0.0, 0.0
    return float(np.max(np.abs(a - b))), float(np.max(np.abs(b)))


last_report = {}


def subset_errors(subsets, allow_zero=()):
    """{name: (gpu values, reference values)} -> {name: dict(rel_l2, max_abs,
    ref_max, n)}; empty subsets are skipped, zero references fail."""
    out = {}
    for name, (g, o) in subsets.items():
        o = np.asarray(o, np.float64)
        if o.size == 0:
            continue
        ma, rm = max_abs(g, o)
        out[name] = dict(rel_l2=rel_l2(g, o, name, allow_zero=name in allow_zero), max_abs=ma, ref_max=rm,
                         n=int(o.size))
    return out


def compare(problem, gpu, ora, member=0, allow_zero=()):
    """Per-subset relative L2 errors (coarse regular unknowns, interface rows,
    e~, h~, each probe series) -- each subset on its own, so an error in the
    512 reduced unknowns cannot hide behind 3 M coarse ones.  Returns
    (worst state-subset error, worst probe error, ||reference state||); the
    full report is in ``parity.last_report``."""
    rec = ora["rec"]
    S = rec.S
    n_if = 0 if problem.get("interface") is None else len(problem["interface"]["unknown"])
    Ne_c = len(rec.e_ids)
    n_reg = Ne_c - n_if

    def gather(ids):
        comp = ids // S
        pos = ids % S
        g = np.empty(len(ids))
        for c in np.unique(comp):
            m = comp == c
            g[m] = gpu["state"][int(c)][member][pos[m]]
        return g

    B = int(problem.get("batch", 1))
    sh = block_shapes(problem)
    subsets = {
        "coarse": (np.concatenate([gather(rec.e_ids[:n_reg]), gather(rec.h_ids)]),
                   np.concatenate([ora["E"][:n_reg], ora["H"][:len(rec.h_ids)]])),
        "interface": (gather(rec.e_ids[n_reg:]), ora["E"][n_reg:Ne_c]),
        "red_e": (reduced_member(gpu["red_e"], sh, B, member, "e"), ora["red_e"]),
        "red_h": (reduced_member(gpu["red_h"], sh, B, member, "h"), ora["red_h"]),
    }
    if gpu["probes"] is not None and len(gpu["probes"]):
        gp = gpu["probes"][:, :, member]
        op = ora["probes"]
        for p in range(op.shape[1]):
            subsets[f"probe{p}"] = (gp[:, p], op[:, p])
    rep = subset_errors(subsets, allow_zero)
    last_report.clear()
    last_report.update(rep)
    es = max([v["rel_l2"] for k, v in rep.items() if not k.startswith("probe")] or [0.0])
    ep = max([v["rel_l2"] for k, v in rep.items() if k.startswith("probe")] or [0.0])
    norm = float(np.sqrt(sum(np.sum(np.asarray(o) ** 2) for k, (g, o) in subsets.items()
                             if not k.startswith("probe"))))
    return es, ep, norm
