"""Random states for one-step sampled parity (oracle.problem_step.
sampled_hybrid_step): seeded values on the ACTIVE unknowns of the recursion
only (inert ones -- holes, PEC plates, walls -- stay zero, as they do in every
real run), and the same state in the oracle's vector ordering."""
import numpy as np

from oracle import problem_step as ps


def active_masks(problem):
    """comp -> boolean [S] mask of unknowns the recursion updates, without the
    matrix form: live (not wall / not eliminated) and coefficient != 0, or an
    interface row."""
    from oracle import yee
    dim = int(problem["dim"])
    n = tuple(int(v) for v in problem["n"]) + ((1,) if len(problem["n"]) == 2 else ())
    shp = yee.storage_shape(dim, n)
    S = int(np.prod(shp))
    comps = (yee.E_COMPS_3D + yee.H_COMPS_3D) if dim == 3 else (yee.E_COMPS_2D + yee.H_COMPS_2D)
    mid = np.asarray(problem["mat_id"]).reshape(-1)
    coef = np.asarray(problem["mat_coef"], np.float64)
    itf = problem.get("interface")
    ifu = np.asarray(itf["unknown"], np.int64) if itf is not None else np.zeros(0, np.int64)
    out = {}
    for c in comps:
        live = (yee.exists_mask(dim, n, c) & ~yee.wall_pec_mask(dim, n, c)).reshape(-1)
        m = live & (coef[mid, c] != 0.0)
        sel = ifu[ifu // S == c] % S
        m[sel] = True
        out[c] = m
    return out, S


def random_state(problem, seed, B=None, window=None):
    """{comp: [B][S]} coarse arrays and per-member reduced vectors."""
    rng = np.random.default_rng(seed)
    masks, S = active_masks(problem)
    B = int(problem.get("batch", 1)) if B is None else B
    arrays = {}
    for c, m in masks.items():
        a = np.zeros((B, S))
        idx = np.nonzero(m)[0]
        if window is not None:
            idx = idx[window(idx)]
        a[:, idx] = rng.uniform(-1.0, 1.0, size=(B, len(idx)))
        arrays[c] = a
    qe = sum(int(b.get("qe", b.get("q"))) * int(b["n_inst"]) for b in problem["blocks"])
    qh = sum(int(b.get("qh", b.get("q"))) * int(b["n_inst"]) for b in problem["blocks"])
    red_e = rng.uniform(-1.0, 1.0, size=(B, qe))
    red_h = rng.uniform(-1.0, 1.0, size=(B, qh))
    return arrays, red_e, red_h


def oracle_vectors(rec, arrays, red_e, red_h, member):
    """The state in the oracle's vector ordering [E_c ; e~], [H_c ; h~]."""
    def gather(ids):
        comp, pos = ids // rec.S, ids % rec.S
        out = np.empty(len(ids))
        for c in np.unique(comp):
            m = comp == c
            out[m] = np.asarray(arrays[int(c)])[member][pos[m]]
        return out
    E = np.concatenate([gather(rec.e_ids), red_e[member]])
    H = np.concatenate([gather(rec.h_ids), red_h[member]])
    return E, H
