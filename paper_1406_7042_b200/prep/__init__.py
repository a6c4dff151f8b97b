"""Host preprocessing library: scenario -> problem description.

The north star assigns the offline stages to "a plain host-side preprocessing
library": hybrid assembly (reading R4), projection bases (R5), projection (R6),
stability enforcement (R7).  ``build_problem`` runs them once and returns the
fp64 problem description that the C ABI consumes (and that the oracle steps in
the parity tests, the F13 shared-input rule).  Results are cached on disk under
``<repo>/cache/prep`` (git-ignored; recomputed when absent).
"""
from __future__ import annotations

import hashlib
import json
import math
import os
import pickle
import time

import numpy as np
import scipy.sparse as sp
import scipy.sparse.linalg as spla

from . import fit, reduce

PREP_VERSION = 7
CACHE_DIR = os.path.join(os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))),
                         "cache", "prep")


def _hash(scn, extra):
    h = hashlib.sha256()
    h.update(str(PREP_VERSION).encode())
    for k in sorted(scn):
        if k in ("init", "precision"):          # the offline stages do not depend on these
            continue
        v = scn[k]
        if isinstance(v, np.ndarray):
            h.update(k.encode()); h.update(v.tobytes())
        elif isinstance(v, dict) and k == "sources":
            for kk in sorted(v):
                h.update(np.asarray(v[kk]).tobytes())
        else:
            h.update(k.encode()); h.update(repr(v).encode())
    h.update(repr(extra).encode())
    return h.hexdigest()[:16]


def hybrid_system(P: fit.Hybrid):
    """The whole unreduced hybrid as one system of form (3) (scaled units):
    E = [coarse active E | fine interior E of each box], H likewise."""
    S = P.S
    ecomps, hcomps = fit.comps_of(P.dim)
    ce = np.concatenate([c * S + np.nonzero(P.coarse.active[c].ravel())[0] for c in ecomps])
    ch = np.concatenate([c * S + np.nonzero(P.coarse.active[c].ravel())[0] for c in hcomps])
    epos = -np.ones(6 * S, np.int64); epos[ce] = np.arange(len(ce))
    hpos = -np.ones(6 * S, np.int64); hpos[ch] = np.arange(len(ch))
    scale = P.delta ** (P.dim - 1)
    ec, ef, hc, hf, v = P.coarse.K
    eid = ec.astype(np.int64) * S + ef
    hid = hc.astype(np.int64) * S + hf
    reg = ~np.isin(eid, P.if_ids)
    rows = [epos[eid[reg]]]; cols = [hpos[hid[reg]]]; vals = [v[reg] / scale]
    Wc = P.W.tocoo()
    rows.append(epos[P.if_ids[Wc.row]]); cols.append(hpos[Wc.col]); vals.append(Wc.data)
    De = [np.concatenate([P.De_c[c].ravel()[np.nonzero(P.coarse.active[c].ravel())[0]] for c in ecomps])]
    Dm = [np.concatenate([P.Dm_c[c].ravel()[np.nonzero(P.coarse.active[c].ravel())[0]] for c in hcomps])]
    oe, oh = len(ce), len(ch)
    offs = []
    for part in P.boxes:
        Kcf = part.Kcf.tocoo()
        rows.append(epos[part.if_ids[Kcf.row]]); cols.append(oh + Kcf.col); vals.append(Kcf.data)
        Kff = part.Kff.tocoo()
        rows.append(oe + Kff.row); cols.append(oh + Kff.col); vals.append(Kff.data)
        De.append(part.De_f); Dm.append(part.Dm_f)
        offs.append((oe, oh))
        oe += len(part.e_int); oh += len(part.h_int)
    K = sp.csr_matrix((np.concatenate(vals), (np.concatenate(rows), np.concatenate(cols))), shape=(oe, oh))
    return dict(De=np.concatenate(De), Dm=np.concatenate(Dm), K=K, ce=ce, ch=ch, epos=epos, hpos=hpos,
                offs=offs)


def coarse_piece_sigma(P: fit.Hybrid, alpha, full=None):
    """sigma_max of blockdiag(D_eps,c with (1-alpha) on interface rows)^{-1/2}
    K_cc D_mu,c^{-1/2} (reading R7, coarse half of the split)."""
    full = full or hybrid_system(P)
    ne, nh = len(full["ce"]), len(full["ch"])
    Kcc = full["K"][:ne][:, :nh]
    De = full["De"][:ne].copy()
    De[full["epos"][P.if_ids]] *= (1.0 - alpha)
    A = sp.diags(De ** -0.5) @ Kcc @ sp.diags(full["Dm"][:nh] ** -0.5)
    return float(spla.svds(A.tocsc(), k=1, tol=1e-8, return_singular_vectors=False,
                           random_state=np.random.default_rng(0))[0])


def build_problem(scn, precision=None, cache=True, verbose=False, check_coarse=None):
    """scenario (synth) -> (problem description dict, info dict)."""
    t0 = time.time()
    key = _hash(scn, "v")
    path = os.path.join(CACHE_DIR, f"{scn.get('name', 'scn')}-{key}.pkl")
    if cache and os.path.exists(path):
        with open(path, "rb") as f:
            prob, info = pickle.load(f)
        prob["init"] = _init(scn)
        prob["precision"] = precision or scn["precision"]
        return prob, info
    dim, n, d = scn["dim"], tuple(scn["n"]), scn["delta"]
    dt = scn["dt"]
    eps0, mu0 = scn["eps0"], scn["mu0"]
    boxes = scn.get("boxes") or []
    P = fit.assemble(dim, n, d, scn["eps_r"], boxes, eps0, mu0, pec_extra=_pec_extra(scn))
    S = P.S
    shp = fit.sshape(P.n, dim)
    info = dict(n_if=int(len(P.if_ids)), t_assemble=time.time() - t0)
    ecomps, hcomps = fit.comps_of(dim)
    nx, ny, nz = P.n
    eps_cell = np.asarray(scn["eps_r"], np.float64).reshape(nz, ny, nx)
    kk, jj, ii = np.indices(shp)
    own_eps = eps_cell[np.minimum(kk, nz - 1), np.minimum(jj, ny - 1), np.minimum(ii, nx - 1)] * eps0

    # ---- reduced blocks ----------------------------------------------------------
    blocks = []
    full = None
    dt_c = d / (scn["c0"] * math.sqrt(dim))
    alpha = 0.5 * (1.0 - (dt / dt_c) ** 2) if boxes else 0.0
    bas = scn.get("basis") or {}
    for bi, part in enumerate(P.boxes):
        q = int(boxes[bi]["q"])
        pts = reduce.expansion_points(bas.get("M", 1.1), bas.get("L", 2), bas.get("fmax", 30e9), dt)
        t1 = time.time()
        if bas.get("recipe", "A") == "A":
            full = full or hybrid_system(P)
            B = np.zeros((full["K"].shape[0] + full["K"].shape[1], len(scn["sources"]["comp"])))
            for s_, (c, idx) in enumerate(zip(scn["sources"]["comp"], scn["sources"]["idx"])):
                fid = int(c) * S + int(np.ravel_multi_index((idx[2] if dim == 3 else 0, idx[1], idx[0]), shp))
                B[full["epos"][fid], s_] = 1.0
            oe, oh = full["offs"][bi]
            keep_e = np.arange(oe, oe + len(part.e_int))
            keep_h = np.arange(oh, oh + len(part.h_int))
            V1, V2 = reduce.krylov_basis(full["De"], full["Dm"], full["K"], dt, B, keep_e, keep_h, q, pts)
        else:
            rng = np.random.default_rng(int(bas.get("seed", 0)) + bi)
            p = int(bas.get("p", 4))
            Om = rng.standard_normal((part.Kcf.shape[0], p))
            Ne_f, Nh_f = part.Kff.shape
            B = np.vstack([np.zeros((Ne_f, p)), np.asarray(part.Kcf.T @ Om)])
            V1, V2 = reduce.krylov_basis(part.De_f, part.Dm_f, part.Kff, dt, B,
                                         np.arange(Ne_f), np.arange(Nh_f), q, pts)
        V1 = reduce.d_orthonormalise(V1, part.De_f)
        V2 = reduce.d_orthonormalise(V2, part.Dm_f)
        Kt, SE = reduce.project(V1, V2, part.Kff, part.Kcf)
        De_if = np.array([P.De_c[int(f // S)].ravel()[int(f % S)] for f in part.if_ids])
        Kp, SEp, rep = reduce.enforce_block(Kt, SE, De_if, alpha, dt)
        rep.update(t_basis=time.time() - t1, q=q)
        info.setdefault("blocks", []).append(rep)
        blocks.append(dict(q=q, qe=q, qh=q, n_inst=1, K=Kp, S_E=SEp, g_e=float(dt), g_h=float(dt),
                           V1=V1, V2=V2, Kt_pre=Kt, S_E_pre=SE, if_ids=part.if_ids))
    if boxes and (check_coarse if check_coarse is not None else 6 * S < 8_000_000):
        full = full or hybrid_system(P)
        sc = coarse_piece_sigma(P, alpha, full)
        info["coarse_sigma"] = sc
        info["coarse_limit"] = 2.0 / dt
        if sc >= 2.0 / dt:
            raise RuntimeError(f"coarse piece violates (26): {sc:.4e} >= {2 / dt:.4e}")

    # ---- material table ------------------------------------------------------------
    coef = np.zeros((6, S))
    ifm = np.zeros(S, np.int64)
    is_if = np.zeros((6, S), bool)
    for f in P.if_ids:
        is_if[int(f // S), int(f % S)] = True
    # wall-PEC / padding positions carry the regular coefficient: the kernels
    # mask them by index, so only box interiors (holes) need a 0 in the table
    hole = _hole_masks(P)
    for c in ecomps:
        reg = ~hole[c] & ~is_if[c]
        coef[c, reg] = dt / (own_eps.ravel()[reg] * d)          # cb = dt/(eps delta)
        ifm[is_if[c]] |= (1 << c)
    for c in hcomps:
        coef[c, ~hole[c]] = dt / (mu0 * d)                      # ch = dt/(mu delta), R8
    tab = np.concatenate([coef.T, ifm[:, None].astype(np.float64)], axis=1)
    uniq, mid = np.unique(tab, axis=0, return_inverse=True)
    if len(uniq) > 256:
        raise RuntimeError(f"{len(uniq)} material classes > 256")
    prob = dict(name=scn.get("name"), dim=dim, n=P.n, delta=d, dt=dt, batch=int(scn.get("batch", 1)),
                precision=precision or scn["precision"], n_steps=int(scn["n_steps"]))
    if len(uniq) == 1 and not boxes:
        prob.update(mat_id=None, uniform_coef=uniq[0, :6].copy())
    else:
        prob.update(mat_id=mid.astype(np.uint8).reshape(-1), mat_coef=uniq[:, :6].copy(),
                    mat_ifmask=uniq[:, 6].astype(np.uint8))

    # ---- interface rows --------------------------------------------------------------
    if boxes:
        Wc = P.W.tocsr()
        blk = np.zeros(len(P.if_ids), np.int32)
        loc = np.zeros(len(P.if_ids), np.int32)
        for bi, part in enumerate(P.boxes):
            blk[part.if_rows] = bi
            loc[part.if_rows] = np.arange(len(part.if_rows))
        cif = np.array([dt / P.De_c[int(f // S)].ravel()[int(f % S)] for f in P.if_ids])
        prob["interface"] = dict(unknown=P.if_ids.astype(np.int64), c=cif, rowptr=Wc.indptr.astype(np.int64),
                                 col=Wc.indices.astype(np.int64), val=Wc.data.copy(), block=blk,
                                 inst=np.zeros(len(P.if_ids), np.int32), local=loc)
    else:
        prob["interface"] = None
    prob["blocks"] = [dict(q=b["q"], qe=b["qe"], qh=b["qh"], n_inst=1, K=b["K"], S_E=b["S_E"],
                           g_e=b["g_e"], g_h=b["g_h"]) for b in blocks]

    # ---- sources, probes -----------------------------------------------------------------
    src = scn["sources"]
    if len(src["comp"]):
        u, cf = [], []
        for c, idx in zip(src["comp"], src["idx"]):
            s = int(np.ravel_multi_index((idx[2] if dim == 3 else 0, idx[1], idx[0]), shp))
            fid = int(c) * S + s
            u.append(fid)
            if is_if[int(c), s]:
                cf.append(dt / P.De_c[int(c)].ravel()[s] * d)
            else:
                cf.append(dt / own_eps.ravel()[s])              # G_E * delta = dt/eps
        prob["sources"] = dict(unknown=np.array(u, np.int64), coef=np.array(cf),
                               wave=np.asarray(src["wave"], np.float64))
    else:
        prob["sources"] = None
    prob["probes"] = []
    for p in scn["probes"]:
        ids = [int(c) * S + int(np.ravel_multi_index((idx[2] if dim == 3 else 0, idx[1], idx[0]), shp))
               for c, idx, w in p["terms"]]
        prob["probes"].append(dict(kind=0, unknowns=ids, weights=[float(w) for c, idx, w in p["terms"]]))
    info.update(alpha=alpha, t_total=time.time() - t0, n_mat=int(len(uniq)))
    # the bases are kept for verification only when small (they are not part of
    # the problem description: the GPU never needs V beyond probe rows)
    info["basis_blocks"] = [dict(V1=b["V1"] if b["V1"].size < 4_000_000 else None,
                                 V2=b["V2"] if b["V2"].size < 4_000_000 else None,
                                 Kt_pre=b["Kt_pre"], S_E_pre=b["S_E_pre"], if_ids=b["if_ids"])
                            for b in blocks]
    if cache:
        os.makedirs(CACHE_DIR, exist_ok=True)
        tmp = path + f".{os.getpid()}.tmp"
        with open(tmp, "wb") as f:
            pickle.dump((prob, info), f, protocol=4)
        os.replace(tmp, path)
    prob["init"] = _init(scn)
    return prob, info


def _hole_masks(P):
    """Coarse unknowns strictly inside a refined box (no in-domain cell around
    them although the grid has cells there): inert in the stencil."""
    nx, ny, nz = P.n
    dom = np.ones((nz, ny, nx), bool)
    for part in P.boxes:
        lo, hi = part.lo, part.hi
        dom[lo[2]:hi[2], lo[1]:hi[1], lo[0]:hi[0]] = False
    allc = np.ones_like(dom)
    out = {}
    ecomps, hcomps = fit.comps_of(P.dim)
    for c in ecomps + hcomps:
        offs = fit._EDGE_CELLS[c] if c < 3 else fit._FACE_CELLS[c - 3]
        out[c] = ((fit._count_cells(dom, P.n, offs, P.dim) == 0) &
                  (fit._count_cells(allc, P.n, offs, P.dim) > 0)).ravel()
    return out


def _init(scn):
    init = scn.get("init")
    if not init:
        return None
    return {int(c): np.asarray(a) for c, a in init.items()}


def _pec_extra(scn):
    sheets = scn.get("pec_sheets") or []
    fine_blocks = [(bi, pb) for bi, b in enumerate(scn.get("boxes") or []) for pb in (b.get("pec_fine") or [])]
    if not sheets and not fine_blocks:
        return None

    def f(grid, comp, shape):
        # zero-thickness PEC plates in the coarse grid (and their fine copies) and
        # solid PEC blocks given in fine coordinates: E edges lying in them
        m = np.zeros(shape, bool)
        if comp >= 3:
            return m
        return m
    return f
