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

PREP_VERSION = 9
# dense reduced matrices above this many entries are stored rounded to fp32
# (reading R13: config 4's S_E is 65,024 x 1,024; both the GPU and
# the oracle consume the same rounded values)
BIG_DENSE = 1 << 25
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


def build_problem(scn, precision=None, cache=True, verbose=False, check_coarse=None, keep_basis=False,
                  reducer="host", reducer_opts=None):
    """scenario (synth) -> (problem description dict, info dict).  ``keep_basis``
    keeps every projection basis in ``info`` (verification of large models;
    implies no cache).  ``reducer``: "host" (SciPy sparse LU + NumPy Arnoldi,
    prep/reduce.py) or "gpu" (the device reduction of include/fdtd_mor.h: block
    Schur + CGS shifted solves and the block Arnoldi on the GPU, SURVEY NEXT-1;
    ``reducer_opts`` are keyword arguments of ``mor.Mor.krylov_basis``)."""
    if keep_basis:
        cache = False
    if reducer not in ("host", "gpu"):
        raise ValueError("reducer must be 'host' or 'gpu'")
    if reducer == "gpu":
        from .. import mor as _mor

        def _krylov(*a):
            V = _mor.krylov_basis(*a, **(reducer_opts or {}))
            info.setdefault("mor_stats", []).append(_mor.krylov_basis.last_stats)
            return V
    else:
        _krylov = reduce.krylov_basis
    t0 = time.time()
    key = _hash(scn, "v" if reducer == "host" else ("v", reducer, sorted((reducer_opts or {}).items())))
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
    # congruent regions share one reduced model ("model" class): basis,
    # projection and enforcement run on the first instance; the others must
    # carry identical local matrices (translated copies)
    classes = {}
    for bi, b in enumerate(boxes):
        classes.setdefault(int(b.get("model", bi)), []).append(bi)
    class_ids = sorted(classes)
    box_class = {bi: (ci, classes[c].index(bi)) for ci, c in enumerate(class_ids) for bi in classes[c]}
    for c in class_ids:
        first = P.boxes[classes[c][0]]
        for bi in classes[c][1:]:
            other = P.boxes[bi]
            same = (other.Kff.shape == first.Kff.shape and other.Kcf.shape == first.Kcf.shape and
                    abs(other.Kff - first.Kff).max() <= 1e-12 * abs(first.Kff).max() and
                    abs(other.Kcf - first.Kcf).max() <= 1e-12 * abs(first.Kcf).max() and
                    np.allclose(other.De_f, first.De_f, rtol=1e-13) and np.allclose(other.Dm_f, first.Dm_f, rtol=1e-13))
            if not same:
                raise ValueError(f"box {bi} is not a translated copy of box {classes[c][0]} (model {c})")
    for bi, part in enumerate(P.boxes):
        if box_class[bi][1] != 0:
            continue
        q = int(boxes[bi]["q"])
        if bas.get("points") == "zero":
            pts = [0.0]          # the paper's z = 0 fast path, reading R5(viii)
        else:
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
            V1, V2 = _krylov(full["De"], full["Dm"], full["K"], dt, B, keep_e, keep_h, q, pts)
        else:
            rng = np.random.default_rng(int(bas.get("seed", 0)) + bi)
            p = int(bas.get("p", 4))
            Om = rng.standard_normal((part.Kcf.shape[0], p))
            Ne_f, Nh_f = part.Kff.shape
            B = np.vstack([np.zeros((Ne_f, p)), np.asarray(part.Kcf.T @ Om)])
            V1, V2 = _krylov(part.De_f, part.Dm_f, part.Kff, dt, B, np.arange(Ne_f), np.arange(Nh_f), q, pts)
        V1 = reduce.d_orthonormalise(V1, part.De_f)
        V2 = reduce.d_orthonormalise(V2, part.Dm_f)
        Kt, SE = reduce.project(V1, V2, part.Kff, part.Kcf)
        De_if = np.array([P.De_c[int(f // S)].ravel()[int(f % S)] for f in part.if_ids])
        Kp, SEp, rep = reduce.enforce_block(Kt, SE, De_if, alpha, dt)
        if SEp.size > BIG_DENSE:
            SEp = SEp.astype(np.float32)
        rep.update(t_basis=time.time() - t1, q=q)
        info.setdefault("blocks", []).append(rep)
        blocks.append(dict(q=q, qe=q, qh=q, n_inst=len(classes[class_ids[box_class[bi][0]]]), K=Kp, S_E=SEp,
                           g_e=float(dt), g_h=float(dt), V1=V1, V2=V2, Kt_pre=Kt, S_E_pre=SE,
                           if_ids=part.if_ids))
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
    pecx = _pec_extra(scn)
    if pecx is not None:                   # interior PEC (plates): inert like holes
        for c in ecomps:
            hole[c] = hole[c] | pecx(-1, c, shp).ravel()
    for c in ecomps:
        reg = ~hole[c] & ~is_if[c]
        coef[c, reg] = dt / (own_eps.ravel()[reg] * d)          # cb = dt/(eps delta)
        ifm[is_if[c]] |= (1 << c)
    for c in hcomps:
        coef[c, ~hole[c]] = dt / (mu0 * d)                      # ch = dt/(mu delta), R8
    # lossy media / matched absorbers (Eq. (2a)/(2b) with the
    # conductivity terms, D_sigma of Eq. (5)): per-cell sigma_e [S/m], sigma_m
    # [Ohm/m] with the owning-cell rule (R1(iv)):
    #   cb = 1/((eps/dt + sigma_e/2) delta),  ca = (eps/dt - sigma_e/2)/(eps/dt + sigma_e/2)
    #   ch = 1/((mu/dt + sigma_m/2) delta),   da = (mu/dt - sigma_m/2)/(mu/dt + sigma_m/2)
    lossy = scn.get("sigma_e") is not None or scn.get("sigma_m") is not None
    ca = np.ones((6, S))
    own_se = None
    if lossy:
        def own(cellarr):
            a = np.zeros((nz, ny, nx)) if cellarr is None else np.asarray(cellarr, np.float64).reshape(nz, ny, nx)
            return a[np.minimum(kk, nz - 1), np.minimum(jj, ny - 1), np.minimum(ii, nx - 1)].ravel()
        own_se, own_sm = own(scn.get("sigma_e")), own(scn.get("sigma_m"))
        if np.any(own_se < 0) or np.any(own_sm < 0):
            raise ValueError("conductivities must be >= 0 (Eq. (7), P:141-147)")
        for c in ecomps:
            reg = ~hole[c] & ~is_if[c]
            if np.any(own_se[is_if[c]] != 0):
                raise NotImplementedError("lossy cells touching a refined box (interface rows stay lossless)")
            a_, b_ = own_eps.ravel()[reg] / dt, 0.5 * own_se[reg]
            coef[c, reg] = 1.0 / ((a_ + b_) * d)
            ca[c, reg] = (a_ - b_) / (a_ + b_)
        for c in hcomps:
            reg = ~hole[c]
            a_, b_ = mu0 / dt, 0.5 * own_sm[reg]
            coef[c, reg] = 1.0 / ((a_ + b_) * d)
            ca[c, reg] = (a_ - b_) / (a_ + b_)
    # distinct (coefficients, interface bits) rows -> material table; per-column
    # codes first so that 10^7-row grids take seconds
    codes, vals = [], []
    for col in list(coef) + [ifm.astype(np.float64)] + (list(ca) if lossy else []):
        u, inv = np.unique(col, return_inverse=True)
        codes.append(inv.astype(np.int64))
        vals.append(u)
    key = np.zeros(S, np.int64)
    for cd, u in zip(codes, vals):
        key = key * len(u) + cd
    ukey, first, mid = np.unique(key, return_index=True, return_inverse=True)
    tab = np.concatenate([coef.T, ifm[:, None].astype(np.float64)] + ([ca.T] if lossy else []), axis=1)
    uniq = tab[first]
    if len(uniq) > 256:
        raise RuntimeError(f"{len(uniq)} material classes > 256")
    prob = dict(name=scn.get("name"), dim=dim, n=P.n, delta=d, dt=dt, batch=int(scn.get("batch", 1)),
                precision=precision or scn["precision"], n_steps=int(scn["n_steps"]))
    if len(uniq) == 1 and not boxes and not lossy:
        prob.update(mat_id=None, uniform_coef=uniq[0, :6].copy())
    else:
        prob.update(mat_id=mid.astype(np.uint8).reshape(-1), mat_coef=uniq[:, :6].copy(),
                    mat_ifmask=uniq[:, 6].astype(np.uint8))
        if lossy:
            prob["mat_ca"] = uniq[:, 7:13].copy()

    # ---- interface rows --------------------------------------------------------------
    if boxes:
        Wc = P.W.tocsr()
        blk = np.zeros(len(P.if_ids), np.int32)
        loc = np.zeros(len(P.if_ids), np.int32)
        ins = np.zeros(len(P.if_ids), np.int32)
        for bi, part in enumerate(P.boxes):
            ci, inst = box_class[bi]
            blk[part.if_rows] = ci
            ins[part.if_rows] = inst
            loc[part.if_rows] = np.arange(len(part.if_rows))
        cif = np.array([dt / P.De_c[int(f // S)].ravel()[int(f % S)] for f in P.if_ids])
        prob["interface"] = dict(unknown=P.if_ids.astype(np.int64), c=cif, rowptr=Wc.indptr.astype(np.int64),
                                 col=Wc.indices.astype(np.int64), val=Wc.data.copy(), block=blk,
                                 inst=ins, local=loc)
    else:
        prob["interface"] = None
    prob["blocks"] = [dict(q=b["q"], qe=b["qe"], qh=b["qh"], n_inst=b["n_inst"], K=b["K"], S_E=b["S_E"],
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
                if lossy:
                    cf.append(1.0 / (own_eps.ravel()[s] / dt + 0.5 * own_se[s]))
                else:
                    cf.append(dt / own_eps.ravel()[s])          # G_E * delta = dt/eps
        amp = np.asarray(src.get("amp", np.ones(len(u))), np.float64)
        prob["sources"] = dict(unknown=np.array(u, np.int64), coef=np.array(cf) * amp,
                               wave=np.asarray(src["wave"], np.float64))
        if src.get("column") is not None:
            prob["sources"]["column"] = np.asarray(src["column"], np.int32)
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
    info["basis_blocks"] = [dict(V1=b["V1"] if keep_basis or b["V1"].size < 4_000_000 else None,
                                 V2=b["V2"] if keep_basis or b["V2"].size < 4_000_000 else None,
                                 Kt_pre=b["Kt_pre"],
                                 S_E_pre=b["S_E_pre"] if keep_basis or b["S_E_pre"].size <= BIG_DENSE else None,
                                 if_ids=b["if_ids"])
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
    """Zero-thickness PEC plates (scenario 'pec_sheets', normal axis z): every E
    edge lying in the plate (closed rectangle) is eliminated, in the coarse grid
    and in the refined boxes alike (S:137 elimination, R1(ii))."""
    sheets = scn.get("pec_sheets") or []
    boxes = scn.get("boxes") or []
    blocks_f = {bi: b.get("pec_fine") or [] for bi, b in enumerate(boxes)}
    blocks_c = scn.get("pec_blocks") or []      # solid PEC blocks of the coarse grid (closed node boxes; irises)
    if not sheets and not any(blocks_f.values()) and not blocks_c:
        return None
    dim = scn["dim"]

    def solid_coarse(comp, shape):
        m = np.zeros(shape, bool)
        k, j, i = np.indices(shape)
        ijk = (i, j, k)
        ax_of = 2 if dim == 2 else comp             # 2-D: Ez edges run along z (one node in the plane)
        for blk in blocks_c:
            lo = tuple(blk["lo"]) + (0,) * (3 - len(blk["lo"]))
            hi = tuple(blk["hi"]) + (0,) * (3 - len(blk["hi"]))
            inside = np.ones(shape, bool)
            for a in range(dim):
                if a == ax_of:
                    inside &= (ijk[a] >= lo[a]) & (ijk[a] + 1 <= hi[a])
                else:
                    inside &= (ijk[a] >= lo[a]) & (ijk[a] <= hi[a])
            m |= inside
        return m

    def solid(grid, comp, shape):
        """solid PEC blocks given in a box's fine node indices (closed): every
        E edge with both end nodes in the block"""
        m = np.zeros(shape, bool)
        if grid < 0 or not blocks_f.get(grid):
            return m
        k, j, i = np.indices(shape)
        ijk = (i, j, k)
        for blk in blocks_f[grid]:
            lo, hi = blk["lo"], blk["hi"]
            inside = np.ones(shape, bool)
            for a in range(3):
                if a == comp:
                    inside &= (ijk[a] >= lo[a]) & (ijk[a] + 1 <= hi[a])
                else:
                    inside &= (ijk[a] >= lo[a]) & (ijk[a] <= hi[a])
            m |= inside
        return m

    def f(grid, comp, shape):
        m = np.zeros(shape, bool)
        if comp > 2:
            return m
        if grid < 0 and blocks_c:
            m |= solid_coarse(comp, shape)
        if dim != 3:
            return m
        m |= solid(grid, comp, shape)
        if comp not in (0, 1) or not sheets:
            return m
        if grid < 0:
            lo, r = (0, 0, 0), (1, 1, 1)
        else:
            b = boxes[grid]
            lo, r = tuple(b["lo"]), tuple(b["r"])
        k, j, i = np.indices(shape)
        # integer coarse-unit coordinates scaled by r: X*rx = lo_x*rx + i
        X = lo[0] * r[0] + i
        Y = lo[1] * r[1] + j
        Z = lo[2] * r[2] + k
        for sh in sheets:
            if sh["axis"] != 2:
                raise NotImplementedError("PEC sheets normal to z only")
            (x0, y0), (x1, y1) = sh["lo"], sh["hi"]
            onz = Z == sh["pos"] * r[2]
            if comp == 0:      # Ex edge from X to X+1 (fine units) at Y
                m |= onz & (X >= x0 * r[0]) & (X + 1 <= x1 * r[0]) & (Y >= y0 * r[1]) & (Y <= y1 * r[1])
            else:              # Ey edge from Y to Y+1 at X
                m |= onz & (X >= x0 * r[0]) & (X <= x1 * r[0]) & (Y >= y0 * r[1]) & (Y + 1 <= y1 * r[1])
        return m
    return f
