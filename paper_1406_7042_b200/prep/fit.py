"""Vectorised finite-integration (FIT) assembly of uniform grids with a cell
domain mask, and the coarse/fine glue of reading R4.

Host preprocessing for the GPU path (not on the hot path).  Independent of
``oracle/`` by construction (different code, same definitions); the oracle's
``oracle.hybrid`` checks this module's output on small grids.

Volume form on a grid with spacings h = (hx, hy, hz):
  D_eps(edge)  = eps(owning cell) * (#in-domain cells around the edge) * V/4
  D_mu(face)   = mu * A_face * Ltilde,  Ltilde = (#in-domain cells beside the face) * h_n/2
  K(edge,face) = sign * L_edge * Ltilde
scaled (what the problem description carries) = volume form / delta^(dim-1).
2-D is the 3-D machinery restricted to {Ez, Hx, Hy} with one cell in z (h_z = 1).

Unknowns are addressed by (component, storage index) with storage shape
(nz+1, ny+1, nx+1); component ids Ex..Hz = 0..5 (fdtd.h).
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np
import scipy.sparse as sp

# the four edges bounding each face: (edge comp, (di, dj, dk), sign); sign is
# that of K = -curl_H in the E equations (fdtd.h header)
FACE_EDGES = {
    3: ((1, (0, 0, 0), -1), (1, (0, 0, 1), +1), (2, (0, 0, 0), +1), (2, (0, 1, 0), -1)),
    4: ((2, (0, 0, 0), -1), (2, (1, 0, 0), +1), (0, (0, 0, 0), +1), (0, (0, 0, 1), -1)),
    5: ((0, (0, 0, 0), -1), (0, (0, 1, 0), +1), (1, (0, 0, 0), +1), (1, (1, 0, 0), -1)),
}
# cells around an edge of direction a: offsets in the two other axes
_EDGE_CELLS = {0: [(0, -1, -1), (0, 0, -1), (0, -1, 0), (0, 0, 0)],
               1: [(-1, 0, -1), (0, 0, -1), (-1, 0, 0), (0, 0, 0)],
               2: [(-1, -1, 0), (0, -1, 0), (-1, 0, 0), (0, 0, 0)]}
_FACE_CELLS = {0: [(-1, 0, 0), (0, 0, 0)], 1: [(0, -1, 0), (0, 0, 0)], 2: [(0, 0, -1), (0, 0, 0)]}


def comps_of(dim):
    return ((0, 1, 2), (3, 4, 5)) if dim == 3 else ((2,), (3, 4))


def sshape(n, dim=3):
    return (n[2] + 1 if dim == 3 else 1, n[1] + 1, n[0] + 1)


def extent_mask(n, comp, dim):
    """Storage positions where the component exists (not padding)."""
    nx, ny, nz = n
    shp = sshape(n, dim)
    k, j, i = np.indices(shp, sparse=True)
    if dim == 2:
        lim = {2: (k < 1) | (i < 0), 3: (j < ny) & (k < 1), 4: (i < nx) & (k < 1)}
    else:
        lim = {0: i < nx, 1: j < ny, 2: k < nz, 3: (j < ny) & (k < nz),
               4: (i < nx) & (k < nz), 5: (i < nx) & (j < ny)}
    return np.broadcast_to(lim[comp], shp)


def _count_cells(dom, n, offsets, dim):
    """Number of in-domain cells at storage index + offset, for all positions."""
    nx, ny, nz = n
    NZ = sshape(n, dim)[0]
    pad = np.zeros((nz + 2, ny + 2, nx + 2), bool)
    pad[1:-1, 1:-1, 1:-1] = dom
    out = np.zeros(sshape(n, dim), np.int32)
    for (di, dj, dk) in offsets:
        out += pad[1 + dk:1 + dk + NZ, 1 + dj:1 + dj + ny + 1, 1 + di:1 + di + nx + 1]
    return out


@dataclass
class Fit:
    """One FIT grid.  Arrays are storage-shaped per component."""
    dim: int
    n: tuple
    h: tuple
    active: dict = field(default_factory=dict)     # comp -> bool (unknown exists, not PEC, touches domain)
    D: dict = field(default_factory=dict)          # comp -> D_eps / D_mu (volume form)
    cnt: dict = field(default_factory=dict)        # comp -> # in-domain adjacent cells
    K: tuple = None                                # COO (e_comp, e_flat, h_comp, h_flat, val)


def build_fit(dim, n, h, dom, eps_cell, mu_cell, pec, need_K=True):
    """dom: bool cells [nz][ny][nx]; eps_cell/mu_cell: absolute eps/mu per cell;
    pec: comp -> bool storage mask of PEC-eliminated unknowns."""
    n = tuple(int(v) for v in n)
    ecomps, hcomps = comps_of(dim)
    F = Fit(dim, n, tuple(float(v) for v in h))
    vol = h[0] * h[1] * h[2]
    k, j, i = np.indices(sshape(n, dim))
    own = (np.minimum(k, n[2] - 1), np.minimum(j, n[1] - 1), np.minimum(i, n[0] - 1))
    for c in ecomps:
        cnt = _count_cells(dom, n, _EDGE_CELLS[c], dim)
        act = extent_mask(n, c, dim) & ~pec[c] & (cnt > 0)
        F.cnt[c] = np.where(act, cnt, 0)
        F.D[c] = np.where(act, eps_cell[own] * cnt * (vol / 4.0), 0.0)
        F.active[c] = act
    for c in hcomps:
        a = c - 3
        cnt = _count_cells(dom, n, _FACE_CELLS[a], dim)
        act = extent_mask(n, c, dim) & ~pec[c] & (cnt > 0)
        Lt = cnt * (h[a] / 2.0)
        F.cnt[c] = np.where(act, cnt, 0)
        F.D[c] = np.where(act, mu_cell[own] * (vol / h[a]) * Lt, 0.0)
        F.active[c] = act
    if not need_K:
        F.K = tuple(np.zeros(0, t) for t in (np.int8, np.int64, np.int8, np.int64, np.float64))
        return F
    # K entries, face by face
    S = int(np.prod(sshape(n, dim)))
    ec_l, ef_l, hc_l, hf_l, v_l = [], [], [], [], []
    flat = np.arange(S).reshape(sshape(n, dim))
    for c in hcomps:
        a = c - 3
        pos = np.nonzero(F.active[c])
        Lt = F.cnt[c][pos] * (h[a] / 2.0)
        for (e, (di, dj, dk), sgn) in FACE_EDGES[c]:
            if e not in ecomps:
                continue
            kk, jj, ii = pos[0] + dk, pos[1] + dj, pos[2] + di
            ok = (kk < flat.shape[0]) & (jj <= n[1]) & (ii <= n[0])
            kk, jj, ii = kk[ok], jj[ok], ii[ok]
            ea = F.active[e][kk, jj, ii]
            L = h[e] if dim == 3 else 1.0
            ec_l.append(np.full(int(ea.sum()), e, np.int8))
            ef_l.append(flat[kk[ea], jj[ea], ii[ea]])
            hc_l.append(np.full(int(ea.sum()), c, np.int8))
            hf_l.append(flat[pos][ok][ea])
            v_l.append(sgn * L * Lt[ok][ea])
    F.K = (np.concatenate(ec_l), np.concatenate(ef_l), np.concatenate(hc_l),
           np.concatenate(hf_l), np.concatenate(v_l))
    return F


def wall_pec(dim, n, h_origin=None, lo=(0, 0, 0), r=(1, 1, 1), n_coarse=None):
    """PEC masks of the outer walls (tangential E, normal H).  For a fine grid
    (lo, r, n_coarse given), only the parts lying on the coarse domain's walls."""
    nc = n if n_coarse is None else n_coarse
    k, j, i = np.indices(sshape(n, dim))
    # coarse-unit positions of node indices (x = lo + i / r), exact in rationals
    # via integer comparisons: on wall iff lo*r + i == 0 or == nc*r
    X = lo[0] * r[0] + i
    Y = lo[1] * r[1] + j
    Z = lo[2] * r[2] + k
    xw = (X == 0) | (X == nc[0] * r[0])
    yw = (Y == 0) | (Y == nc[1] * r[1])
    zw = (Z == 0) | (Z == nc[2] * r[2]) if dim == 3 else np.zeros_like(xw)
    return {0: yw | zw, 1: xw | zw, 2: xw | yw, 3: xw, 4: yw, 5: zw}


# ---------------------------------------------------------------------------
# the hybrid
# ---------------------------------------------------------------------------

@dataclass
class BoxPart:
    """Everything the reduced model of one box needs (scaled units)."""
    lo: tuple
    hi: tuple
    r: tuple
    fine: Fit = None
    e_int: np.ndarray = None        # (comp, flat) of fine interior E, in order
    h_int: np.ndarray = None
    De_f: np.ndarray = None         # scaled
    Dm_f: np.ndarray = None
    Kff: sp.csr_matrix = None       # fine interior E x fine interior H
    if_ids: np.ndarray = None       # coarse interface E unknown ids (comp*S + s), sorted
    Kcf: sp.csr_matrix = None       # interface rows x fine interior H
    Kfc_max: float = 0.0            # must be 0 (reading R4)


@dataclass
class Hybrid:
    dim: int
    n: tuple
    delta: float
    S: int
    coarse: Fit
    boxes: list
    De_c: dict                      # comp -> scaled coarse D_eps incl. lumped fine part (storage)
    Dm_c: dict
    if_ids: np.ndarray              # all interface E unknown ids (sorted)
    W: sp.csr_matrix                # interface rows x coarse H unknown ids (dense id space 6*S)
    eps_abs: np.ndarray = None


def _interp_targets(dim, comp, pos_num, r, lo):
    """Fine surface E at fine node indices pos (k, j, i arrays) -> coarse target
    storage indices and weights (piecewise constant along the edge, linear
    across).  Coordinates in coarse units: X = lo + idx / r."""
    ax = 2 if dim == 2 else comp
    idx = {0: pos_num[2], 1: pos_num[1], 2: pos_num[0]}
    base, frac = {}, {}
    for a in (0, 1, 2):
        num = lo[a] * r[a] + idx[a]
        base[a] = num // r[a]
        frac[a] = (num % r[a]) / r[a]
    trans = [a for a in ((0, 1) if dim == 2 else (0, 1, 2)) if a != ax]
    terms = [(dict(base), np.ones(len(idx[0])))]
    for a in trans:
        new = []
        for b, w in terms:
            b0 = dict(b)
            new.append((b0, w * (1 - frac[a])))
            b1 = dict(b)
            b1[a] = b[a] + 1
            new.append((b1, w * frac[a]))
        terms = new
    return terms


def assemble(dim, n, delta, eps_r, boxes, eps0, mu0, pec_extra=None, need_K=None):
    """Hybrid of reading R4.  eps_r: relative permittivity per coarse cell;
    boxes: list of dict(lo, hi, r).  pec_extra(grid, comp, shape) -> bool mask
    adds interior PEC unknowns (grid = -1 coarse, b for box b)."""
    n = tuple(int(v) for v in n) + ((1,) if len(n) == 2 else ())
    nx, ny, nz = n
    eps = np.asarray(eps_r, np.float64).reshape(nz, ny, nx) * eps0
    mu = np.full((nz, ny, nx), mu0)
    scale = delta ** (dim - 1)
    shp = sshape(n, dim)
    S = int(np.prod(shp))
    dom = np.ones((nz, ny, nx), bool)
    boxes_n = []
    for b in boxes:
        lo = tuple(b["lo"]) + (0,) * (3 - len(b["lo"]))
        hi = tuple(b["hi"]) + (1,) * (3 - len(b["hi"]))
        r = tuple(b["r"]) + (1,) * (3 - len(b["r"]))
        if dim == 2:
            lo, hi, r = (lo[0], lo[1], 0), (hi[0], hi[1], 1), (r[0], r[1], 1)
        boxes_n.append((lo, hi, r))
        dom[lo[2]:hi[2], lo[1]:hi[1], lo[0]:hi[0]] = False
    pec = wall_pec(dim, n)
    if pec_extra:
        for c in pec:
            pec[c] = pec[c] | pec_extra(-1, c, shp)
    hz = delta if dim == 3 else 1.0
    coarse = build_fit(dim, n, (delta, delta, hz), dom, eps, mu, pec, need_K=bool(boxes) if need_K is None else need_K)
    ecomps, hcomps = comps_of(dim)
    De_c = {c: coarse.D[c] / scale for c in ecomps}
    Dm_c = {c: coarse.D[c] / scale for c in hcomps}
    # interface rows: active coarse E with some adjacent cell inside a box
    allcells = np.ones_like(dom)
    if_mask = {}
    for c in ecomps:
        tot = _count_cells(allcells, n, _EDGE_CELLS[c], dim)
        if_mask[c] = coarse.active[c] & (coarse.cnt[c] < tot)
    if_ids = np.sort(np.concatenate([c * S + np.nonzero(if_mask[c].ravel())[0] for c in ecomps]))
    n_if_tot = len(if_ids)
    ec, ef, hc, hf, v = coarse.K
    eid = ec.astype(np.int64) * S + ef
    hid = hc.astype(np.int64) * S + hf
    sel = np.isin(eid, if_ids)
    W_parts = [(np.searchsorted(if_ids, eid[sel]), hid[sel], v[sel] / scale)]

    parts = []
    for bi, (lo, hi, r) in enumerate(boxes_n):
        nf = tuple((hi[a] - lo[a]) * r[a] for a in range(3))
        if dim == 2:
            nf = (nf[0], nf[1], 1)
        shf = sshape(nf, dim)
        Sf = int(np.prod(shf))
        hf_ = (delta / r[0], delta / r[1], (delta / r[2]) if dim == 3 else 1.0)
        kf, jf, if_ = np.indices((nf[2], nf[1], nf[0]))
        pk, pj, pi = lo[2] + kf // r[2], lo[1] + jf // r[1], lo[0] + if_ // r[0]
        pecf = wall_pec(dim, nf, lo=lo, r=r, n_coarse=n)
        if pec_extra:
            for c in pecf:
                pecf[c] = pecf[c] | pec_extra(bi, c, shf)
        fine = build_fit(dim, nf, hf_, np.ones((nf[2], nf[1], nf[0]), bool),
                         eps[pk, pj, pi], mu[pk, pj, pi], pecf)
        kk, jj, ii = np.indices(shf)
        # fine unknowns on the box surface (constrained) vs interior
        e_surf, e_int_l = {}, []
        for c in ecomps:
            ax = 2 if dim == 2 else c
            on = np.zeros(shf, bool)
            for a, arr in ((0, ii), (1, jj), (2, kk)):
                if a == ax or (dim == 2 and a == 2):
                    continue
                on |= (arr == 0) | (arr == nf[a])
            e_surf[c] = fine.active[c] & on
            e_int_l.append(c * Sf + np.nonzero((fine.active[c] & ~on).ravel())[0])
        h_surf, h_int_l = {}, []
        for c in hcomps:
            arr = (ii, jj, kk)[c - 3]
            on = (arr == 0) | (arr == nf[c - 3])
            h_surf[c] = fine.active[c] & on
            h_int_l.append(c * Sf + np.nonzero((fine.active[c] & ~on).ravel())[0])
        e_int = np.concatenate(e_int_l)
        h_int = np.concatenate(h_int_l)
        fe_all = np.concatenate([c * Sf + np.nonzero(fine.active[c].ravel())[0] for c in ecomps])
        fe_index = -np.ones(6 * Sf, np.int64)
        fe_index[fe_all] = np.arange(len(fe_all))
        # T_E: fine active E -> [coarse interface rows | fine interior]
        rowsT = [fe_index[e_int]]
        colsT = [n_if_tot + np.arange(len(e_int))]
        valsT = [np.ones(len(e_int))]
        for c in ecomps:
            pos = np.nonzero(e_surf[c])
            if not len(pos[0]):
                continue
            fids = c * Sf + np.ravel_multi_index(pos, shf)
            for tgt, w in _interp_targets(dim, c, pos, r, lo):
                keep = w > 0
                cidx = np.ravel_multi_index((tgt[2][keep], tgt[1][keep], tgt[0][keep]), shp)
                cid = c * S + cidx
                q = np.minimum(np.searchsorted(if_ids, cid), max(n_if_tot - 1, 0))
                okt = if_ids[q] == cid            # PEC partners drop out
                rowsT.append(fe_index[fids[keep][okt]]); colsT.append(q[okt]); valsT.append(w[keep][okt])
        TE = sp.csr_matrix((np.concatenate(valsT), (np.concatenate(rowsT), np.concatenate(colsT))),
                           shape=(len(fe_all), n_if_tot + len(e_int)))
        # T_H: fine active H -> [coarse H ids (6*S id space) | fine interior]
        fh_all = np.concatenate([c * Sf + np.nonzero(fine.active[c].ravel())[0] for c in hcomps])
        fh_index = -np.ones(6 * Sf, np.int64)
        fh_index[fh_all] = np.arange(len(fh_all))
        rH, cH = [fh_index[h_int]], [6 * S + np.arange(len(h_int))]
        for c in hcomps:
            pos = np.nonzero(h_surf[c])
            if not len(pos[0]):
                continue
            idx = {0: pos[2], 1: pos[1], 2: pos[0]}
            ci = [(lo[a] * r[a] + idx[a]) // r[a] for a in (0, 1, 2)]
            cidx = np.ravel_multi_index((ci[2], ci[1], ci[0]), shp)
            act = coarse.active[c].ravel()[cidx]
            fids = c * Sf + np.ravel_multi_index(pos, shf)
            rH.append(fh_index[fids[act]]); cH.append(c * S + cidx[act])
        rH = np.concatenate(rH)
        cH = np.concatenate(cH)
        THc = sp.csr_matrix((np.ones(len(rH)), (rH, cH)), shape=(len(fh_all), 6 * S + len(h_int)))
        fec, fef, fhc, fhf, fv = fine.K
        Kf = sp.csr_matrix((fv / scale, (fe_index[fec.astype(np.int64) * Sf + fef],
                                         fh_index[fhc.astype(np.int64) * Sf + fhf])),
                           shape=(len(fe_all), len(fh_all)))
        Kg = (TE.T @ Kf @ THc).tocoo()          # [if | fine int E] x [coarse H | fine int H]
        rr, cc, vv = Kg.row, Kg.col, Kg.data
        to_if = rr < n_if_tot
        to_cH = cc < 6 * S
        kfc = vv[(~to_if) & to_cH]
        m = to_if & to_cH
        W_parts.append((rr[m], cc[m], vv[m]))
        m = to_if & ~to_cH
        Kcf = sp.csr_matrix((vv[m], (rr[m], cc[m] - 6 * S)), shape=(n_if_tot, len(h_int)))
        m = (~to_if) & ~to_cH
        Kff = sp.csr_matrix((vv[m], (rr[m] - n_if_tot, cc[m] - 6 * S)), shape=(len(e_int), len(h_int)))
        # lumped interface masses: rowsum-lump(T_E^T D_eps T_E) (reading R4 step 4)
        Dfe = np.concatenate([fine.D[c].ravel()[np.nonzero(fine.active[c].ravel())[0]] for c in ecomps]) / scale
        rowsum = np.asarray(TE.sum(axis=1)).ravel()
        lump = np.asarray(TE.T @ (Dfe * rowsum)).ravel()[:n_if_tot]
        nzl = np.nonzero(lump)[0]
        for c in ecomps:
            mm = (if_ids[nzl] // S) == c
            np.add.at(De_c[c].ravel(), if_ids[nzl][mm] % S, lump[nzl][mm])
        # surface H masses: T_H^T D_mu T_H
        Dfh = np.concatenate([fine.D[c].ravel()[np.nonzero(fine.active[c].ravel())[0]] for c in hcomps]) / scale
        srow = cH < 6 * S
        for c in hcomps:
            mm = srow & ((cH // S) == c)
            np.add.at(Dm_c[c].ravel(), cH[mm] % S, Dfh[rH[mm]])
        # interface rows belonging to this box: touching one of its cells
        bmask = np.zeros_like(dom)
        bmask[lo[2]:hi[2], lo[1]:hi[1], lo[0]:hi[0]] = True
        mine = []
        for c in ecomps:
            touch = _count_cells(bmask, n, _EDGE_CELLS[c], dim) > 0
            mine.append(c * S + np.nonzero((if_mask[c] & touch).ravel())[0])
        rows_b = np.searchsorted(if_ids, np.sort(np.concatenate(mine)))
        part = BoxPart(lo, hi, r, fine, e_int, h_int, Dfe[fe_index[e_int]], Dfh[fh_index[h_int]],
                       Kff, if_ids[rows_b], Kcf[rows_b], float(np.max(np.abs(kfc))) if len(kfc) else 0.0)
        part.if_rows = rows_b
        parts.append(part)
    rr = np.concatenate([p[0] for p in W_parts])
    cc = np.concatenate([p[1] for p in W_parts])
    vv = np.concatenate([p[2] for p in W_parts])
    W = sp.csr_matrix((vv, (rr, cc)), shape=(n_if_tot, 6 * S))
    W.sum_duplicates()
    W.eliminate_zeros()
    return Hybrid(dim, n, delta, S, coarse, parts, De_c, Dm_c, if_ids, W, eps)
