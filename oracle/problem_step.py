"""The reduced-hybrid recursion (4)/(12) driven by a problem description - the
thing the GPU path must match (survey §8(c) O8, reading R8).

A *problem description* is the fp64 data both sides consume (F13 shared-input
rule): coarse per-unknown coefficients through a material table, interface
rows, reduced blocks, sources, probes, initial state.  Its field list is in
DESIGN.md §6.  This module parses it on its own (it shares no code with the
binding or the C library) and advances

    (R~ + F~)(x^{n+1} - x^n) = -2 F~ x^n + B~ u^{n+1}            (from (4), (12))

with x = [E_c ; e~ ; H_c ; h~] and the hybrid curl
    K~ = [[K_cc , S_E],
          [ 0   , K~'_rr]]            (K_fc = 0, survey O6)
by forward substitution with the inverse diagonal blocks given as data:
G_E = cb (coarse), c_if (interface rows), g_e (reduced); G_H = ch, g_h.
K_cc is the oracle's *own* incidence matrix of the coarse grid
(oracle.yee.incidence), restricted to the active unknowns; interface rows
use the problem's W_if instead.  H rows use K^T except that surface H rows are
divided by their common factor (reading R8: a row scaling of the H equations,
which leaves the solution of (4) unchanged), so they carry +-1 with the
regular ch, exactly as stated in the problem.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import scipy.sparse as sp

from . import yee
from .matrix_form import step_leapfrog


def storage_size(dim, n):
    return int(np.prod(yee.storage_shape(dim, n)))


@dataclass
class HybridRecursion:
    dim: int
    n: tuple
    S: int                   # storage size per component
    e_ids: np.ndarray        # flat unknown ids (comp*S + flat) of active coarse E
    h_ids: np.ndarray
    n_red: tuple             # total reduced unknowns (E side, H side)
    red_off: list            # per block: (E, H) offsets of instance 0
    KE: sp.csr_matrix        # rows [E_c ; e~], cols [H_c ; h~]
    KH: sp.csr_matrix        # rows [H_c ; h~], cols [E_c ; e~]
    GE: np.ndarray
    GH: np.ndarray
    src_row: np.ndarray      # E row of each source
    src_coef: np.ndarray
    wave: np.ndarray         # [n_wave][n_cols][B]
    probe_rows: list         # per probe: (side, sparse row vector over that side)
    src_col: np.ndarray = None   # waveform column of each source
    CE: np.ndarray = None        # lossy media: ca per E row (1 on interface / reduced rows), None: lossless
    CH: np.ndarray = None


def build(problem) -> HybridRecursion:
    dim = int(problem["dim"])
    n = tuple(int(v) for v in problem["n"]) + ((1,) if len(problem["n"]) == 2 else ())
    d = float(problem["delta"])
    shp = yee.storage_shape(dim, n)
    S = int(np.prod(shp))
    ys = yee.assemble(dim, n, (d, d, d), 1.0, 1.0, eliminate_pec=True)
    Kinc = yee.incidence(ys)          # +-1 (E rows: K = -curl_H)
    ecomps, hcomps = ys.e_comps, ys.h_comps

    # ---- per-unknown coefficients from the material table --------------------
    def coef_of(comp):
        if problem.get("mat_id") is None:
            return np.full(shp, float(problem["uniform_coef"][comp]))
        mid = np.asarray(problem["mat_id"]).reshape(shp)
        return np.asarray(problem["mat_coef"], dtype=np.float64)[:, comp][mid]

    def ifbit(comp):
        if problem.get("mat_id") is None:
            return np.zeros(shp, bool)
        mid = np.asarray(problem["mat_id"]).reshape(shp)
        return (np.asarray(problem["mat_ifmask"]).astype(np.int64)[mid] >> comp) & 1 == 1

    itf = problem.get("interface")
    if_ids = np.asarray(itf["unknown"], dtype=np.int64) if itf is not None else np.zeros(0, np.int64)
    # the material table's interface bits must mark exactly the interface rows
    marked = np.concatenate([c * S + np.nonzero(ifbit(c).ravel())[0] for c in ecomps])
    if not np.array_equal(np.sort(marked), np.sort(if_ids)):
        raise ValueError("interface rows and material interface bits disagree")

    # active coarse E: regular (cb != 0) or interface rows; yee index gives the
    # wall-PEC elimination and the column numbering of Kinc.
    e_sel, e_ids, e_G, e_isif = [], [], [], []
    for c in ecomps:
        cb = coef_of(c)
        m = ys.index[c] >= 0
        reg = m & (cb != 0.0) & ~ifbit(c)
        e_sel.append((c, reg))
    h_sel = []
    for c in hcomps:
        ch = coef_of(c)
        m = (ys.index[c] >= 0) & (ch != 0.0)
        h_sel.append((c, m))

    # regular E rows
    rows_yee, GE_reg, ids_reg = [], [], []
    for c, reg in e_sel:
        pos = np.nonzero(reg.ravel())[0]
        rows_yee.append(ys.index[c].ravel()[pos])
        GE_reg.append(coef_of(c).ravel()[pos])
        ids_reg.append(c * S + pos)
    rows_yee = np.concatenate(rows_yee)
    GE_reg = np.concatenate(GE_reg)
    ids_reg = np.concatenate(ids_reg)
    cols_yee, GH_c, h_ids = [], [], []
    for c, m in h_sel:
        pos = np.nonzero(m.ravel())[0]
        cols_yee.append(ys.index[c].ravel()[pos] )
        GH_c.append(coef_of(c).ravel()[pos])
        h_ids.append(c * S + pos)
    cols_yee = np.concatenate(cols_yee)
    GH_c = np.concatenate(GH_c)
    h_ids = np.concatenate(h_ids)
    Nh_c = len(h_ids)
    hpos = -np.ones(ys.Nh, np.int64)
    hpos[cols_yee] = np.arange(Nh_c)

    # E ordering: regular rows then interface rows
    n_reg = len(ids_reg)
    n_if = len(if_ids)
    e_ids = np.concatenate([ids_reg, if_ids])
    Ne_c = len(e_ids)

    blocks = problem.get("blocks", []) or []

    def qe_qh(b):
        return int(b.get("qe", b.get("q"))), int(b.get("qh", b.get("q")))

    red_off, off_e, off_h = [], 0, 0
    for b in blocks:
        qe, qh = qe_qh(b)
        red_off.append((off_e, off_h))
        off_e += qe * int(b["n_inst"])
        off_h += qh * int(b["n_inst"])
    n_red = (off_e, off_h)
    NE, NH = Ne_c + off_e, Nh_c + off_h

    # ---- K_E -----------------------------------------------------------------
    Kc = Kinc[rows_yee][:, cols_yee].tocoo()            # regular rows x active H
    r_, c_, v_ = [Kc.row], [Kc.col], [Kc.data]
    # map flat H ids -> column (via yee index of the storage position)
    def hcol(flat_ids):
        comp = flat_ids // S
        pos = flat_ids % S
        out = np.empty(len(flat_ids), np.int64)
        for c in np.unique(comp):
            m = comp == c
            yi = ys.index[int(c)].ravel()[pos[m]]
            if np.any(yi < 0):
                raise ValueError("W_if references an eliminated H unknown")
            out[m] = hpos[yi]
        if np.any(out < 0):
            raise ValueError("W_if references an inactive H unknown")
        return out
    GE_if = np.zeros(n_if)
    if n_if:
        rp = np.asarray(itf["rowptr"], np.int64)
        cols = hcol(np.asarray(itf["col"], np.int64))
        vals = np.asarray(itf["val"], np.float64)
        rr = np.repeat(np.arange(n_if), np.diff(rp))
        r_.append(n_reg + rr); c_.append(cols); v_.append(vals)
        GE_if = np.asarray(itf["c"], np.float64)
        # interface row r couples to every h~ of its block instance with the
        # weights S_E[local(r)] (rows grouped by (block, instance), same entries
        # as a loop over r)
        blk_, ins_, loc_ = (np.asarray(itf[k], np.int64) for k in ("block", "inst", "local"))
        for bl in np.unique(blk_):
            b = blocks[int(bl)]
            qe, qh = qe_qh(b)
            SEb = np.asarray(b["S_E"])
            for inst in np.unique(ins_[blk_ == bl]):
                rows = np.nonzero((blk_ == bl) & (ins_ == inst))[0]
                o = Nh_c + red_off[int(bl)][1] + int(inst) * qh
                r_.append(np.repeat(n_reg + rows, qh)); c_.append(np.tile(o + np.arange(qh), len(rows)))
                v_.append(SEb[loc_[rows]].astype(np.float64).ravel())
    GE_red, GH_red = [], []
    for bl, b in enumerate(blocks):
        qe, qh = qe_qh(b)
        Kt = np.asarray(b["K"], np.float64).reshape(qe, qh)
        for inst in range(int(b["n_inst"])):
            oe = red_off[bl][0] + inst * qe
            oh = red_off[bl][1] + inst * qh
            rr, cc = np.meshgrid(np.arange(qe), np.arange(qh), indexing="ij")
            r_.append(Ne_c + oe + rr.ravel()); c_.append(Nh_c + oh + cc.ravel()); v_.append(Kt.ravel())
            # G_e = (D~_eps/dt)^{-1}: scalar dt (D~ = I) or a diagonal
            GE_red.append(np.broadcast_to(np.asarray(b["g_e"], np.float64), (qe,)).copy())
            GH_red.append(np.broadcast_to(np.asarray(b["g_h"], np.float64), (qh,)).copy())
    KE = sp.csr_matrix((np.concatenate(v_), (np.concatenate(r_), np.concatenate(c_))), shape=(NE, NH))

    # ---- K_H: coarse H rows = K_inc^T over active E (interface E included,
    # with the incidence weights: surface H rows row-scaled, reading R8) -------
    e_yee_rows = np.empty(len(e_ids), np.int64)
    for c in np.unique(e_ids // S):
        m = (e_ids // S) == c
        e_yee_rows[m] = ys.index[int(c)].ravel()[e_ids[m] % S]
    if np.any(e_yee_rows < 0):
        raise ValueError("an active E unknown lies on a PEC wall")
    KHc = (Kinc[e_yee_rows][:, cols_yee].T).tocoo()      # Nh_c x Ne_c
    r_, c_, v_ = [KHc.row], [KHc.col], [KHc.data]
    if n_if:
        # the transpose of the interface-row couplings above (h~ rows, E_if columns)
        for bl in np.unique(blk_):
            b = blocks[int(bl)]
            qe, qh = qe_qh(b)
            SEb = np.asarray(b["S_E"])
            for inst in np.unique(ins_[blk_ == bl]):
                rows = np.nonzero((blk_ == bl) & (ins_ == inst))[0]
                o = red_off[int(bl)][1] + int(inst) * qh
                r_.append(np.tile(Nh_c + o + np.arange(qh), len(rows))); c_.append(np.repeat(n_reg + rows, qh))
                v_.append(SEb[loc_[rows]].astype(np.float64).ravel())
    for bl, b in enumerate(blocks):
        qe, qh = qe_qh(b)
        Kt = np.asarray(b["K"], np.float64).reshape(qe, qh)
        for inst in range(int(b["n_inst"])):
            oe = red_off[bl][0] + inst * qe
            oh = red_off[bl][1] + inst * qh
            rr, cc = np.meshgrid(np.arange(qh), np.arange(qe), indexing="ij")
            # (K^T)[r, c] = K[c, r]
            r_.append(Nh_c + oh + rr.ravel()); c_.append(Ne_c + oe + cc.ravel()); v_.append(Kt.T.ravel())
    KH = sp.csr_matrix((np.concatenate(v_), (np.concatenate(r_), np.concatenate(c_))), shape=(NH, NE))

    GE = np.concatenate([GE_reg, GE_if] + GE_red)
    GH = np.concatenate([GH_c] + GH_red)

    # ---- sources ---------------------------------------------------------------
    src = problem.get("sources")
    e_sort = np.argsort(e_ids, kind="stable")

    def epos_of(u):                       # position of unknown id u in e_ids
        k = int(np.searchsorted(e_ids, u, sorter=e_sort))
        if k >= len(e_ids) or e_ids[e_sort[k]] != u:
            raise KeyError(u)
        return int(e_sort[k])
    if src is not None and len(src["unknown"]):
        src_row = np.array([epos_of(int(u)) for u in src["unknown"]], np.int64)
        src_coef = np.asarray(src["coef"], np.float64)
        wave = np.asarray(src["wave"], np.float64)
        col = src.get("column")
        src_col = (np.asarray(col, np.int64) if col is not None else np.arange(len(src_row)))
    else:
        src_row, src_coef, wave = np.zeros(0, np.int64), np.zeros(0), np.zeros((0, 0, 1))
        src_col = np.zeros(0, np.int64)

    # ---- probes ----------------------------------------------------------------
    h_sort = np.argsort(h_ids, kind="stable")

    def hpos_of(u):
        k = int(np.searchsorted(h_ids, u, sorter=h_sort))
        if k >= len(h_ids) or h_ids[h_sort[k]] != u:
            raise KeyError(u)
        return int(h_sort[k])
    probe_rows = []
    prb = problem.get("probes") or []
    for p in prb:
        kind = int(p["kind"])
        if kind == 0:            # weighted sum of coarse unknowns, all E or all H
            ids = [int(u) for u in p["unknowns"]]
            ws = [float(w) for w in p["weights"]]
            if all((u // S) in ecomps for u in ids):
                probe_rows.append(("E", {epos_of(u): w for u, w in zip(ids, ws)}))
            elif all((u // S) in hcomps for u in ids):
                probe_rows.append(("H", {hpos_of(u): w for u, w in zip(ids, ws)}))
            else:
                raise ValueError("a coarse probe mixes E and H unknowns")
        else:
            bl, inst = int(p["block"]), int(p["inst"])
            qe, qh = qe_qh(blocks[bl])
            if kind == 1:
                vrow = np.asarray(p["vrow"], np.float64)[:qe]
                o = Ne_c + red_off[bl][0] + inst * qe
                probe_rows.append(("E", {o + i: vrow[i] for i in range(qe) if vrow[i] != 0}))
            else:
                vrow = np.asarray(p["vrow"], np.float64)[:qh]
                o = Nh_c + red_off[bl][1] + inst * qh
                probe_rows.append(("H", {o + i: vrow[i] for i in range(qh) if vrow[i] != 0}))
    # lossy media: the diagonal of (R+F)^{-1}(R-F) restricted to
    # the conductivity terms, ca = (eps/dt - sigma/2)/(eps/dt + sigma/2) per E
    # unknown (da likewise), enters as shared data like cb / ch (F13): Eq. (4)
    # with D_sigma reads E' = ca E - cb (K_inc H), H' = da H + ch (K_inc^T E')
    # (pinned against the literal solve of (4), tests/test_oracle_lossy.py)
    CE = CH = None
    if problem.get("mat_ca") is not None:
        mid = np.asarray(problem["mat_id"]).reshape(-1)
        mca = np.asarray(problem["mat_ca"], np.float64)
        CE = np.ones(KE.shape[0])
        CH = np.ones(KH.shape[0])
        CE[:n_reg] = mca[mid[ids_reg % S], ids_reg // S]
        CH[:Nh_c] = mca[mid[h_ids % S], h_ids // S]
    return HybridRecursion(dim, n, S, e_ids, h_ids, n_red, red_off, KE, KH, GE, GH,
                           src_row, src_coef, wave, probe_rows, src_col, CE, CH)


def initial_state(rec: HybridRecursion, problem, member=0):
    NE, NH = rec.KE.shape
    E = np.zeros(NE)
    H = np.zeros(NH)
    init = problem.get("init")
    if init:
        for c, arr in init.items():
            a = np.asarray(arr, np.float64)
            a = a.reshape(-1, rec.S)[member] if a.size != rec.S else a.ravel()
            c = int(c)
            ids = rec.e_ids if c < 3 else rec.h_ids
            m = (ids // rec.S) == c
            tgt = E if c < 3 else H
            tgt[np.nonzero(m)[0]] = a[ids[m] % rec.S]
    return E, H


def probe_matrices(rec: HybridRecursion):
    NE, NH = rec.KE.shape
    P = len(rec.probe_rows)
    PE = sp.lil_matrix((P, NE))
    PH = sp.lil_matrix((P, NH))
    for i, (side, row) in enumerate(rec.probe_rows):
        tgt = PE if side == "E" else PH
        for k, w in row.items():
            tgt[i, k] = w
    return PE.tocsr(), PH.tocsr()


def run(problem, n_steps, member=0, state=None, start_step=0, rec=None):
    """Advance n_steps from the initial (or given) state for one batch member.

    Returns (E, H, probes[n_steps][n_probe], rec).  Probe sampling: E after the
    E half (time (n+1) dt), H after the H half."""
    rec = build(problem) if rec is None else rec
    E, H = initial_state(rec, problem, member) if state is None else state
    PE, PH = probe_matrices(rec)
    probes = np.zeros((n_steps, len(rec.probe_rows)))
    for s in range(n_steps):
        step = start_step + s
        su = None
        if len(rec.src_row) and step < rec.wave.shape[0]:
            su = np.zeros(len(E))
            # E += -coef * J^{n+1/2}   (B holds the sign)
            np.add.at(su, rec.src_row, -rec.src_coef * rec.wave[step, rec.src_col, member])
        if rec.CE is None:
            E, H = step_leapfrog(E, H, rec.GE, rec.GH, rec.KE, rec.KH, su_E=su)
        else:
            E = rec.CE * E - rec.GE * (rec.KE @ H) + (0.0 if su is None else su)
            H = rec.CH * H + rec.GH * (rec.KH @ E)
        probes[s] = PE @ E + PH @ H
    return E, H, probes, rec


def to_storage(rec: HybridRecursion, E, H):
    """Coarse parts as per-component storage arrays (flat), reduced parts split."""
    out = {}
    Ne_c = len(rec.e_ids)
    Nh_c = len(rec.h_ids)
    for ids, vec in ((rec.e_ids, E[:Ne_c]), (rec.h_ids, H[:Nh_c])):
        comp = ids // rec.S
        for c in np.unique(comp):
            a = out.setdefault(int(c), np.zeros(rec.S))
            m = comp == c
            a[ids[m] % rec.S] = vec[m]
    return out, E[Ne_c:], H[Nh_c:]


def sampled_step(problem, arrays, samples, member=0):
    """One step of (4) for SAMPLED coarse unknowns of a problem without
    interface rows or sources, straight from the definitions: E^{n+1} at the
    sampled E unknowns and at every E unknown their H partners need, then
    H^{n+1} = H^n + ch (K_inc^T E^{n+1}).  ``arrays``: comp -> storage array
    [B][S] of the state at step n; ``samples``: list of (comp, (i, j, k)).
    Returns {(comp, idx): value at step n+1}.  For full-size configs the
    oracle cannot hold (16.8 M cells x 6 unknowns), survey §8(d)."""
    dim = int(problem["dim"])
    n = tuple(int(v) for v in problem["n"]) + ((1,) if len(problem["n"]) == 2 else ())
    shp = yee.storage_shape(dim, n)
    if problem.get("interface") or problem.get("sources") or problem.get("mat_ca") is not None:
        raise ValueError("sampled_step covers the pure lossless coarse recursion only")
    curl_h = yee._CURL_H_3D if dim == 3 else yee._CURL_H_2D
    mcurl_e = yee._MCURL_E_3D if dim == 3 else yee._MCURL_E_2D
    ecomps = (0, 1, 2) if dim == 3 else (2,)
    pec = {c: yee.wall_pec_mask(dim, n, c) & yee.exists_mask(dim, n, c) for c in range(6) if c in
           (yee.E_COMPS_3D + yee.H_COMPS_3D if dim == 3 else yee.E_COMPS_2D + yee.H_COMPS_2D)}
    exists = {c: yee.exists_mask(dim, n, c) for c in pec}

    def coef(c, pos):
        if problem.get("mat_id") is None:
            return float(problem["uniform_coef"][c])
        mid = np.asarray(problem["mat_id"]).reshape(shp)
        return float(np.asarray(problem["mat_coef"])[mid[pos], c])

    def val(c, idx):
        i, j, k = idx
        pos = (k, j, i) if dim == 3 else (j, i)
        if any(p < 0 or p >= s for p, s in zip(pos, shp)):
            return 0.0, None
        if not exists[c][pos] or pec[c][pos]:
            return 0.0, None
        return float(np.asarray(arrays[c]).reshape(-1, *shp)[member][pos]), pos

    def e_new(c, idx):
        v, pos = val(c, idx)
        if pos is None:
            return 0.0
        acc = 0.0
        for (hc, off, sign, _) in curl_h[c]:
            hv, _ = val(hc, (idx[0] + off[0], idx[1] + off[1], idx[2] + off[2]))
            acc += sign * hv
        return v + coef(c, pos) * acc          # E + cb curl H  ==  E - cb K_inc H

    out = {}
    for (c, idx) in samples:
        idx = tuple(int(x) for x in idx)
        if c in ecomps:
            out[(c, idx)] = e_new(c, idx)
        else:
            v, pos = val(c, idx)
            if pos is None:
                out[(c, idx)] = 0.0
                continue
            acc = 0.0
            for (ec, off, sign, _) in mcurl_e[c]:
                acc += sign * e_new(ec, (idx[0] + off[0], idx[1] + off[1], idx[2] + off[2]))
            out[(c, idx)] = v + coef(c, pos) * acc   # H - ch curl E == H + ch K_inc^T E
    return out


def sampled_hybrid_step(problem, arrays, red_e, red_h, samples, member=0, step=0):
    """One step of the hybrid recursion (4)/(12) (the same update as ``run``,
    ``step_leapfrog``: E' = E - G_E (K_E H) + s, H' = H + G_H (K_H E')) for
    full-size problems the matrix form cannot hold (config 4: 8.5 M cells and a
    65,024 x 1,024 S_E), evaluated unknown by unknown from the problem
    description:

      * every interface row r (block b, instance i, local l):
            E_if' = E_if - c_r (sum_k w_rk H[col_rk] + S_E[l] . h~_{b,i}) + s_r
      * every reduced block/instance:
            e~' = e~ - g_e (K~ h~)
            h~' = h~ + g_h (K~^T e~' + sum_{rows r of (b, i)} S_E[l_r] E_if'[r])
      * the SAMPLED coarse unknowns: E' = E + cb curl H (+ source) on regular
        rows (only active H: ch != 0), H' = H + ch (K_inc^T E') with E' from
        the two rules above.

    ``arrays``: comp -> [B][S] (or [S]) storage arrays of E^n, H^{n+1/2};
    ``red_e`` / ``red_h``: one member's reduced states, [block][inst][q] order;
    ``step``: the source waveform index of this step.  Returns
    (coarse {(comp, idx): value}, E_if' in interface-row order, e~', h~')."""
    dim = int(problem["dim"])
    n = tuple(int(v) for v in problem["n"]) + ((1,) if len(problem["n"]) == 2 else ())
    shp = yee.storage_shape(dim, n)
    S = int(np.prod(shp))
    curl_h = yee._CURL_H_3D if dim == 3 else yee._CURL_H_2D
    mcurl_e = yee._MCURL_E_3D if dim == 3 else yee._MCURL_E_2D
    ecomps = (0, 1, 2) if dim == 3 else (2,)
    comps = (yee.E_COMPS_3D + yee.H_COMPS_3D) if dim == 3 else (yee.E_COMPS_2D + yee.H_COMPS_2D)
    live = {c: yee.exists_mask(dim, n, c) & ~yee.wall_pec_mask(dim, n, c) for c in comps}
    mid = np.asarray(problem["mat_id"]).reshape(shp)
    mcoef = np.asarray(problem["mat_coef"], np.float64)
    itf = problem["interface"]
    blocks = problem.get("blocks") or []

    def pos_of(idx):
        i, j, k = idx
        return (k, j, i) if dim == 3 else (j, i)

    def inside(pos):
        return all(0 <= p < s for p, s in zip(pos, shp))

    def coef(c, pos):
        return float(mcoef[mid[pos], c])

    def raw(c, pos):
        a = np.asarray(arrays[c])
        return float(a.reshape(-1, *shp)[member if a.size != S else 0][pos])

    def h_val(c, idx):                      # active coarse H (K_E columns)
        pos = pos_of(idx)
        if not inside(pos) or not live[c][pos] or coef(c, pos) == 0.0:
            return 0.0
        return raw(c, pos)

    def flat(pos):
        return int(np.ravel_multi_index(pos, shp))

    # sources: unknown -> list of (coef, column)
    src = problem.get("sources")
    srcs = {}
    if src is not None and len(src["unknown"]):
        cols = src.get("column")
        for q, u in enumerate(np.asarray(src["unknown"], np.int64)):
            srcs.setdefault(int(u), []).append(
                (float(np.asarray(src["coef"])[q]), int(cols[q]) if cols is not None else q))
        wave = np.asarray(src["wave"], np.float64)
    else:
        wave = np.zeros((0, 0, 1))

    def s_term(u):
        v = 0.0
        for cf, col in srcs.get(u, ()):
            if step < wave.shape[0]:
                v -= cf * wave[step, col, member]
        return v

    # reduced states per (block, instance)
    def split(vec, side):
        out, o = {}, 0
        for bl, b in enumerate(blocks):
            q = int(b.get("qe" if side == "e" else "qh", b.get("q")))
            for i in range(int(b["n_inst"])):
                out[(bl, i)] = np.asarray(vec[o:o + q], np.float64)
                o += q
        return out
    e_red, h_red = split(red_e, "e"), split(red_h, "h")

    # interface rows
    unk = np.asarray(itf["unknown"], np.int64)
    rp = np.asarray(itf["rowptr"], np.int64)
    colv = np.asarray(itf["col"], np.int64)
    valv = np.asarray(itf["val"], np.float64)
    cr = np.asarray(itf["c"], np.float64)
    blk, ins, loc = (np.asarray(itf[k], np.int64) for k in ("block", "inst", "local"))
    SE = [np.asarray(b["S_E"]) for b in blocks]
    Eif = np.empty(len(unk))
    row_of = {}
    for r in range(len(unk)):
        u = int(unk[r])
        c, p = u // S, u % S
        pos = np.unravel_index(p, shp)
        acc = 0.0
        for k in range(rp[r], rp[r + 1]):
            hc, hp = int(colv[k] // S), int(colv[k] % S)
            acc += valv[k] * raw(hc, np.unravel_index(hp, shp))
        acc += float(np.dot(SE[blk[r]][loc[r]].astype(np.float64), h_red[(int(blk[r]), int(ins[r]))]))
        Eif[r] = raw(c, pos) - cr[r] * acc + s_term(u)
        row_of[u] = r

    # reduced update
    e_new_red, h_new_red = {}, {}
    for bl, b in enumerate(blocks):
        qe = int(b.get("qe", b.get("q")))
        qh = int(b.get("qh", b.get("q")))
        K = np.asarray(b["K"], np.float64).reshape(qe, qh)
        ge = np.broadcast_to(np.asarray(b["g_e"], np.float64), (qe,))
        gh = np.broadcast_to(np.asarray(b["g_h"], np.float64), (qh,))
        for i in range(int(b["n_inst"])):
            e1 = e_red[(bl, i)] - ge * (K @ h_red[(bl, i)])
            rows = np.nonzero((blk == bl) & (ins == i))[0]
            t = K.T @ e1
            if len(rows):
                t = t + SE[bl][loc[rows]].astype(np.float64).T @ Eif[rows]
            e_new_red[(bl, i)] = e1
            h_new_red[(bl, i)] = h_red[(bl, i)] + gh * t

    def e_new(c, idx):
        pos = pos_of(idx)
        if not inside(pos) or not live[c][pos]:
            return 0.0
        u = c * S + flat(pos)
        if u in row_of:
            return float(Eif[row_of[u]])
        cb = coef(c, pos)
        if cb == 0.0:
            return raw(c, pos)                 # inert (hole / PEC plate): unchanged
        acc = 0.0
        for (hc, off, sign, _) in curl_h[c]:
            acc += sign * h_val(hc, (idx[0] + off[0], idx[1] + off[1], idx[2] + off[2]))
        return raw(c, pos) + cb * acc + s_term(u)

    out = {}
    for (c, idx) in samples:
        idx = tuple(int(x) for x in idx)
        if c in ecomps:
            out[(c, idx)] = e_new(c, idx)
            continue
        pos = pos_of(idx)
        if not inside(pos) or not live[c][pos] or coef(c, pos) == 0.0:
            out[(c, idx)] = raw(c, pos) if inside(pos) else 0.0
            continue
        acc = 0.0
        for (ec, off, sign, _) in mcurl_e[c]:
            acc += sign * e_new(ec, (idx[0] + off[0], idx[1] + off[1], idx[2] + off[2]))
        out[(c, idx)] = raw(c, pos) + coef(c, pos) * acc
    flat_red = lambda d: np.concatenate([d[k] for k in sorted(d)]) if d else np.zeros(0)
    return out, Eif, flat_red(e_new_red), flat_red(h_new_red)
