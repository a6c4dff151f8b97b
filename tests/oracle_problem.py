"""Test infrastructure: build a problem description straight from
the oracle's own hybrid assembly and a given fine-region basis, without the
preprocessing library.  Used to pin oracle.problem_step (the parity path)
against the symmetric reduced-hybrid leap-frog, and as an extra GPU parity
case whose every input and expected value comes from oracle/ alone."""
from __future__ import annotations

import numpy as np
import scipy.sparse as sp

from oracle import hybrid as hy
from oracle import yee


def _flat(dim, n, comp, idx):
    shp = yee.storage_shape(dim, n)
    S = int(np.prod(shp))
    i, j, k = idx
    pos = np.ravel_multi_index((k, j, i) if dim == 3 else (j, i), shp)
    return comp * S + int(pos)


def problem_from_oracle(scn, V1f=None, V2f=None, Kt=None, SEif=None, dt=None):
    """scn: synth scenario (2-D or 3-D with boxes).  V1f/V2f None -> identity
    basis (the unreduced hybrid).  Kt/SEif: optional enforced blocks."""
    dim, n, d = scn["dim"], tuple(scn["n"]), scn["delta"]
    dt = scn["dt"] if dt is None else dt
    boxes = [hy.Box(tuple(b["lo"]), tuple(b["hi"]), tuple(b["r"])) for b in scn["boxes"]]
    hs = hy.assemble(dim, n, d, scn["eps_r"], boxes, scn["eps0"], scn["mu0"])
    b = hy.blocks(hs)
    if V1f is None:
        V1f, V2f = np.eye(len(b["ef"])), np.eye(len(b["hf"]))
    pr = hy.project(hs, V1f, V2f)
    shp = yee.storage_shape(dim, n)
    S = int(np.prod(shp))
    ncomp = 6
    coef = np.zeros((ncomp, S))
    ifm = np.zeros(S, np.int64)
    # coarse E: regular -> cb = dt / D_eps ; surface -> interface row
    if_ids, if_c, rp, cols, vals = [], [], [0], [], []
    Kcsr = hs.K.tocsr()
    hc_set = set(b["hc"].tolist())
    for r, key in enumerate(hs.e_keys):
        if key[0] != "c":
            continue
        fid = _flat(dim, n, key[1], key[2])
        comp, pos = fid // S, fid % S
        if hs.e_tag[r] == 0:
            coef[comp, pos] = dt / hs.De[r]
        else:
            ifm[pos] |= 1 << comp
            if_ids.append(fid)
            if_c.append(dt / hs.De[r])
            row = Kcsr[r]
            for c, v in zip(row.indices, row.data):
                if c in hc_set:
                    cols.append(_flat(dim, n, hs.h_keys[c][1], hs.h_keys[c][2]))
                    vals.append(v)
            rp.append(len(cols))
    mu0 = scn["mu0"]
    for r, key in enumerate(hs.h_keys):
        if key[0] != "c":
            continue
        fid = _flat(dim, n, key[1], key[2])
        coef[fid // S, fid % S] = dt / (mu0 * d)        # regular ch (reading R8)
    # material table = unique coefficient columns
    tab = np.concatenate([coef.T, ifm[:, None].astype(np.float64)], axis=1)
    uniq, mat_id = np.unique(tab, axis=0, return_inverse=True)
    assert len(uniq) <= 256
    # interface local numbering follows the order of pr["if_rows"] (coarse E order)
    SE = np.asarray(pr["S_E"])[pr["if_rows"]] if SEif is None else SEif
    Kt_rr = pr["Kt_rr"] if Kt is None else Kt
    Dte, Dtm = pr["Dt_e"], pr["Dt_m"]
    if np.allclose(Dte, np.diag(np.diag(Dte))):
        ge = dt / np.diag(Dte)
        gh = dt / np.diag(Dtm)
    else:
        raise ValueError("only diagonal D~ supported")
    problem = dict(
        dim=dim, n=n, delta=d, dt=dt, batch=1,
        mat_id=mat_id.astype(np.uint8).reshape(shp), mat_coef=uniq[:, :6],
        mat_ifmask=uniq[:, 6].astype(np.uint8),
        interface=dict(unknown=np.array(if_ids, np.int64), c=np.array(if_c),
                       rowptr=np.array(rp, np.int64), col=np.array(cols, np.int64),
                       val=np.array(vals), block=np.zeros(len(if_ids), np.int32),
                       inst=np.zeros(len(if_ids), np.int32),
                       local=np.arange(len(if_ids), dtype=np.int32)),
        blocks=[dict(qe=Kt_rr.shape[0], qh=Kt_rr.shape[1], n_inst=1, K=Kt_rr, S_E=SE,
                     g_e=ge, g_h=gh)],
        sources=None, probes=[], init=None)
    # sources (coarse E) : coef = G_E * delta   (scaled B = -delta)
    src = scn["sources"]
    if len(src["comp"]):
        u, cf = [], []
        for c, idx in zip(src["comp"], src["idx"]):
            fid = _flat(dim, n, int(c), tuple(int(v) for v in idx))
            r = hs.e_index[("c", int(c), tuple(int(v) for v in idx))]
            u.append(fid)
            cf.append(dt / hs.De[r] * d)
        problem["sources"] = dict(unknown=np.array(u, np.int64), coef=np.array(cf),
                                  wave=np.asarray(src["wave"]))
    for p in scn["probes"]:
        problem["probes"].append(dict(kind=0, unknowns=[_flat(dim, n, c, idx) for c, idx, w in p["terms"]],
                                      weights=[w for c, idx, w in p["terms"]]))
    return problem, hs, pr


def uniform_problem(scn, dt=None):
    """Problem description of a box-free uniform grid with per-cell eps
    (owning-cell rule): cb = dt/(eps delta), ch = dt/(mu delta)."""
    dim, n, d = scn["dim"], tuple(scn["n"]), scn["delta"]
    dt = scn["dt"] if dt is None else dt
    shp = yee.storage_shape(dim, n)
    eps = np.asarray(scn["eps_r"], np.float64)
    if np.all(eps == eps.flat[0]):
        cb = dt / (scn["eps0"] * eps.flat[0] * d)
        ch = dt / (scn["mu0"] * d)
        prob = dict(dim=dim, n=n, delta=d, dt=dt, batch=1, mat_id=None,
                    uniform_coef=np.array([cb, cb, cb, ch, ch, ch]))
    else:
        own = yee.owning_cell(dim, n)
        er = eps[own]
        cbs = dt / (scn["eps0"] * er * d)
        tab, mid = np.unique(cbs.ravel(), return_inverse=True)
        ch = dt / (scn["mu0"] * d)
        coef = np.zeros((len(tab), 6))
        coef[:, 0:3] = tab[:, None]
        coef[:, 3:6] = ch
        prob = dict(dim=dim, n=n, delta=d, dt=dt, batch=1, mat_id=mid.astype(np.uint8).reshape(shp),
                    mat_coef=coef, mat_ifmask=np.zeros(len(tab), np.uint8))
    prob.update(interface=None, blocks=[], sources=None, probes=[],
                init={c: np.asarray(a) for c, a in (scn.get("init") or {}).items()})
    for p in scn["probes"]:
        prob["probes"].append(dict(kind=0, unknowns=[_flat(dim, n, c, idx) for c, idx, w in p["terms"]],
                                   weights=[w for c, idx, w in p["terms"]]))
    return prob
