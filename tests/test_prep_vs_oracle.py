"""The preprocessing library's vectorised hybrid assembly (product) against the
oracle's independent loop-based assembly (reading R4): identical interface
rows, lumped masses, W_if, K_ff, K_cf, surface-H masses, and K_fc = 0."""
import time

import numpy as np
import pytest
from synth import scenario
from oracle import hybrid as hy
from paper_1406_7042_b200.prep import fit

def check(dim, n, eps, boxes):
    t=time.time()
    P = fit.assemble(dim, n, 1e-3, eps, boxes, 8.854e-12, 1.2566e-6)
    t1=time.time()-t
    ob = [hy.Box(tuple(b["lo"]), tuple(b["hi"]), tuple(b["r"])) for b in boxes]
    O = hy.assemble(dim, n, 1e-3, eps, ob, 8.854e-12, 1.2566e-6)
    S = P.S
    shp = fit.sshape(P.n, dim)
    def cflat(key):
        _, c, (i,j,k) = key
        return c*S + np.ravel_multi_index((k if dim==3 else 0, j, i), shp)
    surf = sorted(cflat(O.e_keys[r]) for r in np.nonzero(O.e_tag==1)[0])
    assert np.array_equal(np.array(surf), P.if_ids), "if ids"
    # De at interface rows
    for q, fid in enumerate(P.if_ids):
        c, s = fid//S, fid%S
        r = O.e_index[('c', int(c), tuple(int(v) for v in (lambda t: (t[2], t[1], t[0]))(np.unravel_index(s, shp))))]
        assert abs(P.De_c[c].ravel()[s] - O.De[r]) <= 1e-13*abs(O.De[r]), (P.De_c[c].ravel()[s], O.De[r])
    # W rows
    Kc = O.K.tocsr()
    for q, fid in enumerate(P.if_ids):
        c, s = fid//S, fid%S
        ijk = np.unravel_index(s, shp); key = ('c', int(c), (int(ijk[2]), int(ijk[1]), int(ijk[0])))
        r = O.e_index[key]
        row = Kc[r]
        oref = {}
        for col, v in zip(row.indices, row.data):
            hk = O.h_keys[col]
            if hk[0]=='c': oref[cflat(hk)] = v
        prow = P.W[q]
        pgot = {int(cc): v for cc, v in zip(prow.indices, prow.data)}
        assert set(oref) == set(pgot), (oref, pgot)
        for kk in oref: assert abs(oref[kk]-pgot[kk]) <= 1e-13*abs(oref[kk])
    # fine blocks
    for bi, part in enumerate(P.boxes):
        Sf = int(np.prod(fit.sshape(part.fine.n, dim)))
        shf = fit.sshape(part.fine.n, dim)
        def fflat(key):
            _, b, c, (i,j,k) = key
            return c*Sf + np.ravel_multi_index((k if dim==3 else 0, j, i), shf)
        oe = {fflat(O.e_keys[r]): r for r in np.nonzero((O.e_tag==2)&(O.e_box==bi))[0]}
        oh = {fflat(O.h_keys[r]): r for r in np.nonzero((O.h_tag==2)&(O.h_box==bi))[0]}
        assert set(oe) == set(part.e_int.tolist()) and set(oh) == set(part.h_int.tolist())
        pe = np.array([oe[v] for v in part.e_int]); ph = np.array([oh[v] for v in part.h_int])
        Kff_o = O.K[pe][:, ph]
        assert abs(Kff_o - part.Kff).max() <= 1e-13*abs(Kff_o).max()
        assert np.allclose(O.De[pe], part.De_f, rtol=1e-13) and np.allclose(O.Dm[ph], part.Dm_f, rtol=1e-13)
        # Kcf
        rows = [O.e_index[('c', int(fid//S), (lambda ijk: (int(ijk[2]), int(ijk[1]), int(ijk[0])))(np.unravel_index(fid%S, shp)))] for fid in part.if_ids]
        Kcf_o = O.K[rows][:, ph]
        assert abs(Kcf_o - part.Kcf).max() <= 1e-13*abs(Kcf_o).max()
        assert part.Kfc_max == 0.0
    # surface H masses
    for r in np.nonzero(O.h_tag==1)[0]:
        fid = cflat(O.h_keys[r]); c, s = fid//S, fid%S
        assert abs(P.Dm_c[c].ravel()[s] - O.Dm[r]) <= 1e-13*O.Dm[r]

CASES = [
    ("tiny2d", None, None, None),
    ("config1", 2, (40, 20, 1), [dict(lo=(16, 6, 0), hi=(24, 14, 1), r=(4, 4, 1))]),
    ("zrefined3d", 3, (7, 6, 4), [dict(lo=(2, 2, 1), hi=(5, 4, 3), r=(1, 1, 4))]),
    ("xgraded_wall3d", 3, (9, 6, 5), [dict(lo=(3, 0, 0), hi=(5, 6, 5), r=(5, 1, 1))]),
    ("aniso3d", 3, (8, 7, 6), [dict(lo=(2, 2, 2), hi=(5, 5, 4), r=(2, 3, 2))]),
    ("two_boxes2d", 2, (30, 20, 1), [dict(lo=(3, 3, 0), hi=(8, 9, 1), r=(3, 3, 1)),
                                    dict(lo=(15, 5, 0), hi=(22, 12, 1), r=(2, 2, 1))]),
]


@pytest.mark.parametrize("name,dim,n,boxes", CASES)
def test_prep_hybrid_equals_oracle(name, dim, n, boxes):
    if name == "tiny2d":
        scn = scenario("tiny2d")
        check(2, scn["n"], scn["eps_r"], scn["boxes"])
        return
    rng = np.random.default_rng(0)
    eps = rng.uniform(1, 3, (n[2], n[1], n[0]) if dim == 3 else (n[1], n[0]))
    check(dim, n, eps, boxes)


def test_prep_hybrid_with_pec_sheets_equals_oracle():
    # config-5-like: PEC plates crossing refined regions (z-refined), two
    # shared models; the oracle eliminates the plate edges independently
    from oracle.hybrid import sheet_pec
    from paper_1406_7042_b200.prep import _pec_extra
    scn = scenario("tiny5")
    P = fit.assemble(3, scn["n"], scn["delta"], scn["eps_r"], scn["boxes"], scn["eps0"], scn["mu0"],
                     pec_extra=_pec_extra(scn))
    ob = [hy.Box(tuple(b["lo"]), tuple(b["hi"]), tuple(b["r"])) for b in scn["boxes"]]
    O = hy.assemble(3, scn["n"], scn["delta"], scn["eps_r"], ob, scn["eps0"], scn["mu0"],
                    pec_e_extra=sheet_pec(scn["pec_sheets"], scn["boxes"]))
    S = P.S
    shp = fit.sshape(P.n, 3)

    def cflat(key):
        _, c, (i, j, k) = key
        return c * S + int(np.ravel_multi_index((k, j, i), shp))
    surf = sorted(cflat(O.e_keys[r]) for r in np.nonzero(O.e_tag == 1)[0])
    assert np.array_equal(np.array(surf), P.if_ids)
    # the plate edges are gone in both
    pecx = _pec_extra(scn)
    n_pec = sum(int(pecx(-1, c, shp).sum()) for c in (0, 1))
    assert n_pec > 0
    Kc = O.K.tocsr()
    for q, fid in enumerate(P.if_ids[::7]):
        c, s_ = int(fid // S), int(fid % S)
        k, j, i = np.unravel_index(s_, shp)
        r = O.e_index[("c", c, (int(i), int(j), int(k)))]
        assert abs(P.De_c[c].ravel()[s_] - O.De[r]) <= 1e-13 * O.De[r]
        row = Kc[r]
        ref = {cflat(O.h_keys[cc]): v for cc, v in zip(row.indices, row.data) if O.h_keys[cc][0] == "c"}
        qq = int(np.searchsorted(P.if_ids, fid))
        prow = P.W[qq]
        got = {int(cc): v for cc, v in zip(prow.indices, prow.data)}
        assert set(ref) == set(got)
        assert all(abs(ref[kk] - got[kk]) <= 1e-13 * abs(ref[kk]) for kk in ref)
    for bi, part in enumerate(P.boxes):
        nf = part.fine.n
        shf = fit.sshape(nf, 3)
        Sf = int(np.prod(shf))

        def fflat(key):
            _, b, c, (i, j, k) = key
            return c * Sf + int(np.ravel_multi_index((k, j, i), shf))
        oe = {fflat(O.e_keys[r]): r for r in np.nonzero((O.e_tag == 2) & (O.e_box == bi))[0]}
        assert set(oe) == set(part.e_int.tolist())
        pe = np.array([oe[v] for v in part.e_int])
        oh = {fflat(O.h_keys[r]): r for r in np.nonzero((O.h_tag == 2) & (O.h_box == bi))[0]}
        ph_ = np.array([oh[v] for v in part.h_int])
        assert abs(O.K[pe][:, ph_] - part.Kff).max() <= 1e-13 * abs(part.Kff).max()


def test_prep_hybrid_with_solid_pec_iris_equals_oracle():
    # config-4-like: x-graded slab over the full cross-section with a solid
    # PEC iris inside the refined region
    from oracle.hybrid import block_pec
    from paper_1406_7042_b200.prep import _pec_extra
    scn = scenario("tiny4")
    P = fit.assemble(3, scn["n"], scn["delta"], scn["eps_r"], scn["boxes"], scn["eps0"], scn["mu0"],
                     pec_extra=_pec_extra(scn))
    ob = [hy.Box(tuple(b["lo"]), tuple(b["hi"]), tuple(b["r"])) for b in scn["boxes"]]
    O = hy.assemble(3, scn["n"], scn["delta"], scn["eps_r"], ob, scn["eps0"], scn["mu0"],
                    pec_e_extra=block_pec(scn["boxes"]))
    part = P.boxes[0]
    nf = part.fine.n
    shf = fit.sshape(nf, 3)
    Sf = int(np.prod(shf))

    def fflat(key):
        _, b, c, (i, j, k) = key
        return c * Sf + int(np.ravel_multi_index((k, j, i), shf))
    oe = {fflat(O.e_keys[r]): r for r in np.nonzero(O.e_tag == 2)[0]}
    assert set(oe) == set(part.e_int.tolist())
    oh = {fflat(O.h_keys[r]): r for r in np.nonzero(O.h_tag == 2)[0]}
    pe = np.array([oe[v] for v in part.e_int]); ph_ = np.array([oh[v] for v in part.h_int])
    assert abs(O.K[pe][:, ph_] - part.Kff).max() <= 1e-13 * abs(part.Kff).max()
    assert np.allclose(O.De[pe], part.De_f, rtol=1e-13)
    # the iris removed fine E unknowns
    P0 = fit.assemble(3, scn["n"], scn["delta"], scn["eps_r"], scn["boxes"], scn["eps0"], scn["mu0"])
    assert len(P0.boxes[0].e_int) > len(part.e_int)
