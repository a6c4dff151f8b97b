"""Pins of oracle.problem_step - the recursion the GPU must match - against the
symmetric reduced-hybrid leap-frog of (4)/(12) assembled by oracle.hybrid."""
import numpy as np
import pytest

from oracle import hybrid as hy
from oracle import matrix_form as mf
from oracle import problem_step as ps
from oracle import reduction as rd
from synth import scenario

from oracle_problem import problem_from_oracle


def _symmetric_run(scn, hs, pr, n_steps, Kt=None, SEif=None):
    De, Dm, K = hy.reduced_system(pr, Kt, SEif)
    GE = scn["dt"] / np.diag(De)
    GH = scn["dt"] / np.diag(Dm)
    E = np.zeros(K.shape[0]); H = np.zeros(K.shape[1])
    ec = pr["ec"]
    src = scn["sources"]
    c, idx = int(src["comp"][0]), tuple(int(v) for v in src["idx"][0])
    row = int(np.nonzero(ec == hs.e_index[("c", c, idx)])[0][0])
    KT = K.T.tocsr()
    for s in range(n_steps):
        su = np.zeros(len(E))
        su[row] = -GE[row] * scn["delta"] * src["wave"][s, 0, 0]
        E, H = mf.step_leapfrog(E, H, GE, GH, K, KT, su_E=su)
    return E, H


@pytest.mark.parametrize("basis", ["identity", "random"])
def test_problem_step_matches_symmetric_hybrid(basis):
    scn = scenario("tiny2d", n_steps=300)
    V1 = V2 = None
    if basis == "random":
        # any full-rank basis: D-orthonormalised random columns (q = 24)
        from oracle import hybrid as _h
        boxes = [_h.Box(tuple(b["lo"]), tuple(b["hi"]), tuple(b["r"])) for b in scn["boxes"]]
        hs0 = _h.assemble(2, scn["n"], scn["delta"], scn["eps_r"], boxes, scn["eps0"], scn["mu0"])
        b = _h.blocks(hs0)
        rng = np.random.default_rng(11)
        V1 = rd.d_orthonormal(rng.standard_normal((len(b["ef"]), 24)), hs0.De[b["ef"]])
        V2 = rd.d_orthonormal(rng.standard_normal((len(b["hf"]), 24)), hs0.Dm[b["hf"]])
    prob, hs, pr = problem_from_oracle(scn, V1, V2)
    E, H, probes, rec = ps.run(prob, 300)
    Er, Hr = _symmetric_run(scn, hs, pr, 300)
    # map the symmetric ordering (coarse in hs order, then reduced) onto rec's
    Ne_c = len(rec.e_ids)
    fid = {}
    for pos, r in enumerate(pr["ec"]):
        key = hs.e_keys[r]
        fid[int(_flat(hs, key))] = pos
    perm = np.array([fid[int(u)] for u in rec.e_ids])
    assert np.linalg.norm(E[:Ne_c] - Er[perm]) <= 1e-12 * np.linalg.norm(Er)
    assert np.linalg.norm(E[Ne_c:] - Er[len(pr["ec"]):]) <= 1e-12 * np.linalg.norm(Er)
    assert np.linalg.norm(H[len(rec.h_ids):] - Hr[len(pr["hc"]):]) <= 1e-12 * np.linalg.norm(Hr)
    assert np.linalg.norm(Er) > 0


def _flat(hs, key):
    from oracle import yee
    shp = yee.storage_shape(hs.dim, hs.n)
    S = int(np.prod(shp))
    i, j, k = key[2]
    pos = np.ravel_multi_index((k, j, i) if hs.dim == 3 else (j, i), shp)
    return key[1] * S + int(pos)


def test_problem_step_pure_stencil_3d_equals_yee():
    # no boxes: the problem path is the plain Yee recursion of (4)
    from oracle import yee
    from oracle_problem import uniform_problem
    scn = scenario("tiny3d", n_steps=20)
    prob = uniform_problem(scn)
    E, H, _, rec = ps.run(prob, 20)
    s = yee.assemble(3, scn["n"], (scn["delta"],) * 3, scn["eps0"], scn["mu0"])
    x0 = np.zeros(s.Ne + s.Nh)
    arrs = {c: np.asarray(scn["init"][c]).reshape(yee.storage_shape(3, scn["n"])) for c in (0, 1, 2)}
    for c in (3, 4, 5):
        arrs[c] = np.zeros(yee.storage_shape(3, scn["n"]))
    x0 = s.from_storage(arrs)
    R, F = mf.build_RF(s.De, s.Dm, s.K, s.Dse, s.Dsm, scn["dt"])
    x = x0
    for _ in range(20):
        x = mf.step_literal(x, R, F, np.zeros_like(x))
    st, _, _ = ps.to_storage(rec, E, H)
    got = s.from_storage({c: st.get(c, np.zeros(rec.S)).reshape(yee.storage_shape(3, scn["n"]))
                          for c in range(6)})
    assert np.linalg.norm(got - x) <= 1e-12 * np.linalg.norm(x)
