"""Pins of oracle.hybrid (reading R4: coarse grid + refined box as one system of
form (3)) and of the split enforcement (reading R7)."""
import math

import numpy as np
import pytest
import scipy.sparse as sp

from oracle import hybrid as hy
from oracle import matrix_form as mf
from oracle import physics as ph
from oracle import reduction as rd
from oracle import stability as st
from oracle import yee
from synth import C0, EPS0, MU0

CG = 1 / math.sqrt(EPS0 * MU0)


def _yee_scaled(dim, n, d, eps_cell):
    s = yee.assemble(dim, n, (d, d, d), EPS0, MU0, eps_r=eps_cell)
    # paper form x delta -> K = +-1, D = eps*delta, mu*delta
    return s, s.K * d, s.De * d, s.Dm * d


def _key_to_yee(s, key):
    _, comp, idx = key
    i, j, k = idx
    return int(s.index[comp][(k, j, i)] if s.dim == 3 else s.index[comp][(j, i)])


@pytest.mark.parametrize("dim,n", [(2, (9, 7, 1)), (3, (5, 4, 3))])
def test_no_box_equals_uniform_yee(dim, n):
    rng = np.random.default_rng(0)
    eps = rng.uniform(1, 3, (n[2], n[1], n[0]) if dim == 3 else (n[1], n[0]))
    d = 1e-3
    hs = hy.assemble(dim, n, d, eps, [], EPS0, MU0)
    s, K, De, Dm = _yee_scaled(dim, n, d, eps)
    pe = np.array([_key_to_yee(s, k) for k in hs.e_keys])
    ph_ = np.array([_key_to_yee(s, k) for k in hs.h_keys])
    assert sorted(pe) == list(range(s.Ne)) and sorted(ph_) == list(range(s.Nh))
    assert np.allclose(hs.De, De[pe], rtol=1e-14)
    assert np.allclose(hs.Dm, Dm[ph_], rtol=1e-14)
    Kh = hs.K.toarray()
    Ky = K.toarray()[np.ix_(pe, ph_)]
    assert np.allclose(Kh, Ky, rtol=1e-14, atol=1e-14)


@pytest.mark.parametrize("dim,n,box", [
    (2, (11, 9, 1), hy.Box((3, 2, 0), (7, 6, 1), (1, 1, 1))),
    (3, (7, 6, 5), hy.Box((2, 1, 1), (5, 4, 3), (1, 1, 1)))])
def test_ratio_one_box_reproduces_uniform_grid(dim, n, box):
    # reading R4 with r = 1: the glued system is exactly the uniform Yee grid
    rng = np.random.default_rng(1)
    eps = rng.uniform(1, 3, (n[2], n[1], n[0]) if dim == 3 else (n[1], n[0]))
    d = 1e-3
    hs = hy.assemble(dim, n, d, eps, [box], EPS0, MU0)
    s, K, De, Dm = _yee_scaled(dim, n, d, eps)

    def ykey(key):
        if key[0] == "c":
            return _key_to_yee(s, key)
        _, b, comp, fidx = key
        idx = tuple(box.lo[a] + fidx[a] for a in range(3)) if dim == 3 else \
            (box.lo[0] + fidx[0], box.lo[1] + fidx[1], 0)
        return _key_to_yee(s, ("c", comp, idx))

    pe = np.array([ykey(k) for k in hs.e_keys])
    ph_ = np.array([ykey(k) for k in hs.h_keys])
    assert sorted(pe) == list(range(s.Ne)) and sorted(ph_) == list(range(s.Nh))
    assert np.allclose(hs.De, De[pe], rtol=1e-13)
    assert np.allclose(hs.Dm, Dm[ph_], rtol=1e-13)
    assert np.allclose(hs.K.toarray(), K.toarray()[np.ix_(pe, ph_)], rtol=1e-13, atol=1e-13)


def _config1_hybrid():
    box = hy.Box((16, 6, 0), (24, 14, 1), (4, 4, 1))
    return hy.assemble(2, (40, 20, 1), 1e-3, np.ones((20, 40)), [box], EPS0, MU0)


def test_config1_counts_and_structure_F10():
    hs = _config1_hybrid()
    ne_c = int(np.sum(hs.e_tag < 2)); ne_f = int(np.sum(hs.e_tag == 2))
    nh_c = int(np.sum(hs.h_tag < 2)); nh_f = int(np.sum(hs.h_tag == 2))
    assert (ne_c, ne_f, hs.Ne, hs.Nh) == (692, 961, 1653, 3412)     # survey F10
    assert int(np.sum(hs.e_tag == 1)) == 32                           # n_if = 32
    assert nh_c + nh_f == 3412
    b = hy.blocks(hs)
    assert b["Kfc"].nnz == 0 or abs(b["Kfc"]).max() == 0.0             # K_fc = 0
    assert np.all(hs.De > 0) and np.all(hs.Dm > 0)
    d, delta = 1e-3, 0.25e-3
    # lumped interface mass on a non-corner side node: eps (d + delta)/2 (scaled)
    i = hs.e_index[("c", 2, (16, 9, 0))]
    assert math.isclose(hs.De[i], EPS0 * (d + delta) / 2, rel_tol=1e-14)
    # surface H rows keep the regular update coefficient: K_ij / D_mu,j = +-1/(mu d)
    Kc = hs.K.tocsc()
    for j in np.nonzero(hs.h_tag == 1)[0]:
        col = Kc[:, j].toarray().ravel()
        nz = col[col != 0]
        assert len(nz) == 2
        assert np.allclose(np.abs(nz) / hs.Dm[j], 1 / (MU0 * d), rtol=1e-13)
    # regular coarse rows: +-1 and eps*d
    reg = np.nonzero(hs.e_tag == 0)[0]
    assert np.allclose(hs.De[reg], EPS0 * d, rtol=1e-15)
    assert set(np.unique(np.abs(hs.K[reg].data))) == {1.0}


def test_config1_exact_limit_and_spectrum_F10():
    hs = _config1_hybrid()
    dt_max = st.exact_dt_max(hs.De, hs.K, hs.Dm)
    fine_cfl = 0.25e-3 / (CG * math.sqrt(2))
    assert 1.0 <= dt_max / fine_cfl <= 1.02          # F10: 0.17699 vs 0.17678
    # semi-discrete resonances (omega = sigma) vs analytic TM modes of the 40x20 mm
    # cavity: within 0.5 % for the lowest modes (F10: 0.1-0.5 %)
    sig = np.sort(st.singular_values(hs.De, hs.K, hs.Dm))
    f = sig[sig > 1e6] / (2 * math.pi)
    ana = ph.cavity_modes((0.04, 0.02), C0, count=10, dim=2)
    got = np.unique(np.round(f[:16], -4))[:8]      # (2,2) and (4,1) are degenerate
    err = np.array([np.min(np.abs(g / ana - 1)) for g in got])
    assert np.all(err < 5e-3)
    assert got[0] / ana[0] - 1 < 2e-3


def test_hybrid_energy_conserved():
    hs = _config1_hybrid()
    dt = 0.99 * st.exact_dt_max(hs.De, hs.K, hs.Dm)
    R, F = mf.build_RF(hs.De, hs.Dm, hs.K, np.zeros(hs.Ne), np.zeros(hs.Nh), dt)
    rng = np.random.default_rng(2)
    E = rng.standard_normal(hs.Ne); H = rng.standard_normal(hs.Nh) * 2.6e-3
    e0 = mf.energy(np.concatenate([E, H]), R)
    KT = hs.K.T.tocsr()
    for _ in range(1000):
        E, H = mf.step_leapfrog(E, H, dt / hs.De, dt / hs.Dm, hs.K, KT)
    assert abs(mf.energy(np.concatenate([E, H]), R) / e0 - 1) < 1e-10


def _small_hybrid():
    box = hy.Box((5, 4, 0), (11, 8, 1), (3, 3, 1))
    rng = np.random.default_rng(7)
    eps = np.ones((12, 16)); eps[2:6, 9:14] = 2.5
    return hy.assemble(2, (16, 12, 1), 1e-3, eps, [box], EPS0, MU0)


def test_naive_clipping_unstable_split_enforcement_stable_F7():
    # reading R7 / survey F7: at dt = 2x fine CFL clipping only K~_rr leaves the
    # coupled hybrid unstable; clipping the local block [K~_rr; S_E] with the
    # split interface mass makes every update eigenvalue |lambda| <= 1.
    hs = _small_hybrid()
    d, r = 1e-3, 3
    dt = 2.0 * (d / r) / (CG * math.sqrt(2))
    dtc = d / (CG * math.sqrt(2))
    b = hy.blocks(hs)
    # identity basis (the unreduced hybrid) -- the strongest case
    V1, V2 = np.eye(len(b["ef"])), np.eye(len(b["hf"]))
    pr = hy.project(hs, V1, V2)
    De, Dm, K = hy.reduced_system(pr)
    R, F = mf.build_RF(np.diag(De), np.diag(Dm), K, np.zeros(len(De)), np.zeros(len(Dm)), dt)
    assert np.max(np.abs(mf.update_eigenvalues(R, F))) > 1.01
    # naive: §III-A on K~_rr alone
    Kn, _ = st.enforce(np.diag(pr["Dt_e"]), pr["Kt_rr"], np.diag(pr["Dt_m"]), dt)
    De, Dm, K = hy.reduced_system(pr, Kt_rr=Kn)
    R, F = mf.build_RF(np.diag(De), np.diag(Dm), K, np.zeros(len(De)), np.zeros(len(Dm)), dt)
    assert np.max(np.abs(mf.update_eigenvalues(R, F))) > 1.01
    # split enforcement
    alpha = st.split_alpha(dt, dtc)
    SEif = np.asarray(pr["S_E"])[pr["if_rows"]]
    Kp, SEp, rep = st.enforce_hybrid_block(np.diag(pr["Dt_e"]), pr["Kt_rr"], SEif,
                                           np.diag(pr["Dt_m"]), pr["De_c"][pr["if_rows"]],
                                           alpha, dt)
    assert rep["n_clipped"] > 0
    sc = st.coarse_piece_sigma_max(pr["De_c"], pr["Dm_c"], pr["Kcc"], pr["if_rows"], alpha)
    assert sc < 2 / dt
    De, Dm, K = hy.reduced_system(pr, Kt_rr=Kp, S_E_if=SEp)
    R, F = mf.build_RF(np.diag(De), np.diag(Dm), K, np.zeros(len(De)), np.zeros(len(Dm)), dt)
    lam = np.abs(mf.update_eigenvalues(R, F))
    assert np.max(lam) <= 1 + 1e-9
    assert np.max(np.abs(lam - 1)) < 1e-9            # lossless: on the unit circle
    assert st.is_R_positive_definite(R)


def test_split_enforcement_noop_when_below_limits():
    # with n_if = 0 the split enforcement is exactly §III-A; below the limit it is a no-op
    rng = np.random.default_rng(8)
    q = 10
    Kt = rng.standard_normal((q, q))
    dt = 0.5 * 2 / np.linalg.svd(Kt, compute_uv=False)[0]
    Kp, SEp, rep = st.enforce_hybrid_block(np.ones(q), Kt, np.zeros((0, q)), np.ones(q),
                                           np.zeros(0), 0.3, dt)
    assert rep["n_clipped"] == 0 and np.allclose(Kp, Kt, rtol=1e-12)
    Kp2, _ = st.enforce(np.ones(q), Kt, np.ones(q), 4 * dt)
    Kp3, _, _ = st.enforce_hybrid_block(np.ones(q), Kt, np.zeros((0, q)), np.ones(q),
                                        np.zeros(0), 0.3, 4 * dt)
    assert np.allclose(Kp2, Kp3, rtol=1e-13)


def test_3d_single_axis_refinement_structure():
    # config-5-like box refined 10x... (reduced here to r_z = 4) in z only:
    # K_fc = 0, D_mu diagonal positive, exact limit near the fine CFL limit
    box = hy.Box((2, 2, 1), (5, 4, 3), (1, 1, 4))
    hs = hy.assemble(3, (7, 6, 4), 1e-3, np.ones((4, 6, 7)), [box], EPS0, MU0)
    b = hy.blocks(hs)
    assert b["Kfc"].nnz == 0 or abs(b["Kfc"]).max() == 0.0
    assert np.all(hs.De > 0) and np.all(hs.Dm > 0)
    dt_max = st.exact_dt_max(hs.De, hs.K, hs.Dm)
    d = 1e-3
    fine = 1 / (CG * math.sqrt(1 / d ** 2 + 1 / d ** 2 + (4 / d) ** 2))
    assert 0.95 < dt_max / fine < 1.3
    # energy conservation below the limit
    dt = 0.98 * dt_max
    R, F = mf.build_RF(hs.De, hs.Dm, hs.K, np.zeros(hs.Ne), np.zeros(hs.Nh), dt)
    lam = np.abs(mf.update_eigenvalues(R, F))
    assert np.max(np.abs(lam - 1)) < 1e-9
