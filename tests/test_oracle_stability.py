"""Pins of oracle.stability / oracle.reduction / oracle.physics: the §III-B
eigenvalue demo, the §III-A enforcement laws, congruence (§II-D) and the
cube resonances the paper prints."""
import math

import numpy as np
import pytest
import scipy.sparse as sp

from oracle import matrix_form as mf
from oracle import physics as ph
from oracle import reduction as rd
from oracle import stability as st
from oracle import yee
from synth import C0, EPS0, MU0

CG = 1 / math.sqrt(EPS0 * MU0)


def _cube(N=9):
    d = 1.0 / N                      # reading R-A9: Delta = 1/9 m
    s = yee.assemble(3, (N, N, N), (d, d, d), EPS0, MU0)
    return s, d


def test_cube_demo_s099_stable_s198_unstable():
    # §III-B (Fig. 1): s = 0.99 below CFL -> R > 0, |lambda| <= 1;
    # s = 1.98 -> some eigenvalues leave the unit circle.
    s, d = _cube(9)
    dtc = st.cfl_dt((d, d, d), CG)
    sig = st.singular_values(s.De, s.K, s.Dm)
    R, F = mf.build_RF(s.De, s.Dm, s.K, s.Dse, s.Dsm, 0.99 * dtc)
    assert sig[0] < 2 / (0.99 * dtc)
    assert st.is_R_positive_definite(R)
    lam = np.abs(mf.update_eigenvalues(R, F))           # dense, 3672 x 3672
    assert np.max(np.abs(lam - 1.0)) < 1e-9             # lossless: on the unit circle
    R2, F2 = mf.build_RF(s.De, s.Dm, s.K, s.Dse, s.Dsm, 1.98 * dtc)
    assert not st.is_R_positive_definite(R2)
    lam2 = np.max(np.abs(mf.update_eigenvalues(R2, F2)))
    assert 13.0 < lam2 < 13.3                           # survey F11 measured 13.13
    # the exact limit exceeds Eq. (1) by the closed-form factor (F11: 1.0154 at 9^3)
    assert 1.0 < st.exact_dt_max(s.De, s.K, s.Dm) / dtc < 1.03


def test_cube_demo_enforced_on_unit_circle():
    # §III-A applied to the full system (Fig. 2): after enforcement
    # every eigenvalue is on the unit circle (lossless), none outside.
    s, d = _cube(9)
    dt = 1.98 * st.cfl_dt((d, d, d), CG)
    Kp, rep = st.enforce(s.De, s.K, s.Dm, dt)
    assert rep["n_clipped"] > 0                     # F11: 1051 of 1728
    assert rep["n_clipped"] == 1051
    R, F = mf.build_RF(s.De, s.Dm, sp.csr_matrix(Kp), s.Dse, s.Dsm, dt)
    lam = np.abs(mf.update_eigenvalues(R, F))
    assert np.max(np.abs(lam - 1.0)) < 1e-9             # on the unit circle
    assert st.is_R_positive_definite(R)


def test_small_cube_all_eigenvalues_on_unit_circle():
    # brute force on the whole spectrum (dense eig) for a 5^3 cube at s = 1.98
    s, d = _cube(5)
    dt = 1.98 * st.cfl_dt((d, d, d), CG)
    Kp, rep = st.enforce(s.De, s.K, s.Dm, dt)
    R, F = mf.build_RF(s.De, s.Dm, sp.csr_matrix(Kp), s.Dse, s.Dsm, dt)
    lam = mf.update_eigenvalues(R, F)
    assert np.max(np.abs(np.abs(lam) - 1.0)) < 1e-9
    R0, F0 = mf.build_RF(s.De, s.Dm, s.K, s.Dse, s.Dsm, dt)
    assert np.max(np.abs(mf.update_eigenvalues(R0, F0))) > 1.0 + 1e-3


def test_enforcement_laws_S348_S365():
    rng = np.random.default_rng(3)
    q = 30
    K = rng.standard_normal((q, q)) * 5
    De = rd.d_orthonormal(np.eye(q), np.eye(q))   # identity
    Dt_e = np.diag(rng.uniform(1, 2, q))
    A = rng.standard_normal((q, q)); Dt_m = A @ A.T + q * np.eye(q)
    sig = st.singular_values(Dt_e, K, Dt_m)
    # no-op when nothing violates
    dt_ok = 0.5 * 2 / sig[0]
    Kp, rep = st.enforce(Dt_e, K, Dt_m, dt_ok)
    assert rep["n_clipped"] == 0
    assert np.linalg.norm(Kp - K) <= 1e-10 * np.linalg.norm(K)
    # clipping regime
    dt = 2.0 / sig[q // 3]
    Kp, rep = st.enforce(Dt_e, K, Dt_m, dt)
    s_new = st.singular_values(Dt_e, Kp, Dt_m)
    lim = 0.9999 * 2 / dt                          # gamma = 0.9999
    assert rep["n_clipped"] == int(np.sum(sig >= lim))
    assert math.isclose(s_new[0], min(sig[0], lim), rel_tol=1e-10)
    # idempotent
    Kpp, _ = st.enforce(Dt_e, Kp, Dt_m, dt)
    assert np.linalg.norm(Kpp - Kp) <= 1e-10 * np.linalg.norm(Kp)
    # perturbation bounded by the clipped excess in the scaled norm
    A0 = st.scaled_curl(Dt_e, K, Dt_m)
    A1 = st.scaled_curl(Dt_e, Kp, Dt_m)
    assert np.linalg.norm(A1 - A0, 2) <= np.sum(np.maximum(sig - lim, 0)) + 1e-9 * sig[0]
    # matrix square root choice does not matter (F5): Cholesky factors instead
    Lc = np.linalg.cholesky(Dt_m)
    Ae = np.diag(np.diag(Dt_e) ** -0.5) @ K @ np.linalg.inv(Lc).T
    U, s, Wt = np.linalg.svd(Ae)
    s2 = np.minimum(s, lim)
    Kc = np.diag(np.diag(Dt_e) ** 0.5) @ (U * s2) @ Wt @ Lc.T
    assert np.linalg.norm(Kc - Kp) <= 1e-12 * np.linalg.norm(Kp)


def test_reduced_update_angles_F4():
    # with D~ = I and no loss the update eigenvalues are exp(+-j theta_i),
    # theta_i = 2 arcsin(dt sigma_i / 2)
    rng = np.random.default_rng(4)
    q = 12
    K = rng.standard_normal((q, q))
    sig = np.linalg.svd(K, compute_uv=False)
    dt = 1.5 / sig[0]
    R, F = mf.build_RF(np.ones(q), np.ones(q), sp.csr_matrix(K), np.zeros(q), np.zeros(q), dt)
    lam = mf.update_eigenvalues(R, F)
    ang = np.sort(np.abs(np.angle(lam)))
    ref = np.sort(np.concatenate([2 * np.arcsin(dt * sig / 2)] * 2))
    assert np.allclose(np.abs(lam), 1.0, atol=1e-12)
    assert np.allclose(ang, ref, atol=1e-10)


def test_congruence_structure_and_stability_below_cfl_S297_S300():
    # any full-rank block-diagonal V: R~ from (13) equals V^T R V; below the CFL
    # limit R~ > 0 and the reduced spectrum is in the unit disk (§II-D)
    s = yee.assemble(2, (9, 7, 1), (1e-3, 1e-3, 1.0), EPS0, MU0)
    dt = 0.97 * st.cfl_dt((1e-3, 1e-3), CG)
    rng = np.random.default_rng(5)
    Dse = rng.uniform(0, 0.05, s.Ne)
    R, F = mf.build_RF(s.De, s.Dm, s.K, Dse, s.Dsm, dt)
    for q in (5, 17):
        V1 = rd.random_orthonormal(s.Ne, q, rng)
        V2 = rd.random_orthonormal(s.Nh, q, rng)
        red = rd.project(V1, V2, s.De, s.Dm, s.K, Dse, s.Dsm)
        Rr, Fr = mf.build_RF(red["De"], red["Dm"], red["K"], red["Dse"], red["Dsm"], dt)
        V = sp.block_diag([V1, V2]).toarray()
        assert np.allclose(Rr.toarray(), V.T @ R.toarray() @ V, rtol=0, atol=1e-10 * abs(R).max())
        assert np.allclose(Fr.toarray(), V.T @ F.toarray() @ V, rtol=0, atol=1e-10 * abs(F).max())
        assert st.is_R_positive_definite(Rr)
        assert np.min(np.linalg.eigvalsh((Fr + Fr.T).toarray())) >= -1e-12 * abs(F).max()
        assert np.max(np.abs(mf.update_eigenvalues(Rr, Fr))) <= 1 + 1e-10


def test_identity_and_square_basis_transfer_function_S286_S295():
    s = yee.assemble(2, (6, 5, 1), (1e-3, 1e-3, 1.0), EPS0, MU0)
    dt = 0.9 * st.cfl_dt((1e-3, 1e-3), CG)
    R, F = mf.build_RF(s.De, s.Dm, s.K, s.Dse, s.Dsm, dt)
    N = s.Ne + s.Nh
    B = np.zeros((N, 1)); B[3, 0] = -1.0
    C = np.zeros((N, 1)); C[7, 0] = 1.0
    # identity projection reproduces the original matrices
    red = rd.project(np.eye(s.Ne), np.eye(s.Nh), s.De, s.Dm, s.K, s.Dse, s.Dsm, B)
    assert np.array_equal(red["K"], s.K.toarray())
    assert np.allclose(red["De"], np.diag(s.De), rtol=1e-15)
    # a square orthogonal block-diagonal V is a change of basis: identical
    # transfer function at every expansion point of Eq. (19)
    rng = np.random.default_rng(6)
    V1 = rd.random_orthonormal(s.Ne, s.Ne, rng)
    V2 = rd.random_orthonormal(s.Nh, s.Nh, rng)
    redV = rd.project(V1, V2, s.De, s.Dm, s.K, s.Dse, s.Dsm, B)
    Rr, Fr = mf.build_RF(redV["De"], redV["Dm"], redV["K"], redV["Dse"], redV["Dsm"], dt)
    Vs = sp.block_diag([V1, V2]).toarray()
    for z in rd.expansion_points(1.1, 2, 30e9, dt):
        h_full = rd.transfer(R, F, B, C, z)
        h_red = rd.transfer(Rr.toarray(), Fr.toarray(), redV["B"], Vs.T @ C, z)
        assert np.allclose(h_red, h_full, rtol=1e-9)


def test_expansion_points_eq19():
    dt = 1e-12
    z = rd.expansion_points(1.1, 2, 30e9, dt)
    assert len(z) == 5                                  # P:423 "Five expansion points"
    assert np.isclose(z[2], 1.1)                        # l = 0 -> M
    assert np.allclose(np.abs(z), 1.1)
    assert np.allclose(z[::-1], np.conj(z))             # z_{-l} = conj(z_l)
    assert np.allclose(rd.expansion_points(1.1, 0, 30e9, dt), [1.1])
    # the angles of Eq. (19), evaluated by hand: f_max dt = 0.03, so
    # l = 1: 2 pi (1/2) 0.03 = 0.0942478 rad, 1.1 (cos, sin) = (1.0951182, 0.1035191)
    # l = 2: 2 pi (2/2) 0.03 = 0.1884956 rad, 1.1 (cos, sin) = (1.0805160, 0.2061194)
    # (a wrong angle -- a dropped 2 pi, l instead of l/L, f_max instead of
    # f_max dt -- moves these)
    want = [1.0805160 - 0.2061194j, 1.0951182 - 0.1035191j, 1.1 + 0j,
            1.0951182 + 0.1035191j, 1.0805160 + 0.2061194j]
    assert np.allclose(z, want, rtol=0, atol=2e-7)


def test_cube_resonances_P311():
    # 1 m PEC cube: analytic (1,1,0) = 0.21199 GHz and (1,1,1) = 0.25963 GHz
    # (P:311); the discrete leap-frog at s = 0.99 is within 1 %.
    modes = ph.cavity_modes((1.0, 1.0, 1.0), C0, count=2, dim=3)
    assert np.allclose(modes / 1e9, [0.21199, 0.25963], atol=5e-6)
    s, d = _cube(9)
    dt = 0.99 * st.cfl_dt((d, d, d), CG)
    sig = np.sort(st.singular_values(s.De, s.K, s.Dm))
    f = np.unique(np.round(ph.discrete_frequency(sig[sig > 1], dt), 1))
    f = f[f > 0.1e9]
    assert abs(f[0] / 0.21199e9 - 1) < 0.01 and abs(f[1] / 0.25963e9 - 1) < 0.01


@pytest.mark.slow
def test_cube_time_domain_peaks():
    # run the cube demo in the time domain (Gaussian, fmax 0.3 GHz) and
    # find the two resonances in the probe spectrum within 1 %
    s, d = _cube(9)
    dt = 0.99 * st.cfl_dt((d, d, d), CG)
    tau = math.sqrt(2 * math.log(10)) / (2 * math.pi * 0.3e9)
    n = 12000
    src = s.index[2][2, 3, 2]          # an off-centre Ez edge
    prb = s.index[2][6, 5, 7]
    E, H = np.zeros(s.Ne), np.zeros(s.Nh)
    GE, GH = dt / s.De, dt / s.Dm
    KT = s.K.T.tocsr()
    rec = np.zeros(n)
    for k in range(n):
        t = (k + 0.5) * dt
        su = np.zeros(s.Ne)
        su[src] = -GE[src] * math.exp(-((t - 4 * tau) ** 2) / (2 * tau * tau))
        E, H = mf.step_leapfrog(E, H, GE, GH, s.K, KT, su_E=su)
        rec[k] = E[prb]
    f, mag = ph.spectrum(rec, dt, window="hann")
    pk = ph.find_peaks(f, mag, prominence=0.02, fmin=0.15e9, fmax=0.3e9)
    for target in (0.21199e9, 0.25963e9):
        assert np.min(np.abs(pk / target - 1)) < 0.01
