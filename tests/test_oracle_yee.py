"""Pins of oracle.yee / oracle.matrix_form against what the paper and the
mathematics fix (not against the oracle's own formulas)."""
import math

import numpy as np
import pytest
import scipy.sparse as sp

from oracle import matrix_form as mf
from oracle import stability as st
from oracle import yee
from synth import C0, EPS0, MU0


def test_1d_K_pattern_S109():
    # 3 E-nodes / 2 H-nodes, dz = 1: rows {(+1), (-1,+1), (-1)}
    K, De, Dm = yee.line_1d(2, 1.0, EPS0, MU0, eliminate_ends=False)
    assert np.array_equal(K.toarray(), np.array([[1.0, 0.0], [-1.0, 1.0], [0.0, -1.0]]))
    assert np.all(De == EPS0) and np.all(Dm == MU0)      # S:110 vacuum D


def test_2d_system_size_table1():
    # Table I: 2-D cavity 101 x 101 cells -> N = 30,200
    s = yee.assemble(2, (101, 101, 1), (0.01, 0.01, 0.01), EPS0, MU0)
    assert s.Ne + s.Nh == 30200


def test_cube_demo_unknown_counts():
    # 9^3 PEC cube with tangential E / normal H eliminated: 3*9*8*8 and 3*8*9*9
    s = yee.assemble(3, (9, 9, 9), (1 / 9,) * 3, EPS0, MU0)
    assert (s.Ne, s.Nh) == (1728, 1944)


@pytest.mark.parametrize("dim,n", [(2, (7, 5, 1)), (3, (4, 3, 5))])
def test_H_rows_carry_K_transpose(dim, n):
    # (3) P:78-96: the E rows use K, the H rows use K^T of the same matrix.  K is
    # built from Ampere's law, the H operator independently from Faraday's.
    s = yee.assemble(dim, n, (1e-3, 2e-3, 1.5e-3), EPS0, MU0)
    assert abs(s.L - s.K.T).max() == 0.0
    # every entry of K is +-1/d_axis
    vals = np.unique(np.abs(s.K.data))
    allowed = {1 / 1e-3, 1 / 2e-3, 1 / 1.5e-3}
    assert all(min(abs(v - a) for a in allowed) < 1e-9 * v for v in vals)


def _one_step_map_1d(nz, dz, dt, printed_2b):
    """Dense one-step map of the 1-D line: (2a) for E, then (2b) either as
    printed (mu dH/dt = +(E_{k+1}-E_k)/dz) or as implied by (3) (= K^T E)."""
    K, De, Dm = yee.line_1d(nz, dz, EPS0, MU0)
    K = K.toarray()
    Ne, Nh = K.shape
    # E^{n+1} = E + dt/eps (-K H);  H^{n+1} = H + dt/mu (S E^{n+1})
    A = np.zeros((Ne + Nh, Ne + Nh))
    A[:Ne, :Ne] = np.eye(Ne)
    A[:Ne, Ne:] = -(dt / EPS0) * K
    S = (-K.T) if printed_2b else K.T          # printed (2b) has the opposite curl sign
    A[Ne:, :] = (dt / MU0) * S @ A[:Ne, :]
    A[Ne:, Ne:] += np.eye(Nh)
    return A


def test_eq2b_printed_sign_is_unstable_F1():
    # reading R1(i): Eq. (2b) as printed is inconsistent with (3).  At
    # dt = 0.9 dz / c the (3) leap-frog has all |lambda| = 1, the printed one
    # grows (survey F1 measured 4.87).
    nz, dz = 40, 1e-3
    dt = 0.9 * dz / C0
    lam_ok = np.abs(np.linalg.eigvals(_one_step_map_1d(nz, dz, dt, False)))
    lam_bad = np.abs(np.linalg.eigvals(_one_step_map_1d(nz, dz, dt, True)))
    assert np.max(np.abs(lam_ok - 1.0)) < 1e-9
    assert np.max(lam_bad) > 2.0


def test_cfl_values_S51_53():
    # S:51-53 evaluated from Eq. (1) by hand
    assert math.isclose(st.cfl_dt((0.02, 0.02, 0.02), C0), 3.8517e-11, rel_tol=1e-4)
    assert math.isclose(st.cfl_dt((0.01, 0.01), C0), 2.3587e-11, rel_tol=1e-4)
    assert math.isclose(st.cfl_dt((0.01, 0.01), C0 / 2.0), 2 * st.cfl_dt((0.01, 0.01), C0),
                        rel_tol=1e-15)


def test_2d_singular_values_closed_form_F2():
    # Dirichlet Laplacian spectrum: sigma_mn = 2c sqrt(sin^2(m pi/2Nx)/dx^2 +
    # sin^2(n pi/2Ny)/dy^2), m < Nx, n < Ny (survey F2; textbook result)
    Nx, Ny, dx, dy = 7, 5, 1e-3, 1.3e-3
    s = yee.assemble(2, (Nx, Ny, 1), (dx, dy, 1.0), EPS0, MU0)
    sig = np.sort(st.singular_values(s.De, s.K, s.Dm))
    c = 1 / math.sqrt(EPS0 * MU0)
    ref = np.sort([2 * c * math.sqrt(math.sin(m * math.pi / (2 * Nx)) ** 2 / dx ** 2 +
                                      math.sin(n * math.pi / (2 * Ny)) ** 2 / dy ** 2)
                   for m in range(1, Nx) for n in range(1, Ny)])
    sig = sig[-len(ref):]
    assert np.allclose(sig, ref, rtol=1e-12)
    # exact limit 2/sigma_max lies above Eq. (1)'s CFL ((8) <=> CFL)
    assert st.exact_dt_max(s.De, s.K, s.Dm) > st.cfl_dt((dx, dy), c)


def test_3d_singular_values_closed_form_F11():
    # nonzero sigma = (2c/d) sqrt(sum sin^2(m_i pi / 2N)), >= 2 indices nonzero,
    # multiplicity 2 when all three are nonzero (survey F11)
    N, d = 5, 1 / 9
    s = yee.assemble(3, (N, N, N), (d, d, d), EPS0, MU0)
    sig = np.sort(st.singular_values(s.De, s.K, s.Dm))
    c = 1 / math.sqrt(EPS0 * MU0)
    ref = []
    for m in range(N):
        for n in range(N):
            for p in range(N):
                nz = (m > 0) + (n > 0) + (p > 0)
                if nz < 2:
                    continue
                v = 2 * c / d * math.sqrt(sum(math.sin(t * math.pi / (2 * N)) ** 2 for t in (m, n, p)))
                ref += [v] * (2 if nz == 3 else 1)
    ref = np.sort(ref)
    nonzero = sig[sig > 1e-6 * sig.max()]
    assert len(nonzero) == len(ref)
    assert np.allclose(nonzero, ref, rtol=1e-10)


def _random_system(rng, Ne, Nh, lossy):
    K = sp.random(Ne, Nh, density=0.3, random_state=rng.integers(1 << 30)).toarray()
    De = rng.uniform(1, 2, Ne)
    Dm = rng.uniform(1, 2, Nh)
    Dse = rng.uniform(0, 1, Ne) if lossy else np.zeros(Ne)
    Dsm = rng.uniform(0, 1, Nh) if lossy else np.zeros(Nh)
    return De, Dm, sp.csr_matrix(K), Dse, Dsm


@pytest.mark.parametrize("lossy", [False, True])
def test_leapfrog_equals_dense_solve_S185(lossy):
    # the two-sweep leap-frog equals the algebraic solve of (4)
    rng = np.random.default_rng(0)
    for trial in range(5):
        Ne, Nh = int(rng.integers(5, 60)), int(rng.integers(5, 60))
        De, Dm, K, Dse, Dsm = _random_system(rng, Ne, Nh, lossy)
        dt = 0.3
        R, F = mf.build_RF(De, Dm, K, Dse, Dsm, dt)
        B = rng.standard_normal((Ne + Nh, 2))
        u = rng.standard_normal(2)
        x = rng.standard_normal(Ne + Nh)
        ref = mf.step_literal(x, R, F, B @ u)
        GE = 1.0 / (De / dt + Dse / 2)
        GH = 1.0 / (Dm / dt + Dsm / 2)
        Bu = B @ u
        # G B u split: E part solved first; H part sees the E increment through K^T
        E1, H1 = mf.step_leapfrog(x[:Ne], x[Ne:], GE, GH, K, K.T.tocsr(), Dse, Dsm,
                                  su_E=GE * Bu[:Ne], su_H=GH * Bu[Ne:])
        # the E source increment also enters H via K^T E^{n+1}; step_leapfrog
        # already uses E1 (which contains it), so the two must agree
        got = np.concatenate([E1, H1])
        assert np.linalg.norm(got - ref) <= 1e-12 * np.linalg.norm(ref)


def test_energy_conserved_lossless_F3():
    # x^T R x is invariant for the lossless recursion (F3)
    s = yee.assemble(2, (24, 17, 1), (1e-3, 1e-3, 1.0), EPS0, MU0)
    dt = 0.95 * st.cfl_dt((1e-3, 1e-3), 1 / math.sqrt(EPS0 * MU0))
    R, F = mf.build_RF(s.De, s.Dm, s.K, s.Dse, s.Dsm, dt)
    rng = np.random.default_rng(1)
    E = rng.standard_normal(s.Ne)
    H = rng.standard_normal(s.Nh) * math.sqrt(EPS0 / MU0)
    e0 = mf.energy(np.concatenate([E, H]), R)
    GE, GH = dt / s.De, dt / s.Dm
    KT = s.K.T.tocsr()
    for _ in range(1000):
        E, H = mf.step_leapfrog(E, H, GE, GH, s.K, KT)
    e1 = mf.energy(np.concatenate([E, H]), R)
    assert abs(e1 - e0) / abs(e0) < 1e-10


def test_1d_impulse_S172():
    # S:172 hand-evaluates the printed (2b).  With the sign of (3) (reading
    # R1(i); Maxwell's mu dH/dt = -dE/dz for the (2a) orientation) a unit E
    # impulse at node k changes H_{k+1/2} by +dt/(mu dz), H_{k-1/2} by -dt/(mu dz).
    nz, dz = 10, 1e-2
    K, De, Dm = yee.line_1d(nz, dz, EPS0, MU0)
    dt = 0.5 * dz / C0
    E = np.zeros(K.shape[0]); E[4] = 1.0          # node k = 5
    H = np.zeros(K.shape[1])
    E1, H1 = mf.step_leapfrog(E, H, dt / De, dt / Dm, K, K.T.tocsr())
    assert np.allclose(E1, E)
    ref = np.zeros(nz); ref[5] = dt / (MU0 * dz); ref[4] = -dt / (MU0 * dz)
    assert np.allclose(H1, ref, rtol=1e-14, atol=0)


def test_zero_in_zero_out_S171():
    s = yee.assemble(3, (4, 3, 3), (1e-3,) * 3, EPS0, MU0)
    E, H = np.zeros(s.Ne), np.zeros(s.Nh)
    E1, H1 = mf.step_leapfrog(E, H, 1.0 / s.De, 1.0 / s.Dm, s.K, s.K.T.tocsr())
    assert not E1.any() and not H1.any()
