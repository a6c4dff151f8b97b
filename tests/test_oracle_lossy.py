"""Pins of the lossy recursion (conductivity terms of Eq. (2a)/
(2b) P:64-74, D_sigma in F of Eq. (5), stability condition (7)
P:141-147) as oracle.problem_step advances it from the problem's shared
coefficients (ca, cb; da, ch):

* the definition: Eq. (4) assembled by oracle.yee (per-cell eps_r, sigma_e,
  sigma_m; its own owning-cell rule) and solved literally (matrix_form.
  step_literal) gives the same trajectory, source included;
* closed form: with uniform matched loss sigma_e/eps = sigma_m/mu = 2 alpha every
  oscillating mode of the one-step map has |lambda| = (1 - alpha dt)/(1 + alpha dt)
  exactly (the 2 x 2 mode map has determinant ca^2), brute force on the dense map;
* invariant: x^T R x never increases when F + F^T >= 0 (condition (7));
* the graded absorber: the 4th-order 5-cell profile is matched (sigma_m =
  sigma_e mu/eps) and a pulse sent into it comes back >= 40 dB down.
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle import matrix_form as mf, problem_step as ps, yee  # noqa: E402
from synth import scenario  # noqa: E402
from synth.scenarios import EPS0, MU0, absorber_profile, lossy_box  # noqa: E402


def _problem(scn):
    from paper_1406_7042_b200 import prep
    prob, _ = prep.build_problem(scn, cache=False)
    return prob


def _yee(scn):
    dim = scn["dim"]
    d = (scn["delta"],) * 3
    return yee.assemble(dim, scn["n"], d, scn["eps0"], scn["mu0"], eps_r=scn["eps_r"], sig_e=scn["sigma_e"],
                        sig_m=scn["sigma_m"])


def _to_yee_vector(s, rec, E, H, dim, n):
    st, _, _ = ps.to_storage(rec, E, H)
    shp = yee.storage_shape(dim, n)
    comps = range(6) if dim == 3 else (2, 3, 4)
    return s.from_storage({c: st.get(c, np.zeros(rec.S)).reshape(shp) for c in comps})


def test_lossy_problem_step_equals_literal_eq4():
    for scn in (lossy_box("l3", 311, 3, 16, 9, 7, 1e-3, 0.9, 60, 64, axes=(0, 2)),
                lossy_box("l2", 312, 2, 24, 17, 1, 1e-3, 0.9, 80, 64, axes=(0, 1))):
        prob = _problem(scn)
        assert prob.get("mat_ca") is not None and np.asarray(prob["mat_ca"]).min() < 0.9
        n = scn["n_steps"]
        E, H, pr, rec = ps.run(prob, n)
        s = _yee(scn)
        R, F = mf.build_RF(s.De, s.Dm, s.K, s.Dse, s.Dsm, scn["dt"])
        # B u: J at the source unknown with the sign of S:139
        i, j, k = scn["sources"]["idx"][0]
        shp = yee.storage_shape(scn["dim"], scn["n"])
        row = s.index[2][(k, j, i) if scn["dim"] == 3 else (j, i)]
        x = np.zeros(s.Ne + s.Nh)
        for q in range(n):
            Bu = np.zeros_like(x)
            Bu[row] = -scn["sources"]["wave"][q, 0, 0]
            x = mf.step_literal(x, R, F, Bu)
        got = _to_yee_vector(s, rec, E, H, scn["dim"], scn["n"])
        assert np.linalg.norm(x) > 0
        assert np.linalg.norm(got - x) <= 1e-12 * np.linalg.norm(x)


def test_uniform_matched_loss_every_mode_decays_by_ca():
    # sigma_e / eps = sigma_m / mu = 2 alpha everywhere: det of each 2 x 2 mode map = ca^2
    nx, ny = 9, 7
    dt_scn = lossy_box("u2", 313, 2, nx, ny, 1, 1e-3, 0.9, 4, 64, axes=())
    alpha = 0.13 / dt_scn["dt"]
    dt_scn["eps_r"] = np.ones((ny, nx))
    dt_scn["sigma_e"] = np.full((ny, nx), 2 * alpha * EPS0)
    dt_scn["sigma_m"] = np.full((ny, nx), 2 * alpha * MU0)
    prob = _problem(dt_scn)
    prob["sources"] = None
    rec = ps.build(prob)
    NE, NH = rec.KE.shape
    M = np.zeros((NE + NH, NE + NH))
    for q in range(NE + NH):
        x = np.zeros(NE + NH); x[q] = 1.0
        E, H, _, _ = ps.run(prob, 1, state=(x[:NE].copy(), x[NE:].copy()), rec=rec)
        M[:, q] = np.concatenate([E, H])
    lam = np.linalg.eigvals(M)
    ca = (1 - alpha * dt_scn["dt"]) / (1 + alpha * dt_scn["dt"])
    osc = np.abs(lam.imag) > 1e-9
    assert osc.sum() >= NE and np.allclose(np.abs(lam[osc]), ca, rtol=1e-10, atol=0)
    assert np.all(np.abs(lam) <= 1 + 1e-12)


def test_energy_never_increases_condition_7():
    scn = lossy_box("l3e", 314, 3, 14, 8, 6, 1e-3, 0.95, 10, 64, axes=(0, 1))
    prob = _problem(scn)
    prob["sources"] = None
    rec = ps.build(prob)
    s = _yee(scn)
    R, _ = mf.build_RF(s.De, s.Dm, s.K, s.Dse, s.Dsm, scn["dt"])
    rng = np.random.default_rng(0)
    NE, NH = rec.KE.shape
    E, H = rng.standard_normal(NE), rng.standard_normal(NH)
    prev = None
    for _ in range(60):
        x = _to_yee_vector(s, rec, E, H, 3, scn["n"])
        en = mf.energy(x, R)
        assert prev is None or en <= prev * (1 + 1e-13)
        first = en if prev is None else first
        prev = en
        E, H, _, _ = ps.run(prob, 5, state=(E, H), rec=rec)
    assert en < first * 0.5          # and the absorbers do take energy out


def test_graded_absorber_is_matched_and_absorbs():
    se, sm = absorber_profile(40, 40e-3, 1e-3, EPS0, MU0)
    assert np.allclose(sm * EPS0, se * MU0) and se[5:35].max() == 0 and se[0] > se[4] > 0
    assert np.allclose(se[:5] / se[0], ((4.5 - np.arange(5)) / 4.5) ** 4)         # 4th order
    # a 100 x 100-cell box with the layer on all four sides against the same box
    # with its PEC walls alone: after the pulse (-20 dB at 10 GHz, 30 cells per
    # wavelength) has crossed the box a few times the probe sees > 50 dB less
    from synth.scenarios import _gauss_deriv, _times, gaussian_derivative_tau

    def run(absorb, n=100, steps=900):
        scn = lossy_box("g2", 315, 2, n, n, 1, 1e-3, 0.95, steps, 64, axes=())
        scn["eps_r"] = np.ones((n, n))
        se_, sm_ = absorber_profile(n, n * 1e-3, 1e-3, EPS0, MU0)
        f = 1.0 if absorb else 0.0
        scn["sigma_e"] = f * (se_[None, :] + se_[:, None])
        scn["sigma_m"] = f * (sm_[None, :] + sm_[:, None])
        scn["sources"]["wave"] = _gauss_deriv(_times(scn["dt"], steps), gaussian_derivative_tau(10e9)).reshape(steps, 1, 1)
        scn["sources"]["idx"] = np.array([[50, 50, 0]])
        scn["probes"] = [dict(terms=[(2, (30, 40, 0), 1.0)])]
        _, _, pr, _ = ps.run(_problem(scn), steps)
        return pr[:, 0]
    with_abs, with_wall = run(True), run(False)
    late = slice(600, 900)
    assert np.max(np.abs(with_wall[late])) >= 0.3 * np.max(np.abs(with_wall))
    assert np.max(np.abs(with_abs[late])) <= 3e-3 * np.max(np.abs(with_abs))
