"""Pins of oracle/rom.py (the whole-domain reduced model, Eq. (12))
against what the paper and the mathematics fix -- none of them re-types the
oracle's own forward substitution:

* closed form: with D~ = I and K~ = diag(sigma) every mode is a rotation by
  theta = 2 arcsin(dt sigma / 2) per step (survey F4):
  e_n = cos((n - 1/2) theta) / cos(theta / 2) from e_0 = 1, h_0 = 0;
* invariant: x~^T R~ x~ is conserved by the lossless recursion (F3);
* special case: the identity basis reproduces the full FDTD recursion (4)
  (oracle.matrix_form.step_literal, the dense solve of the definition);
* the paper's numbers: the reduced model of the 2-D PEC cavity (Table I,
  P:403-421: 101 cells of 1 cm, order 80, 5 points, M = 1.1, f_max = 0.5 GHz)
  shows the analytic TM resonances within 1 % at s = 0.99 and s = 4.95 (P:401,
  P:440), N = 30,200, and stays bounded over a late-time run (E7);
* the enforcement law of the model the preprocessing emits: sigma_max(K~') =
  gamma 2/dt when clipped, checked with the oracle's own SVD.
"""
import math
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle import matrix_form as mf, physics, rom as orom, yee  # noqa: E402
from synth import scenario  # noqa: E402
from synth.scenarios import C0, EPS0, MU0  # noqa: E402


def test_single_modes_rotate_by_closed_form_angle_F4():
    dt = 0.7
    sig = np.array([0.3, 1.1, 1.7, 1.98]) / dt                  # dt sigma / 2 < 1
    model = dict(K=np.diag(sig), dt=dt, B_e=np.zeros((4, 1)), L_e=np.eye(4))
    e0 = np.ones((4, 1))
    n = 400
    _, _, pr = orom.run(model, np.zeros((1, 1)), np.zeros((1, 1)), n, state=(e0, np.zeros((4, 1))))
    theta = 2.0 * np.arcsin(dt * sig / 2.0)
    steps = np.arange(1, n + 1)[:, None]
    ref = np.cos((steps - 0.5) * theta[None, :]) / np.cos(theta / 2.0)[None, :]
    assert np.allclose(pr[:, :, 0], ref, rtol=0, atol=1e-10 * np.abs(ref).max())


def test_energy_invariant_and_forced_linearity_F3():
    rng = np.random.default_rng(3)
    q, B = 12, 5
    dt = 0.4
    K = rng.standard_normal((q, q))
    K *= 1.9 / dt / np.linalg.svd(K, compute_uv=False)[0]
    model = dict(K=K, dt=dt, B_e=rng.standard_normal((q, 2)), L_e=rng.standard_normal((3, q)),
                 L_h=rng.standard_normal((2, q)))
    e0, h0 = rng.standard_normal((q, B)), rng.standard_normal((q, B))
    e, h, _ = orom.run(model, np.zeros((2, B)), np.zeros((1, B)), 1000, state=(e0, h0))
    en0, en1 = orom.energy(model, e0, h0), orom.energy(model, e, h)
    assert np.all(np.abs(en1 - en0) <= 1e-10 * np.abs(en0))
    # the response is linear in the excitation and the batch columns are independent
    amp = rng.standard_normal((2, B))
    wave = rng.standard_normal((50, B))
    _, _, p_all = orom.run(model, amp, wave, 80)
    for b in (0, 3):
        _, _, p_b = orom.run(model, amp[:, b:b + 1], wave[:, b:b + 1], 80)
        assert np.allclose(p_all[:, :, b], p_b[:, :, 0], rtol=0, atol=1e-12 * np.abs(p_all).max())
    _, _, p2 = orom.run(model, 2.0 * amp, wave, 80)
    assert np.allclose(p2, 2.0 * p_all, rtol=1e-12, atol=0)


def test_identity_basis_is_the_full_fdtd_recursion():
    # V = I: K~ = K, D~ = D (dense) -- Eq. (12) must be Eq. (4)
    n, d = (7, 5, 1), (1e-3, 1.3e-3, 1.0)
    ys = yee.assemble(2, n, d, EPS0, MU0)
    K = ys.K.toarray()
    dt = 0.9 * 1.0 / (C0 * math.sqrt(1 / d[0] ** 2 + 1 / d[1] ** 2))
    Ne, Nh = K.shape
    rng = np.random.default_rng(0)
    Be = np.zeros((Ne, 1)); Be[5, 0] = -1.0
    model = dict(K=K, De=ys.De, Dm=ys.Dm, dt=dt, B_e=Be, L_e=np.eye(Ne)[[2, 9]])
    wave = rng.standard_normal((30, 1))
    e, h, pr = orom.run(model, np.ones((1, 1)), wave, 30)
    R, F = mf.build_RF(ys.De, ys.Dm, ys.K, np.zeros(Ne), np.zeros(Nh), dt)
    x = np.zeros(Ne + Nh)
    for s in range(30):
        Bu = np.zeros(Ne + Nh); Bu[5] = -wave[s, 0]
        x = mf.step_literal(x, R, F, Bu)
        assert abs(pr[s, 0, 0] - x[2]) <= 1e-12 * max(1.0, np.abs(x).max())
    assert np.allclose(np.concatenate([e[:, 0], h[:, 0]]), x, rtol=0, atol=1e-12 * np.abs(x).max())


@pytest.fixture(scope="module")
def cavity_models():
    from paper_1406_7042_b200.prep import rom as prom
    out = {}
    for s in (0.99, 4.95):
        scn = scenario("rom2d", s_factor=s, batch=1)
        out[s] = (scn, *prom.build_rom(scn))
    return out


@pytest.mark.parametrize("s", [0.99, 4.95])
def test_paper_2d_cavity_resonances_within_one_percent(cavity_models, s):
    scn, model, info = cavity_models[s]
    assert info["Ne"] + info["Nh"] == 30200                      # Table I
    n_steps = scn["n_steps"]
    _, _, pr = orom.run(model, model["amp"], model["wave"], n_steps)
    L = 101 * 0.01
    ana = physics.cavity_modes((L, L), C0, count=12, dim=2)
    ana = ana[ana < 0.5e9]         # TM11, TM12/21, TM22, TM13/31 (6 modes, 4 distinct) inside the pulse band
    found = set()
    for p in range(pr.shape[1]):
        f, mag = physics.spectrum(pr[:, p, 0], scn["dt"], pad_factor=8, window="hann")
        pk = physics.find_peaks(f, mag, prominence=0.01, fmin=0.15e9, fmax=0.5e9)
        for fa in ana:
            if len(pk) and np.min(np.abs(pk - fa)) <= 0.01 * fa:
                found.add(float(fa))
    # every analytic TM mode below f_max = 0.5 GHz is seen by some probe within 1 %
    assert len(ana) == 4 and found == set(float(v) for v in ana), (sorted(found), ana)


def test_enforced_model_obeys_sigma_law_and_stays_bounded(cavity_models):
    scn, model, info = cavity_models[4.95]
    dt = model["dt"]
    sv = np.linalg.svd(np.asarray(model["K"]), compute_uv=False)
    assert info["clipped"] > 0 and info["sigma_max"] * dt / 2 > 1.0      # unstable before
    assert abs(sv[0] * dt / 2 - 0.9999) <= 1e-9                          # gamma = 0.9999
    # E7: late-time run stays bounded; lossless -> energy conserved
    rng = np.random.default_rng(1)
    q = sv.size
    e0, h0 = rng.standard_normal((q, 2)), rng.standard_normal((q, 2))
    e, h, _ = orom.run(dict(model, L_e=None), np.zeros((1, 2)), np.zeros((1, 2)), 100000, state=(e0, h0))
    en0, en1 = orom.energy(model, e0, h0), orom.energy(model, e, h)
    assert np.all(np.abs(en1 - en0) <= 1e-8 * np.abs(en0))
