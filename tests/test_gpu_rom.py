"""GPU parity of the whole-domain reduced model (rom_* calls of libfdtd,
csrc/rom.cu: K~' resident in registers as fp64 tensor-core fragments, cluster
DSMEM exchange) against oracle/rom.py through the C ABI.  fp64: every subset
(e~, h~, each probe series) within 1e-12 relative L2 of the oracle."""
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

pytestmark = pytest.mark.gpu

from parity import rel_l2  # noqa: E402


def _check(tag, gpu_e, gpu_h, gpu_p, e, h, pr, tol=1e-12):
    rep = {"e": rel_l2(gpu_e.T, e, "e~"), "h": rel_l2(gpu_h.T, h, "h~")}
    for p in range(pr.shape[1]):
        rep[f"probe{p}"] = rel_l2(gpu_p[:, p, :], pr[:, p, :], f"probe{p}")
    assert max(rep.values()) <= tol, (tag, rep)
    return rep


def _random_model(q_e, q_h, n_in, n_oe, n_oh, dt, seed):
    rng = np.random.default_rng(seed)
    K = rng.standard_normal((q_e, q_h))
    K *= 1.95 / dt / np.linalg.svd(K, compute_uv=False)[0]
    return dict(K=K, dt=dt, g_e=dt, g_h=dt, B_e=rng.standard_normal((q_e, n_in)),
                L_e=rng.standard_normal((n_oe, q_e)) if n_oe else None,
                L_h=rng.standard_normal((n_oh, q_h)) if n_oh else None)


@pytest.mark.parametrize("cols", [0, 8, 16, 32])
def test_rom2d_small_matches_oracle(cols):
    from oracle import rom as orom
    from paper_1406_7042_b200.prep import rom as prom
    from paper_1406_7042_b200.rom import Rom
    from synth import scenario
    scn = scenario("rom2d_small")
    model, _ = prom.build_rom(scn)
    n = scn["n_steps"]
    sim = Rom(model, model["amp"], model["wave"], cols_per_cluster=cols)
    sim.step(137)                      # ragged chunks: one persistent launch each
    sim.step(n - 137)
    pr_g = sim.probe()
    e, h, pr = orom.run(model, model["amp"], model["wave"], n)
    _check(("rom2d_small", cols, sim.info()), sim.get_state(0), sim.get_state(1), pr_g, e, h, pr)
    assert sim.get_state(2)[0] == n
    sim.close()


@pytest.mark.parametrize("q_e,q_h,batch,cols", [(80, 80, 20, 8), (96, 70, 9, 16), (160, 160, 20, 8), (150, 131, 37, 16),
                                                  (250, 256, 12, 8), (33, 47, 70, 32)])
def test_random_models_all_cluster_sizes(q_e, q_h, batch, cols):
    # rectangular K~, E and H probes, random start, forced: every cluster size
    # (1, 2, 4, 8 CTAs) and padded q
    from oracle import rom as orom
    from paper_1406_7042_b200.rom import Rom
    dt = 0.37
    model = _random_model(q_e, q_h, 3, 5, 11, dt, seed=q_e + batch)
    rng = np.random.default_rng(7)
    amp = rng.standard_normal((3, batch))
    wave = rng.standard_normal((150, batch))
    e0, h0 = rng.standard_normal((q_e, batch)), rng.standard_normal((q_h, batch))
    sim = Rom(model, amp, wave, cols_per_cluster=cols)
    sim.set_state(0, e0.T)
    sim.set_state(1, h0.T)
    assert np.array_equal(sim.get_state(0), e0.T) and np.array_equal(sim.get_state(1), h0.T)
    sim.step(200)                      # 50 steps beyond the waveform record (u = 0 there)
    pr_g = sim.probe()
    e, h, pr = orom.run(model, amp, wave, 200, state=(e0, h0))
    _check((q_e, q_h, batch, cols, sim.info()), sim.get_state(0), sim.get_state(1), pr_g, e, h, pr)
    sim.close()


def test_rom2d_paper_cavity_full_run():
    # the NEXT-3 workload: Table I's 2-D cavity, order 80, s = 4.95, 64 excitation
    # waveforms, the physical time of the paper's 10,000 steps (2,000 steps here)
    from oracle import rom as orom
    from paper_1406_7042_b200.prep import rom as prom
    from paper_1406_7042_b200.rom import Rom
    from synth import scenario
    scn = scenario("rom2d")
    model, info = prom.build_rom(scn)
    n = scn["n_steps"]
    sim = Rom(model, model["amp"], model["wave"])
    sim.step(n)
    pr_g = sim.probe()
    e, h, pr = orom.run(model, model["amp"], model["wave"], n)
    rep = _check(("rom2d", sim.info()), sim.get_state(0), sim.get_state(1), pr_g, e, h, pr)
    print("rom2d parity", rep, sim.info())
    sim.close()


def test_restart_equals_straight_run():
    # get_state / set_state / step counter: a restored checkpoint continues bit for bit
    from paper_1406_7042_b200.rom import Rom
    dt = 0.2
    model = _random_model(40, 40, 2, 2, 0, dt, seed=5)
    rng = np.random.default_rng(2)
    amp, wave = rng.standard_normal((2, 13)), rng.standard_normal((300, 13))
    a = Rom(model, amp, wave)
    a.step(300)
    pa = a.probe()
    b = Rom(model, amp, wave)
    b.step(120)
    pb1 = b.probe()
    e, h, k = b.get_state(0), b.get_state(1), b.get_state(2)
    c = Rom(model, amp, wave)
    c.set_state(0, e); c.set_state(1, h); c.set_state(2, k)
    c.step(180)
    pc = c.probe()
    assert np.array_equal(np.concatenate([pb1, pc]), pa)
    assert np.array_equal(a.get_state(0), c.get_state(0)) and np.array_equal(a.get_state(1), c.get_state(1))
    for s in (a, b, c):
        s.close()
