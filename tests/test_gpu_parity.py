"""GPU parity: the CUDA path (through the C ABI) against the oracle on the same
seeded inputs.  Every input and expected value here comes from oracle/ and
synth/ alone (problem descriptions built by tests/oracle_problem.py).

Tolerances (north star): fp64 relative L2 <= 1e-12 on the final state; fp32
relative L2 <= 1e-4 on the state and on every probe series."""
import math

import numpy as np
import pytest

from oracle import hybrid as hy
from oracle import reduction as rd
from oracle import stability as st
from synth import scenario

from oracle_problem import problem_from_oracle, uniform_problem
import parity
from parity import compare, run_gpu, run_oracle

pytestmark = pytest.mark.gpu

TOL = {64: 1e-12, 32: 1e-4}


def _check(problem, n, prec, **kw):
    gpu = run_gpu(problem, n, precision=prec, **kw)
    ora = run_oracle(problem, n)
    es, ep, norm = compare(problem, gpu, ora)
    assert norm > 0
    assert es <= TOL[prec], f"state rel L2 {es:.3e}"
    assert ep <= TOL[prec] * (1 if prec == 64 else 1), f"probe rel L2 {ep:.3e}"
    assert gpu["launches"] > 0
    return es, ep


@pytest.mark.parametrize("prec", [64, 32])
def test_uniform_3d_random_field(prec):
    scn = scenario("tiny3d", precision=prec, n_steps=100)
    _check(uniform_problem(scn), 100, prec)


def test_dielectric_3d_table_mode():
    scn = scenario("tiny3d", precision=64, n_steps=60)
    rng = np.random.default_rng(5)
    nx, ny, nz = scn["n"]
    eps = np.ones((nz, ny, nx))
    eps[3:9, 4:15, 10:30] = 2.7
    eps[:, :, 31:] = 1.6
    scn["eps_r"] = eps
    _check(uniform_problem(scn), 60, 64)


def _fine_cfl(scn):
    r = scn["boxes"][0]["r"][0]
    return scn["delta"] / r / (scn["c0"] * math.sqrt(scn["dim"]))


@pytest.mark.parametrize("prec", [64, 32])
def test_hybrid_2d_identity_basis(prec):
    # identity V_f: the unreduced coarse+fine hybrid through the reduced-block
    # kernels, below its stability limit
    scn = scenario("tiny2d", n_steps=300)
    dt = 0.9 * _fine_cfl(scn)
    prob, hs, pr = problem_from_oracle(scn, dt=dt)
    _check(prob, 300, prec)


def _enforced_problem(scn, q=24, seed=11):
    boxes = [hy.Box(tuple(b["lo"]), tuple(b["hi"]), tuple(b["r"])) for b in scn["boxes"]]
    hs = hy.assemble(2, scn["n"], scn["delta"], scn["eps_r"], boxes, scn["eps0"], scn["mu0"])
    b = hy.blocks(hs)
    rng = np.random.default_rng(seed)
    V1 = rd.d_orthonormal(rng.standard_normal((len(b["ef"]), q)), hs.De[b["ef"]])
    V2 = rd.d_orthonormal(rng.standard_normal((len(b["hf"]), q)), hs.Dm[b["hf"]])
    pr = hy.project(hs, V1, V2)
    dt = scn["dt"]
    dtc = scn["delta"] / (scn["c0"] * math.sqrt(2))
    alpha = st.split_alpha(dt, dtc)
    SEif = np.asarray(pr["S_E"])[pr["if_rows"]]
    Kp, SEp, rep = st.enforce_hybrid_block(np.ones(q), pr["Kt_rr"], SEif, np.ones(q),
                                           pr["De_c"][pr["if_rows"]], alpha, dt)
    prob, _, _ = problem_from_oracle(scn, V1, V2, Kt=Kp, SEif=SEp)
    return prob


@pytest.mark.parametrize("form", ["fused", "leapfrog"])
@pytest.mark.parametrize("prec", [64, 32])
def test_hybrid_2d_reduced_enforced(prec, form):
    # q = 24 reduced block above the fine CFL limit (dt = 1.5x fine CFL) after
    # the split enforcement (reading R7)
    scn = scenario("tiny2d", n_steps=400)
    prob = _enforced_problem(scn)
    prob["blocks"][0]["g_e"] = float(scn["dt"])       # D~ = I: scalar G
    prob["blocks"][0]["g_h"] = float(scn["dt"])
    _check(prob, 400, prec, reduced_form=form)


def test_graphs_match_eager_bitwise():
    scn = scenario("tiny2d", n_steps=200)
    prob = _enforced_problem(scn)
    a = run_gpu(prob, 200, precision=32, graph_steps=0)
    b = run_gpu(prob, 200, precision=32, graph_steps=32, chunks=[37, 64, 99])
    for c in a["state"]:
        assert np.array_equal(a["state"][c], b["state"][c])
    assert np.array_equal(a["red_h"], b["red_h"])
    assert np.array_equal(a["probes"], b["probes"])


@pytest.mark.parametrize("form", ["fused", "leapfrog"])
def test_reduced_probes_and_state_roundtrip(form):
    # probes on e~ / h~ (Eq. (10) reconstruction rows) and set_state of the
    # reduced state mid-run
    scn = scenario("tiny2d", n_steps=120)
    prob = _enforced_problem(scn)
    q = prob["blocks"][0]["qe"]
    rng = np.random.default_rng(3)
    prob["probes"] = prob["probes"] + [
        dict(kind=1, block=0, inst=0, vrow=rng.standard_normal(q)),
        dict(kind=2, block=0, inst=0, vrow=rng.standard_normal(q))]
    _check(prob, 120, 64, reduced_form=form)
    from paper_1406_7042_b200.fdtd import Sim
    from parity import run_oracle
    ora = run_oracle(prob, 60)
    sim = Sim(prob, precision=64, reduced_form=form)
    sim.step(60)
    e6, h7 = sim.get_state(6), sim.get_state(7)
    st = {c: sim.get_state(c) for c in (2, 3, 4)}
    sim.close()
    sim2 = Sim(prob, precision=64, reduced_form=form)
    for c, a in st.items():
        sim2.set_state(c, a)
    sim2.set_state(6, e6)
    sim2.set_state(7, h7)
    sim2.set_state(8, [60.0])
    sim2.step(60)
    a = sim2.get_state(7)
    sim2.close()
    ref = run_oracle(prob, 120)
    assert np.linalg.norm(a - ref["red_h"]) <= 1e-11 * np.linalg.norm(ref["red_h"])


def test_batch_members_independent():
    # B = 3 independent excitations: member m must equal the single run with
    # member m's waveform (exactly, in fp64 up to the oracle tolerance)
    scn = scenario("tiny2d", n_steps=150)
    prob = _enforced_problem(scn)
    w = np.asarray(prob["sources"]["wave"])[:, :, :1]
    prob["sources"]["wave"] = np.concatenate([w, -0.5 * w, 2.0 * w], axis=2)
    prob["batch"] = 3
    gpu = run_gpu(prob, 150, precision=64)
    for m in range(3):
        ora = run_oracle(prob, 150, member=m)
        es, ep, _ = compare(prob, gpu, ora, member=m)
        assert es <= 1e-12 and ep <= 1e-12


def test_divergence_detected():
    from paper_1406_7042_b200.fdtd import DivergenceError
    scn = scenario("tiny3d", precision=64, n_steps=10)
    prob = uniform_problem(scn, dt=1.3 * scn["dt"] / 0.99)     # above the exact limit
    with pytest.raises(DivergenceError):
        run_gpu(prob, 3000, precision=64)


@pytest.mark.parametrize("B", [3, 4])
def test_uniform_3d_batched_members(B):
    # batch innermost in device storage; B = 4 uses the TMA stencil, B = 3 the
    # cp.async one (unaligned rows); every member against its own oracle run
    scn = scenario("tiny3d", precision=64, n_steps=40)
    prob = uniform_problem(scn)
    init = {c: np.concatenate([np.asarray(a) * (1.0 + 0.3 * m) * (-1) ** m for m in range(B)], axis=0)
            for c, a in prob["init"].items()}
    prob["init"] = init
    prob["batch"] = B
    gpu = run_gpu(prob, 40, precision=64)
    for m in range(B):
        ora = run_oracle(prob, 40, member=m)
        es, ep, _ = compare(prob, gpu, ora, member=m)
        assert es <= 1e-12 and ep <= 1e-12, (m, es, ep)
