"""GPU parity on the BASELINE.json configurations, with problems emitted by the
preprocessing library (the product path) and the oracle stepping the same fp64
problem description (F13 shared-input rule)."""
import numpy as np
import pytest

from oracle import problem_step as ps
from synth import scenario

import parity
from parity import compare, run_gpu, run_oracle

pytestmark = pytest.mark.gpu


def _prep(which, precision=None, n_steps=None):
    from paper_1406_7042_b200 import prep
    scn = scenario(which, precision=precision, n_steps=n_steps)
    prob, info = prep.build_problem(scn, precision=precision)
    return scn, prob


def test_config1_full_run_fp64():
    # config 1: 2000 steps, fp64, q = 32 reduced block at 2x fine CFL: <= 1e-12
    scn, prob = _prep(1)
    gpu = run_gpu(prob, 2000, precision=64)
    ora = run_oracle(prob, 2000)
    es, ep, norm = compare(prob, gpu, ora)
    assert norm > 0 and es <= 1e-12 and ep <= 1e-12, (es, ep, parity.last_report)


@pytest.mark.parametrize("prec", [32, 64])
def test_tiny2d_recipe_B(prec):
    scn, prob = _prep("tiny2d_B", precision=prec)
    gpu = run_gpu(prob, 300, precision=prec)
    ora = run_oracle(prob, 300)
    es, ep, _ = compare(prob, gpu, ora)
    tol = 1e-12 if prec == 64 else 1e-4
    assert es <= tol and ep <= tol, (es, ep, parity.last_report)


def _random_state_run(which, n, seed, step0, graph_steps, members=(0,), window=None):
    """Full-size problem from a seeded random state on the active unknowns
    (coarse, interface rows, e~, h~ all non-zero), n steps on the GPU in the
    bench's launch configuration and in the oracle (ps.run from the same state
    and source step): per-subset parity."""
    from paper_1406_7042_b200.fdtd import Sim
    from sampled_state import oracle_vectors, random_state
    scn, prob = _prep(which, precision=32)
    prob = dict(prob, init={})
    arrays, red_e, red_h = random_state(prob, seed=seed, window=window)
    sim = Sim(prob, precision=32, graph_steps=graph_steps)
    comps = (0, 1, 2, 3, 4, 5) if prob["dim"] == 3 else (2, 3, 4)
    for c in comps:
        sim.set_state(c, arrays[c])
    sim.set_state(6, _gpu_red_order(red_e, prob))
    sim.set_state(7, _gpu_red_order(red_h, prob))
    sim.set_state(8, [float(step0)])
    sim.step(n)
    sim.sync()
    gpu = dict(state={c: sim.get_state(c) for c in comps}, red_e=sim.get_state(6), red_h=sim.get_state(7),
               probes=sim.probe())
    paths = sim.path()
    sim.close()
    rec = ps.build(prob)
    out = []
    for m in members:
        E0, H0 = oracle_vectors(rec, arrays, red_e, red_h, m)
        E, H, probes, _ = ps.run(prob, n, member=m, state=(E0, H0), start_step=step0, rec=rec)
        st, re_, rh_ = ps.to_storage(rec, E, H)
        ora = dict(state=st, red_e=re_, red_h=rh_, probes=probes, rec=rec, E=E, H=H)
        out.append(compare(prob, gpu, ora, member=m) + (dict(parity.last_report),))
    return out, paths


def test_config2_full_size_random_state_fp32():
    # full 1024^2 grid, q = 256, in the persistent kernel bench.py times, from
    # a seeded random state: the 40 reduced CTAs (LL y / G exchange at q = 256),
    # the interface tiles and the probes all carry data from step 0 (a zero
    # start leaves the reduced part at exactly 0 for ~865 steps)
    (res,), paths = _random_state_run(2, 200, seed=21, step0=40, graph_steps=32)
    es, ep, _, rep = res
    assert "persistent2d" in paths, paths
    assert es <= 1e-4 and ep <= 1e-4, rep


def test_config5_full_size_random_state_fp32():
    # full 400x200x40 grid, 64 regions in two 32-instance models (the N = 32,
    # 8-way K-split cluster GEMM), the bench's graphs of 32 steps, from a
    # seeded random state so every region and interface row carries data
    (res,), paths = _random_state_run(5, 40, seed=51, step0=10, graph_steps=32)
    es, ep, _, rep = res
    assert es <= 1e-4 and ep <= 1e-4, rep


@pytest.mark.parametrize("prec", [32, 64])
def test_config3_small_fp(prec):
    scn, prob = _prep("config3_small", precision=prec)
    gpu = run_gpu(prob, 200, precision=prec)
    ora = run_oracle(prob, 200)
    es, ep, _ = compare(prob, gpu, ora)
    tol = 1e-12 if prec == 64 else 1e-4
    assert es <= tol and ep <= tol, (es, ep, parity.last_report)


@pytest.mark.parametrize("prec", [32, 64])
def test_config3_full_size_sampled_one_step(prec):
    # 256^3: the oracle recomputes one step for 400 sampled unknowns from the
    # GPU state and compares with the GPU's next state, element by element
    from paper_1406_7042_b200.fdtd import Sim
    scn, prob = _prep(3, precision=prec)
    sim = Sim(prob, precision=prec)
    for c, a in prob["init"].items():
        sim.set_state(c, a)
    sim.step(7)
    st0 = {c: sim.get_state(c) for c in range(6)}
    sim.step(1)
    st1 = {c: sim.get_state(c) for c in range(6)}
    sim.close()
    rng = np.random.default_rng(0)
    nx, ny, nz = prob["n"]
    samples = [(int(rng.integers(0, 6)), (int(rng.integers(0, nx + 1)), int(rng.integers(0, ny + 1)),
                                          int(rng.integers(0, nz + 1)))) for _ in range(400)]
    ref = ps.sampled_step(prob, st0, samples)
    shp = (nz + 1, ny + 1, nx + 1)
    got = np.array([st1[c].reshape(shp)[idx[2], idx[1], idx[0]] for c, idx in samples])
    want = np.array([ref[(c, tuple(idx))] for c, idx in samples])
    scale = np.max(np.abs(want))
    tol = 1e-13 if prec == 64 else 2e-6
    assert scale > 0
    assert np.max(np.abs(got - want)) <= tol * scale


@pytest.mark.parametrize("kernel", ["gemv", "gemm"])
@pytest.mark.parametrize("prec", [64, 32])
def test_tiny5_shared_models_pec_plates(prec, kernel, monkeypatch):
    # config-5 structure: z-refined regions around stub tips, PEC plates through
    # the regions, two shared models with two instances each (N = 2 columns:
    # both fused kernels)
    monkeypatch.setenv("FDTD_FUSED", kernel)
    scn, prob = _prep("tiny5", precision=prec)
    assert [b["n_inst"] for b in prob["blocks"]] == [2, 2]
    gpu = run_gpu(prob, 300, precision=prec)
    ora = run_oracle(prob, 300)
    es, ep, _ = compare(prob, gpu, ora)
    tol = 1e-12 if prec == 64 else 1e-4
    assert es <= tol and ep <= tol, (es, ep, parity.last_report)


@pytest.mark.parametrize("form", ["fused", "fused-gemv", "leapfrog"])
@pytest.mark.parametrize("prec", [64, 32])
def test_tiny4_batched_iris_guide(prec, form, monkeypatch):
    # config-4 structure: x-graded refined slab with a PEC iris, B = 4
    # excitations of a TE10 sheet source, z = 0 Krylov basis (reading R5(viii));
    # "fused" takes the cluster-split GEMM kernel (N = 4), "fused-gemv" forces
    # the warp-per-row kernel
    if form == "fused-gemv":
        monkeypatch.setenv("FDTD_FUSED", "gemv")
        form = "fused"
    # from a seeded random state (every subset -- coarse, interface rows,
    # e~, h~ -- carries O(1) data from step 0; a zero start leaves the reduced
    # state in its first-arrival transient, where its own norm is tiny)
    # fp32 leap-frog (K~', S_E rounded to fp32 once) runs
    # the physical excitation: a random state puts O(1) energy into the modes
    # the enforcement clipped to the stability edge, where the phase is ~70x
    # more sensitive to the matrix rounding than anywhere in the excited band
    # (R14) -- the fused forms (compensated matrix) and fp64 take it
    from sampled_state import random_state
    scn, prob = _prep("tiny4", precision=prec)
    prob = dict(prob, init={})
    start = None
    n = 600
    if prec == 64 or form == "fused":
        arrays, red_e, red_h = random_state(prob, seed=41)
        start = dict(arrays=arrays, red_e=red_e, red_h=red_h, step=30)
        n = 300
    gpu = run_gpu(prob, n, precision=prec, reduced_form=form, start=start)
    tol = 1e-12 if prec == 64 else 1e-4
    for m in (0, 3):
        ora = run_oracle(prob, n, member=m, start=start)
        es, ep, _ = compare(prob, gpu, ora, member=m)
        assert es <= tol and ep <= tol, (m, es, ep, parity.last_report)


def test_tma_stencil_bitwise_equals_cp_async_stencil(monkeypatch):
    # the TMA and the cp.async 3-D stencils do the same arithmetic: from random
    # states they must agree bit for bit (regression: a cross-warp race on the
    # E-plane buffers of the TMA kernel showed up as whole wrong tile rows)
    from paper_1406_7042_b200.fdtd import Sim
    scn, prob = _prep("tiny5", precision=64)
    prob = dict(prob, init={})
    nx, ny, nz = prob["n"]
    S = (nx + 1) * (ny + 1) * (nz + 1)
    rng = np.random.default_rng(0)

    def run(no_tma, state):
        if no_tma:
            monkeypatch.setenv("FDTD_NO_TMA", "1")
        else:
            monkeypatch.delenv("FDTD_NO_TMA", raising=False)
        sim = Sim(prob, precision=64, graph_steps=0)
        for c in range(6):
            sim.set_state(c, state[c])
        sim.step(3)
        sim.sync()
        out = [sim.get_state(c) for c in range(6)]
        sim.close()
        return out

    for _ in range(12):
        state = [rng.standard_normal((1, S)) for _ in range(6)]
        a, b = run(True, state), run(False, state)
        for c in range(6):
            assert np.array_equal(a[c], b[c]), c


from parity import gpu_reduced_order as _gpu_red_order  # noqa: E402


def test_config4_full_size_sampled_one_step():
    # config 4 at full size (512 x 128 x 128, q = 1024 block with 65,024
    # interface rows, B = 16, leap-frog reduced path) in the launch
    # configuration bench.py times: one step from a seeded random state
    # (active unknowns of a window around the refined slab and the source
    # plane), against the unknown-by-unknown oracle (sampled_hybrid_step,
    # pinned in test_oracle_sampled.py) for two members
    from paper_1406_7042_b200.fdtd import Sim
    from sampled_state import random_state
    scn, prob = _prep(4, precision=32)
    prob = dict(prob, init={})
    nx, ny, nz = prob["n"]
    px = nx + 1
    win = lambda idx: ((idx % px >= 240) & (idx % px <= 272)) | ((idx % px >= 28) & (idx % px <= 36))
    arrays, red_e, red_h = random_state(prob, seed=4, window=win)
    step = 60
    sim = Sim(prob, precision=32, graph_steps=0)
    assert sim.B == 16
    for c in range(6):
        sim.set_state(c, arrays[c])
    sim.set_state(6, _gpu_red_order(red_e, prob))
    sim.set_state(7, _gpu_red_order(red_h, prob))
    sim.set_state(8, [float(step)])
    sim.step(1)
    sim.sync()
    got = {c: sim.get_state(c) for c in range(6)}
    ge, gh = sim.get_state(6), sim.get_state(7)
    sim.close()
    S = (nx + 1) * (ny + 1) * (nz + 1)
    rng = np.random.default_rng(2)
    samples = []
    for c in range(6):
        for _ in range(60):
            samples.append((c, (int(rng.integers(240, 273)), int(rng.integers(0, ny + 1)), int(rng.integers(0, nz + 1)))))
        for _ in range(20):
            samples.append((c, (int(rng.integers(28, 37)), int(rng.integers(0, ny + 1)), int(rng.integers(0, nz + 1)))))
    ifu = np.asarray(prob["interface"]["unknown"], np.int64)
    from parity import reduced_member, block_shapes
    for m in (0, 11):
        out, Eif, e1, h1 = ps.sampled_hybrid_step(prob, arrays, red_e[m], red_h[m], samples, member=m, step=step)
        scale = max(abs(v) for v in out.values())
        for (c, (i, j, k)), want in out.items():
            g = got[c][m][(k * (ny + 1) + j) * (nx + 1) + i]
            assert abs(g - want) <= 2e-5 * scale, (m, c, (i, j, k), g, want)
        gif = np.array([got[int(u // S)][m][int(u % S)] for u in ifu])
        assert np.abs(gif - Eif).max() <= 2e-5 * np.abs(Eif).max()
        sh = block_shapes(prob)
        gre = reduced_member(ge, sh, 16, m, "e")
        grh = reduced_member(gh, sh, 16, m, "h")
        assert np.abs(gre - e1).max() <= 2e-5 * np.abs(e1).max()
        assert np.abs(grh - h1).max() <= 2e-5 * np.abs(h1).max()


@pytest.mark.parametrize("which,prec,K", [("tiny2d_B", 32, None), ("tiny2d_B", 64, None), (1, 64, None),
                                          (2, 32, None), (2, 32, "4"), (2, 32, "2"),
                                          ("tiny2d_B", 32, "2"), ("tiny2d_B", 32, "0"), (1, 32, "4"), (1, 32, "2")])
def test_persistent_2d_bitwise_equals_per_step_kernels(which, prec, K, monkeypatch):
    # the persistent on-chip-resident 2-D kernel (one cooperative launch per
    # step() call) against the per-step stencil + fused-reduced kernels: same
    # arithmetic, so states, reduced states and probe series agree bit for bit,
    # across several launches (ragged chunks)
    # (from a seeded random state: every tile, interface row and reduced row
    # carries data, config 2's q = 256 block included)
    from sampled_state import random_state
    scn, prob = _prep(which, precision=prec)
    prob = dict(prob, init={})
    arrays, red_e, red_h = random_state(prob, seed=17)
    start = dict(arrays=arrays, red_e=red_e, red_h=red_h, step=5)
    n = 150
    chunks = [37, 1, 64, 48]
    # K: the temporal-blocking halo depth of the fp32 persistent kernel
    # (persist2d_tb_tile; None = the default (0, the per-step exchange);
    # tiny2d_B: 2 x 1 tiles of 64, config 1: one tile, config 2: 16 x 16)
    if K is not None:
        monkeypatch.setenv("FDTD_P2K", K)
    monkeypatch.setenv("FDTD_PERSIST", "0")
    a = run_gpu(prob, n, precision=prec, chunks=chunks, start=start)
    monkeypatch.delenv("FDTD_PERSIST")
    b = run_gpu(prob, n, precision=prec, chunks=chunks, start=start)
    assert b["launches"] == len(chunks), "persistent path not taken"
    assert np.linalg.norm(a["red_e"]) > 0 and np.linalg.norm(a["red_h"]) > 0
    for c in a["state"]:
        assert np.array_equal(a["state"][c], b["state"][c]), c
    assert np.array_equal(a["red_e"], b["red_e"]) and np.array_equal(a["red_h"], b["red_h"])
    assert np.array_equal(a["probes"], b["probes"])


@pytest.mark.parametrize("prec", [32, 64])
def test_batched_vec_stencil_bitwise_equals_scalar_tma(prec, monkeypatch):
    # B = 4: the batched TMA stencil (16 bytes of members per thread) against
    # the scalar TMA stencil, from random states incl. the interface rows:
    # per-member arithmetic in the same order -> bit for bit
    from paper_1406_7042_b200.fdtd import Sim
    scn, prob = _prep("tiny4", precision=prec)
    prob = dict(prob, init={})
    nx, ny, nz = prob["n"]
    S = (nx + 1) * (ny + 1) * (nz + 1)
    rng = np.random.default_rng(1)

    def run(no_vec, state):
        if no_vec:
            monkeypatch.setenv("FDTD_NO_VEC", "1")
        else:
            monkeypatch.delenv("FDTD_NO_VEC", raising=False)
        sim = Sim(prob, precision=prec, graph_steps=0)
        for c in range(6):
            sim.set_state(c, state[c])
        sim.step(5)
        sim.sync()
        out = [sim.get_state(c) for c in range(7)]
        sim.close()
        return out

    from sampled_state import random_state
    arrays, _, _ = random_state(prob, seed=3)
    state = [arrays[c] for c in range(6)]
    a, b = run(True, state), run(False, state)
    for c in range(7):
        assert np.array_equal(a[c], b[c]), c


@pytest.mark.parametrize("skinny", ["force", "off"])
def test_tiny4_batch8_leapfrog_skinny_gemm(skinny, monkeypatch):
    # the fp32 tall-skinny GEMM kernels of the leap-frog path (config 4's
    # S_E products, N in {8, 16, 32}) on the small iris guide with B = 8
    # members (waveforms duplicated with distinct amplitudes), against the
    # oracle for two members; "off" runs the GEMV kernels on the same problem
    scn, prob = _prep("tiny4", precision=32)
    w = np.asarray(prob["sources"]["wave"])
    prob = dict(prob, sources=dict(prob["sources"], wave=np.concatenate([w, -0.7 * w], axis=2)), batch=8)
    if skinny == "force":
        monkeypatch.setenv("FDTD_FORCE_SKINNY", "1")
    else:
        monkeypatch.setenv("FDTD_NO_SKINNY", "1")
    # (the physical excitation, 600 steps: see test_tiny4_batched_iris_guide)
    gpu = run_gpu(prob, 600, precision=32, reduced_form="leapfrog")
    for m in (1, 6):
        ora = run_oracle(prob, 600, member=m)
        es, ep, _ = compare(prob, gpu, ora, member=m)
        assert es <= 1e-4 and ep <= 1e-4, (m, es, ep, parity.last_report)


@pytest.mark.parametrize("case,prec,tile,grid", [
    ("config3_small", 32, "2,4", 0), ("config3_small", 32, "2,6", 7), ("config3_small", 32, "4,3", 0),
    ("config3_small", 64, "2,3", 5), ("config3_small", 64, "1,6", 0),
    ("tiny5", 32, "2,6", 0), ("tiny5", 32, "2,4", 13), ("tiny5", 64, "2,3", 0), ("tiny5", 32, "4,3", 3),
    ("tiny4_b16", 32, "4,3", 0), ("tiny4_b16", 32, "4,3", 11), ("tiny4_b16", 64, "2,3", 0),
    ("config3_small", 32, "2,4,16", 0), ("config3_small", 64, "1,4,16", 0), ("tiny5", 32, "2,4,16", 0),
    ("tiny4_b16", 32, "4,3,16", 0),
])
def test_tile_stencil_bitwise_equals_tma_stencil(case, prec, tile, grid, monkeypatch):
    # the tile stencil (stencil3d.cuh: persistent CTAs on balanced ranges of
    # column-planes, W elements per thread, NS-stage ring across segment
    # boundaries, mask multipliers, z-wall fix-ups) against the reference TMA
    # stencils (stencil3d_tma_kernel / stencil3d_tma_vec_kernel), from random
    # states on the unknowns incl. interface / source rows: bit for bit, 7
    # steps; small grids make ranges start and end mid-column
    from paper_1406_7042_b200.fdtd import Sim
    from sampled_state import random_state
    if case == "tiny4_b16":
        scn, prob = _prep("tiny4", precision=prec)
        w = np.asarray(prob["sources"]["wave"])
        amp = np.linspace(1.0, -1.3, 16)
        prob = dict(prob, sources=dict(prob["sources"], wave=w[:, :, :1] * amp[None, None, :]), batch=16)
    else:
        scn, prob = _prep(case, precision=prec)
    prob = dict(prob, init={})
    if "mat_coef" in prob:
        arrays, _, _ = random_state(prob, seed=5)
    else:
        # uniform problem: random values everywhere (fdtd_set_state stores the
        # E entries that are not unknowns as 0; H keeps them, both kernels alike)
        nx, ny, nz = prob["n"]
        S = (nx + 1) * (ny + 1) * (nz + 1)
        rng = np.random.default_rng(5)
        arrays = {c: rng.uniform(-1, 1, (int(prob.get("batch", 1)), S)) for c in range(6)}
    monkeypatch.setenv("FDTD_KCHUNK", "9")

    def run(old):
        if old:
            monkeypatch.setenv("FDTD_STENCIL_OLD", "1")
            monkeypatch.delenv("FDTD_TILE", raising=False)
        else:
            monkeypatch.delenv("FDTD_STENCIL_OLD", raising=False)
            monkeypatch.setenv("FDTD_TILE", tile)
            if grid:
                monkeypatch.setenv("FDTD_TILE_GRID", str(grid))
        sim = Sim(prob, precision=prec, graph_steps=0)
        paths = sim.path()
        for c in range(6):
            sim.set_state(c, arrays[c])
        sim.step(7)
        sim.sync()
        out = [sim.get_state(c) for c in range(8)]
        sim.close()
        return out, paths

    (a, pa), (b, pb) = run(True), run(False)
    assert "tile3d" in pb and "tile3d" not in pa, (pa, pb)
    for c in range(8):
        assert np.array_equal(a[c], b[c]), c


@pytest.mark.parametrize("tc", ["on", "off"])
def test_tiny4_batch16_leapfrog_tensor_core_gemm(tc, monkeypatch):
    # y = S_E h~ on the tensor cores (tcgen05 kind::tf32, 3xTF32; N = 16
    # members) against the oracle for two members over 300 steps, and "off"
    # (SIMT GEMM) as the control
    scn, prob = _prep("tiny4", precision=32)
    w = np.asarray(prob["sources"]["wave"])
    amp = np.linspace(1.0, -1.3, 16)
    prob = dict(prob, sources=dict(prob["sources"], wave=w[:, :, :1] * amp[None, None, :]), batch=16)
    monkeypatch.setenv("FDTD_FORCE_SKINNY", "1")
    if tc == "off":
        monkeypatch.setenv("FDTD_NO_TC", "1")
    from paper_1406_7042_b200.fdtd import Sim
    sim = Sim(prob, precision=32, reduced_form="leapfrog")
    assert ("tc_gemm" in sim.path()) == (tc == "on"), sim.path()
    sim.close()
    # (the physical excitation, 600 steps: see test_tiny4_batched_iris_guide)
    gpu = run_gpu(prob, 600, precision=32, reduced_form="leapfrog")
    for m in (0, 13):
        ora = run_oracle(prob, 600, member=m)
        es, ep, _ = compare(prob, gpu, ora, member=m)
        assert es <= 1e-4 and ep <= 1e-4, (m, es, ep, parity.last_report)


@pytest.mark.parametrize("case,prec", [("tiny5", 32), ("tiny5", 64)])
def test_rows_prepass_bitwise_equals_in_kernel_rows(case, prec, monkeypatch):
    # explicit rows evaluated ahead of the tile stencil (rows_prepass_kernel: the
    # row's E^{n+1} stored into the new parity and read back by the stencil
    # thread that owns the unknown) against the reference stencils that walk
    # each row inside the kernel (eval_row): states and probe series bit for bit
    # (batch 16 with interface rows: test_tile_stencil_bitwise...[tiny4_b16-*])
    from paper_1406_7042_b200.fdtd import Sim
    from sampled_state import random_state
    scn, prob = _prep(case, precision=prec)
    prob = dict(prob, init={})
    arrays, re_, rh_ = random_state(prob, seed=11)

    def run(tile):
        if tile:
            monkeypatch.delenv("FDTD_STENCIL_OLD", raising=False)
        else:
            monkeypatch.setenv("FDTD_STENCIL_OLD", "1")
        sim = Sim(prob, precision=prec, graph_steps=0)
        paths = sim.path()
        for c in range(6):
            sim.set_state(c, arrays[c])
        sim.step(9)
        sim.sync()
        out = [sim.get_state(c) for c in range(8)]
        pr = sim.probe()
        sim.close()
        return out, pr, paths

    (a, pa, ta), (b, pb, tb) = run(True), run(False)
    assert "tile3d" in ta and "tile3d" not in tb, (ta, tb)
    for c in range(8):
        assert np.array_equal(a[c], b[c]), c
    assert np.array_equal(pa, pb)


@pytest.mark.parametrize("case,prec", [("tiny5", 32), ("config3_small", 64), ("tiny4", 32)])
def test_device_set_state_equals_host_set_state(case, prec, monkeypatch):
    # fdtd_set_state's device scatter (fp64 copy + one kernel) against the host
    # scatter loop: identical device arrays (E off the unknowns stored as 0)
    from paper_1406_7042_b200.fdtd import Sim
    scn, prob = _prep(case, precision=prec)
    prob = dict(prob, init={})
    nx, ny, nz = prob["n"]
    S = (nx + 1) * (ny + 1) * (nz + 1)
    rng = np.random.default_rng(7)
    arrays = {c: rng.uniform(-1, 1, (int(prob.get("batch", 1)), S)) for c in range(6)}

    def run(host):
        if host:
            monkeypatch.setenv("FDTD_HOST_SET_STATE", "1")
        else:
            monkeypatch.delenv("FDTD_HOST_SET_STATE", raising=False)
        sim = Sim(prob, precision=prec, graph_steps=0)
        for c in range(6):
            sim.set_state(c, arrays[c])
        out = [sim.get_state(c) for c in range(6)]
        sim.step(3)
        sim.sync()
        out += [sim.get_state(c) for c in range(6)]
        sim.close()
        return out

    a, b = run(True), run(False)
    for c in range(12):
        assert np.array_equal(a[c], b[c]), c


@pytest.mark.parametrize("case,prec,graph", [("tiny5", 32, 0), ("tiny5", 32, 8), ("tiny5", 64, 8), ("tiny5", 64, 0)])
def test_rows_fused_into_reduced_gemm_bitwise_equals_prepass(case, prec, graph, monkeypatch):
    # the explicit rows of the next step evaluated by the reduced GEMM thread that
    # finalises their y (no pre-pass launch in steady state)
    # against the pre-pass launch every step: states, reduced states and probe
    # series bit for bit -- eager and in CUDA graphs, across a set_state in the
    # middle of the run (which invalidates the rows evaluated ahead), an odd number
    # of steps (parity of the two G buffers) and a profiled step
    from paper_1406_7042_b200.fdtd import Sim
    from sampled_state import random_state
    scn, prob = _prep(case, precision=prec)
    prob = dict(prob, init={})
    arrays, re_, rh_ = random_state(prob, seed=13)
    arrays2, _, _ = random_state(prob, seed=14)
    monkeypatch.setenv("FDTD_FUSED", "gemm")        # tiny5's few instances would take the GEMV kernel

    def run(fused):
        if fused:
            monkeypatch.delenv("FDTD_NO_ROWFUSE", raising=False)
        else:
            monkeypatch.setenv("FDTD_NO_ROWFUSE", "1")
        sim = Sim(prob, precision=prec, graph_steps=graph)
        assert ("fused_rows" in sim.path()) == fused, sim.path()
        for c in range(6):
            sim.set_state(c, arrays[c])
        sim.set_state(6, parity.gpu_reduced_order(re_, prob))
        sim.set_state(7, parity.gpu_reduced_order(rh_, prob))
        sim.step(19)
        mid = [sim.get_state(c) for c in range(8)]
        sim.set_state(3, arrays2[3])            # new Hx: the rows evaluated ahead are stale
        sim.step(1)
        sim.step(26)
        sim.set_state(7, parity.gpu_reduced_order(0.5 * rh_, prob))
        sim.step(17)
        sim.sync()
        out = [sim.get_state(c) for c in range(8)]
        pr = sim.probe()
        n = sim.launch_count()
        sim.close()
        return mid, out, pr, n

    (ma, a, pa, na), (mb, b, pb, nb) = run(True), run(False)
    assert na < nb
    for c in range(8):
        assert np.array_equal(ma[c], mb[c]), ("mid", c)
        assert np.array_equal(a[c], b[c]), c
    assert np.array_equal(pa, pb) and pa.shape[0] == 63
