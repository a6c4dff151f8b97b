"""Race evidence by perturbation (compute-sanitizer is closed on this GPU
pool): every kernel family runs once as is and again with
FDTD_JITTER, which makes every warp sleep a pseudo-random 0..jitter ns at its
phase points (the persistent kernel's E / H phases and reduced steps, every
plane of the TMA tile stencil), reshuffling the inter-CTA exchange order (the
fp32 LL words, the fp64 flags, the y / G chain of PAPER.md:109-112's
recursion) and the intra-CTA TMA ring / barrier interleaving.  A missing
fence, a write-after-read on a halo buffer or a stage refilled too early
changes the result; the results must stay bitwise identical, run after run."""
import numpy as np
import pytest

from synth import scenario

from parity import run_gpu

pytestmark = pytest.mark.gpu


def _prep(which, precision):
    from paper_1406_7042_b200 import prep
    scn = scenario(which, precision=precision)
    prob, _ = prep.build_problem(scn, precision=precision)
    return prob


def _batch16(prob):
    w = np.asarray(prob["sources"]["wave"])
    amp = np.linspace(1.0, -1.3, 16)
    return dict(prob, sources=dict(prob["sources"], wave=w[:, :, :1] * amp[None, None, :]), batch=16)


def _same(a, b):
    for c in a["state"]:
        assert np.array_equal(a["state"][c], b["state"][c]), c
    if len(a["red_e"]):
        assert np.array_equal(a["red_e"], b["red_e"]) and np.array_equal(a["red_h"], b["red_h"])
    assert np.array_equal(a["probes"], b["probes"])


CASES = [
    # (scenario, precision, env, steps, random start, extra kwargs)
    ("tiny2d_B", 32, {}, 120, True, {}),                      # persistent, fp32 LL exchange
    ("tiny2d_B", 64, {}, 80, True, {}),                       # persistent, fp64 flags + counters
    (2, 32, {}, 60, True, {}),                                # config 2: 256 tiles + 40 reduced CTAs
    ("tiny2d_B", 32, {"FDTD_P2K": "2"}, 90, True, {}),        # temporal blocking: bands, y / G rings
    ("config3_small", 32, {}, 12, False, {}),                 # TMA tile stencil, batch 1
    ("tiny5", 64, {}, 12, True, {}),                          # tile stencil + local rows + cluster GEMM
    ("tiny4_b16", 32, {"FDTD_FORCE_SKINNY": "1"}, 12, True, {"reduced_form": "leapfrog"}),  # batched + tcgen05
]


@pytest.mark.parametrize("case,prec,env,n,rnd,kw", CASES,
                         ids=[f"{c[0]}-fp{c[1]}" + ("-" + "-".join(c[2].values()) if c[2] else "") for c in CASES])
def test_jitter_bitwise_identical(case, prec, env, n, rnd, kw, monkeypatch):
    from sampled_state import random_state
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    prob = _batch16(_prep("tiny4", prec)) if case == "tiny4_b16" else _prep(case, prec)
    start = None
    if rnd:
        prob = dict(prob, init={})
        arrays, red_e, red_h = random_state(prob, seed=99)
        start = dict(arrays=arrays, red_e=red_e, red_h=red_h, step=3)
    chunks = [n // 3, 1, n - n // 3 - 1]
    monkeypatch.delenv("FDTD_JITTER", raising=False)
    ref = run_gpu(prob, n, precision=prec, chunks=chunks, start=start, **kw)
    again = run_gpu(prob, n, precision=prec, chunks=chunks, start=start, **kw)
    _same(ref, again)
    for jit in ("700", "3000"):
        monkeypatch.setenv("FDTD_JITTER", jit)
        shaken = run_gpu(prob, n, precision=prec, chunks=chunks, start=start, **kw)
        _same(ref, shaken)
