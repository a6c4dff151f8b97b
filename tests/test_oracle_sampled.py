"""Pin of oracle.problem_step.sampled_hybrid_step (the full-size config-4
parity oracle) against the matrix-form recursion ``run`` (O8) on the small
config-4 / config-5 shaped problems: every interface row, both reduced
states, and coarse samples (near the refined regions, at sources, random)
must agree to rounding, for several members and steps with live sources."""
import numpy as np
import pytest

from oracle import problem_step as ps
from synth import scenario

from sampled_state import oracle_vectors, random_state


def _prep(which):
    from paper_1406_7042_b200 import prep
    scn = scenario(which, precision=64)
    prob, _ = prep.build_problem(scn, precision=64)
    return prob


@pytest.mark.parametrize("which,member,step", [("tiny4", 0, 3), ("tiny4", 3, 10), ("tiny5", 0, 5)])
def test_sampled_hybrid_step_matches_recursion(which, member, step):
    prob = _prep(which)
    prob["init"] = {}
    rec = ps.build(prob)
    arrays, red_e, red_h = random_state(prob, seed=7)
    E, H = oracle_vectors(rec, arrays, red_e, red_h, member)
    E1, H1, _, _ = ps.run(prob, 1, member=member, state=(E, H), start_step=step, rec=rec)
    rng = np.random.default_rng(1)
    S = rec.S
    # samples: all interface unknowns' H partners region + sources + random
    ids = list(rec.e_ids[rng.choice(len(rec.e_ids), 300, replace=False)]) + \
        list(rec.h_ids[rng.choice(len(rec.h_ids), 300, replace=False)]) + \
        [int(u) for u in np.asarray(prob["sources"]["unknown"])[:20]]
    dim = prob["dim"]
    nx, ny, nz = prob["n"]
    samples = []
    for u in ids:
        c, p = int(u // S), int(u % S)
        i, j, k = p % (nx + 1), (p // (nx + 1)) % (ny + 1), p // ((nx + 1) * (ny + 1))
        samples.append((c, (i, j, k)))
    out, Eif, e1, h1 = ps.sampled_hybrid_step(prob, arrays, red_e[member], red_h[member], samples,
                                              member=member, step=step)
    epos = {int(u): q for q, u in enumerate(rec.e_ids)}
    hpos = {int(u): q for q, u in enumerate(rec.h_ids)}
    scale = max(np.abs(E1).max(), np.abs(H1).max())
    for (c, idx), u in zip(samples, ids):
        want = E1[epos[int(u)]] if int(u) in epos else H1[hpos[int(u)]]
        assert abs(out[(c, idx)] - want) <= 1e-12 * scale, (c, idx)
    ifu = np.asarray(prob["interface"]["unknown"], np.int64)
    want_if = np.array([E1[epos[int(u)]] for u in ifu])
    assert np.abs(Eif - want_if).max() <= 1e-12 * scale
    ne, nh = len(rec.e_ids), len(rec.h_ids)
    assert np.abs(e1 - E1[ne:]).max() <= 1e-12 * np.abs(E1[ne:]).max()
    assert np.abs(h1 - H1[nh:]).max() <= 1e-12 * np.abs(H1[nh:]).max()
