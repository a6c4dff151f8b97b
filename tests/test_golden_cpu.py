"""The committed oracle goldens (tests/golden/config*.npz, tools/make_golden.py)
are what the full-length GPU parity tests compare against; these CPU checks pin
them to the oracle and to the problem description, so a stale or hand-edited
golden cannot pass:

* every required golden exists and every subset it carries is non-zero (no
  vacuous comparison downstream);
* its norms are consistent: ||state||^2 = sum of the subset norms^2, the
  reduced-state norms equal the stored vectors' norms;
* its problem fingerprint equals that of the problem rebuilt here (F13: the
  same fp64 description both sides consume);
* a prefix of its probe series is reproduced by re-running the oracle
  (config 2, 1500 steps).
"""
import json
import os
import sys

import numpy as np
import pytest

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "tools"))

REQUIRED = [(2, 32, 0), (3, 64, 0), (3, 32, 0), (5, 32, 0), (4, 32, 0), (4, 32, 15)]


def _load(c, p, m):
    path = os.path.join(GOLD, f"config{c}_fp{p}_m{m}.npz")
    z = np.load(path, allow_pickle=False)
    return {k: z[k] for k in z.files}


@pytest.mark.parametrize("c,p,m", REQUIRED, ids=[f"config{c}-fp{p}-m{m}" for c, p, m in REQUIRED])
def test_golden_present_and_nonvacuous(c, p, m):
    g = _load(c, p, m)
    meta = json.loads(str(g["meta"]))
    assert meta["config"] == c and meta["member"] == m and meta["precision"] == p
    assert g["probes"].shape[0] == meta["n_steps"]
    # every probe series, the interface rows and the reduced states carry data
    assert np.all(np.linalg.norm(g["probes"], axis=0) > 0), "a probe series is identically zero"
    assert np.linalg.norm(g["sample_val"]) > 0
    if c != 3:
        assert np.linalg.norm(g["if_E"]) > 0 and np.linalg.norm(g["red_e"]) > 0 and np.linalg.norm(g["red_h"]) > 0
    n = g["norms"]
    assert np.isclose(n[2], np.linalg.norm(g["if_E"]), rtol=1e-14)
    assert np.isclose(n[3], np.linalg.norm(g["red_e"]), rtol=1e-14)
    assert np.isclose(n[4], np.linalg.norm(g["red_h"]), rtol=1e-14)
    assert np.isclose(n[5] ** 2, np.sum(n[:5] ** 2), rtol=1e-12)
    # the sample is distinct, sorted unknown ids
    ids = g["sample_ids"]
    assert np.all(np.diff(ids) > 0) and len(ids) == min(100_000, len(ids))


@pytest.mark.parametrize("c,p", [(2, 32), (5, 32), (3, 64)])
def test_golden_fingerprint_matches_problem(c, p):
    from make_golden import apply_model, fingerprint, problem_for
    g = _load(c, p, 0)
    _, prob = problem_for(c, p)
    prob = apply_model(prob, g)
    assert np.allclose(fingerprint(prob), g["fingerprint"], rtol=1e-11, atol=0)


def test_config2_golden_prefix_reproduced_by_oracle():
    # 1500 steps: the pulse (source 306 cells from the box) has reached several
    # probes, the reduced block is still at zero -- the prefix pins the coarse
    # recursion and the probe bookkeeping of the golden
    from make_golden import problem_for
    from oracle import problem_step as ps
    from make_golden import apply_model
    g = _load(2, 32, 0)
    _, prob = problem_for(2, 32)
    prob = apply_model(prob, g)
    n = 1500
    _, _, probes, _ = ps.run(prob, n)
    assert np.linalg.norm(probes) > 0
    assert np.allclose(probes, g["probes"][:n], rtol=0, atol=1e-13 * np.abs(g["probes"][:n]).max())
