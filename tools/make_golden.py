#!/usr/bin/env python
"""Full-length oracle goldens for the BASELINE.json configurations.

Writes ``tests/golden/config{C}{tag}_m{member}.npz`` from the CPU oracle ONLY
(``oracle.problem_step.run``, the literal recursion (4)/(12) of PAPER.md:109-112
and :182-185 in the leap-frog order of :211).  The problem description both
sides consume (R8, the F13 shared-input rule) comes from the host
preprocessing library; nothing here touches the CUDA path.

Contents of a golden (all fp64 unless noted):
  probes      [n_steps][n_probe]   the full probe series of one batch member
  if_E        [n_if]               final E at every interface row (interface order)
  red_e/red_h [q_total]            final reduced states ([block][inst][q] order)
  sample_ids  int64 [n_sample]     seeded uniform sample of active coarse
                                   unknowns (flat id comp*S + storage index),
                                   interface rows excluded (they are in if_E)
  sample_val  [n_sample]           their final values
  norms       [6]                  ||coarse E (regular)||, ||coarse H||, ||E_if||,
                                   ||e~||, ||h~||, ||whole state||
  fingerprint [8]                  float checksums of the problem description
                                   (tests assert the rebuilt problem matches)
  meta        json string          config, member, steps, precision, timings

    python tools/make_golden.py --config 2 [--member 0] [--prec 32] [--chunk 500]

Long runs checkpoint every --chunk steps under cache/golden_ckpt (resumable).
"""
from __future__ import annotations

import argparse
import hashlib
import json
import os
import resource
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle import problem_step as ps  # noqa: E402
from synth import scenario  # noqa: E402

N_SAMPLE = 100_000


def fingerprint(prob):
    """Order-sensitive float checksums of everything the recursion reads."""
    f = []
    mid = prob.get("mat_id")
    if mid is not None:
        w = np.arange(1, np.asarray(mid).size + 1, dtype=np.float64) % 9973
        f.append(float(np.dot(np.asarray(mid, np.float64).ravel(), w)))
        f.append(float(np.sum(np.asarray(prob["mat_coef"], np.float64) * np.arange(1, np.asarray(prob["mat_coef"]).size + 1).reshape(np.asarray(prob["mat_coef"]).shape))))
    else:
        f += [float(np.sum(prob["uniform_coef"])), 0.0]
    kk, se = 0.0, 0.0
    for b in prob.get("blocks") or []:
        K = np.asarray(b["K"], np.float64).ravel()
        kk += float(np.dot(K, np.cos(np.arange(K.size) * 0.001)))
        S = np.asarray(b["S_E"], np.float64).ravel()
        se += float(np.dot(S, np.cos(np.arange(S.size) * 0.001)))
    f += [kk, se]
    itf = prob.get("interface")
    if itf is not None:
        f.append(float(np.dot(np.asarray(itf["val"], np.float64), np.cos(np.arange(len(itf["val"])) * 0.01))))
        f.append(float(np.sum(np.asarray(itf["c"], np.float64))))
    else:
        f += [0.0, 0.0]
    src = prob.get("sources")
    f.append(float(np.sum(np.asarray(src["wave"], np.float64) ** 2)) if src is not None else 0.0)
    init = prob.get("init") or {}
    f.append(float(sum(np.sum(np.asarray(a, np.float64) * np.cos(np.arange(np.asarray(a).size) * 0.01)
                                .reshape(np.asarray(a).shape)) for a in init.values())))
    return np.array(f)


MODEL_EMBED_MAX = 4_000_000     # entries; config 4's S_E (6.7e7) stays in the prep cache


def model_arrays(prob):
    """The reduced models (K~', S_E per block) when small enough to commit: a
    projection basis is not unique across LAPACK builds (signs / rotations
    within the Krylov space), so a golden's reduced states are tied to the exact
    matrices it was stepped with; the GPU test steps those (apply_model)."""
    blocks = prob.get("blocks") or []
    tot = sum(np.asarray(b["K"]).size + np.asarray(b["S_E"]).size for b in blocks)
    if not blocks or tot > MODEL_EMBED_MAX:
        return {}
    out = {}
    for i, b in enumerate(blocks):
        out[f"blk{i}_K"] = np.asarray(b["K"], np.float64)
        out[f"blk{i}_SE"] = np.asarray(b["S_E"], np.float64)
    return out


def apply_model(prob, golden):
    """Replace the problem's reduced matrices by the golden's (same shapes)."""
    blocks = prob.get("blocks") or []
    if not blocks or "blk0_K" not in golden:
        return prob
    nb = []
    for i, b in enumerate(blocks):
        K, SE = golden[f"blk{i}_K"], golden[f"blk{i}_SE"]
        assert K.shape == np.asarray(b["K"]).shape and SE.shape == np.asarray(b["S_E"]).shape
        nb.append(dict(b, K=K, S_E=SE))
    return dict(prob, blocks=nb)


def embed(path, prob):
    """Add the model arrays to an existing golden written from ``prob`` (its
    fingerprint must be the problem's)."""
    z = np.load(path, allow_pickle=False)
    d = {k: z[k] for k in z.files}
    assert np.allclose(fingerprint(prob), d["fingerprint"], rtol=1e-13, atol=0), "golden is not of this problem"
    d.update(model_arrays(prob))
    np.savez_compressed(path, **d)


def problem_for(config, prec):
    from paper_1406_7042_b200 import prep
    scn = scenario(config, precision=prec)
    prob, _ = prep.build_problem(scn, precision=prec)
    return scn, prob


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, required=True)
    ap.add_argument("--member", type=int, default=0)
    ap.add_argument("--prec", type=int, default=None)
    ap.add_argument("--steps", type=int, default=None, help="default: the config's full length")
    ap.add_argument("--chunk", type=int, default=500)
    ap.add_argument("--tag", default="")
    ap.add_argument("--embed", action="store_true", help="only add the reduced-model arrays to the existing golden")
    a = ap.parse_args()
    if a.embed:
        scn, prob = problem_for(a.config, a.prec)
        embed(os.path.join(ROOT, "tests", "golden", f"config{a.config}{a.tag}_fp{int(prob['precision'])}_m{a.member}.npz"), prob)
        return
    t0 = time.time()
    scn, prob = problem_for(a.config, a.prec)
    prec = int(prob["precision"])
    n_steps = int(a.steps or scn["n_steps"])
    t_prep = time.time() - t0
    rec = ps.build(prob)
    t_build = time.time() - t0 - t_prep
    print(f"config {a.config} m{a.member} fp{prec}: prep {t_prep:.1f} s, oracle build {t_build:.1f} s, "
          f"NE {rec.KE.shape[0]} NH {rec.KH.shape[0]}, nnz {rec.KE.nnz + rec.KH.nnz}", flush=True)
    fp = fingerprint(prob)
    tag = f"config{a.config}{a.tag}_fp{prec}_m{a.member}"
    ck_dir = os.path.join(ROOT, "cache", "golden_ckpt")
    os.makedirs(ck_dir, exist_ok=True)
    ck = os.path.join(ck_dir, tag + ".npz")
    s0, state, probes = 0, None, np.zeros((n_steps, len(rec.probe_rows)))
    if os.path.exists(ck):
        z = np.load(ck)
        if np.array_equal(z["fingerprint"], fp) and int(z["n_steps"]) == n_steps:
            s0 = int(z["step"])
            state = (z["E"].copy(), z["H"].copy())
            probes[:s0] = z["probes"][:s0]
            print(f"resuming at step {s0}", flush=True)
    t_run = time.time()
    while s0 < n_steps:
        n = min(a.chunk, n_steps - s0)
        E, H, pr, _ = ps.run(prob, n, member=a.member, state=state, start_step=s0, rec=rec)
        probes[s0:s0 + n] = pr
        s0 += n
        state = (E, H)
        tmp = ck + ".tmp.npz"
        np.savez(tmp, E=E, H=H, probes=probes[:s0], step=s0, n_steps=n_steps, fingerprint=fp)
        os.replace(tmp, ck)
        el = time.time() - t_run
        print(f"  step {s0}/{n_steps}  {el:.0f} s  |E| {np.linalg.norm(E):.4e}", flush=True)
    E, H = state if state is not None else ps.initial_state(rec, prob, a.member)
    Ne_c, Nh_c = len(rec.e_ids), len(rec.h_ids)
    n_if = 0 if prob.get("interface") is None else len(prob["interface"]["unknown"])
    n_reg = Ne_c - n_if
    # interface rows sit at the end of the coarse E block (ps.build order);
    # re-order them as the problem lists them (ps.build keeps that order)
    if_E = E[n_reg:Ne_c].copy()
    red_e, red_h = E[Ne_c:].copy(), H[Nh_c:].copy()
    rng = np.random.default_rng(70420 + a.config)
    pool_ids = np.concatenate([rec.e_ids[:n_reg], rec.h_ids])
    pool_val = np.concatenate([E[:n_reg], H[:Nh_c]])
    k = min(N_SAMPLE, len(pool_ids))
    pick = np.sort(rng.choice(len(pool_ids), size=k, replace=False))
    norms = np.array([np.linalg.norm(E[:n_reg]), np.linalg.norm(H[:Nh_c]), np.linalg.norm(if_E),
                      np.linalg.norm(red_e), np.linalg.norm(red_h),
                      np.sqrt(np.sum(E ** 2) + np.sum(H ** 2))])
    meta = dict(config=a.config, member=a.member, n_steps=n_steps, precision=prec,
                t_prep_s=round(t_prep, 1), t_build_s=round(t_build, 1),
                t_run_s=round(time.time() - t_run, 1),
                peak_rss_gb=round(resource.getrusage(resource.RUSAGE_SELF).ru_maxrss / 2**20, 2),
                host=os.uname().nodename, cpu_count=os.cpu_count(),
                script="tools/make_golden.py (calls oracle.problem_step.run only)",
                sha256_probes=hashlib.sha256(probes.tobytes()).hexdigest()[:16])
    out_dir = os.path.join(ROOT, "tests", "golden")
    os.makedirs(out_dir, exist_ok=True)
    out = os.path.join(out_dir, tag + ".npz")
    np.savez_compressed(out, probes=probes, if_E=if_E, red_e=red_e, red_h=red_h,
                        sample_ids=pool_ids[pick].astype(np.int64), sample_val=pool_val[pick],
                        norms=norms, fingerprint=fp, meta=np.array(json.dumps(meta)), **model_arrays(prob))
    print(f"wrote {out}: {json.dumps(meta)}  norms {norms}", flush=True)


if __name__ == "__main__":
    main()
