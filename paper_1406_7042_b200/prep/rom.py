"""Whole-domain reduced model (the paper's own mode, P:158-211 and §III-A):
scenario -> model description consumed by rom_create (include/fdtd_rom.h) and,
bit for bit, by the oracle (oracle/rom.py) -- the F13 shared-input rule.

  1. FIT assembly of the whole grid (Eq. (3)) in the library's scaled
     units, B_E = -1 at each source unknown;
  2. multi-point block Arnoldi at the points of Eq. (19) (reading
     R5(i) for the shifted-operator sign), V = blockdiag(V1, V2) (Eq. (9));
  3. D-orthonormalisation (R5(vi)) so that D~_eps = D~_mu = I;
  4. projection K~ = V1^T K V2, B~_e = V1^T B_E (Eqs. (15)-(16));
  5. stability enforcement: sigma' = min(sigma, gamma 2/dt);
  6. probe rows L_e = rows of V1 (Eq. (10)).
"""
from __future__ import annotations

import hashlib
import os
import pickle
import time

import numpy as np

from . import fit, reduce
from . import CACHE_DIR, hybrid_system

ROM_VERSION = 1


def enforce_full(Kt, dt, gamma=reduce.GAMMA):
    """§III-A with D~ = I: clip the singular values of K~ at gamma 2/dt."""
    U, s, Wt = np.linalg.svd(Kt, full_matrices=False)
    lim = gamma * 2.0 / dt
    return (U * np.minimum(s, lim)) @ Wt, dict(sigma_max=float(s[0]), limit=float(lim), clipped=int(np.sum(s > lim)))


def build_rom(scn, cache=True):
    """scenario (synth.rom_cavity2d) -> (model dict, info dict).  model: K [q][q],
    g_e, g_h (scalars = dt), B_e [q][n_in], L_e [n_probe][q], dt, amp, wave."""
    h = hashlib.sha256(repr((ROM_VERSION, scn["name"], scn["dim"], tuple(scn["n"]), scn["delta"], scn["dt"], scn["q"],
                             sorted(scn["basis"].items()), np.asarray(scn["sources"]["idx"]).tolist(),
                             [p["terms"] for p in scn["probes"]])).encode())
    h.update(np.asarray(scn["eps_r"]).tobytes())
    path = os.path.join(CACHE_DIR, f"{scn['name']}-rom-{h.hexdigest()[:16]}.pkl")
    if cache and os.path.exists(path):
        with open(path, "rb") as f:
            model, info = pickle.load(f)
    else:
        t0 = time.time()
        dim, n, d, dt = scn["dim"], tuple(scn["n"]), scn["delta"], scn["dt"]
        P = fit.assemble(dim, n, d, scn["eps_r"], [], scn["eps0"], scn["mu0"], need_K=True)
        full = hybrid_system(P)
        De, Dm, K = full["De"], full["Dm"], full["K"].tocsr()
        Ne, Nh = K.shape
        S = P.S
        shp = fit.sshape(P.n, dim)

        def uid(comp, ijk):
            i, j, k = ijk
            return int(comp) * S + int(np.ravel_multi_index((k, j, i), shp))
        src = [uid(c, ijk) for c, ijk in zip(scn["sources"]["comp"], scn["sources"]["idx"])]
        rows = full["epos"][np.asarray(src)]
        if np.any(rows < 0):
            raise ValueError("a source is not an E unknown")
        B = np.zeros((Ne + Nh, len(src)))
        B[rows, np.arange(len(src))] = -1.0
        bas = scn["basis"]
        pts = reduce.expansion_points(bas["M"], bas["L"], bas["fmax"], dt)
        q = int(scn["q"])
        V1, V2 = reduce.krylov_basis(De, Dm, K, dt, B, np.arange(Ne), np.arange(Nh), q, pts)
        V1 = reduce.d_orthonormalise(V1, De)
        V2 = reduce.d_orthonormalise(V2, Dm)
        Kt = V1.T @ (K @ V2)
        Kp, einfo = enforce_full(Kt, dt)
        L_e = []
        for p in scn["probes"]:
            row = np.zeros(q)
            for comp, ijk, wgt in p["terms"]:
                r = full["epos"][uid(comp, ijk)]
                if r < 0:
                    raise ValueError("a probe term is not an E unknown")
                row += wgt * V1[r]
            L_e.append(row)
        model = dict(q_e=q, q_h=q, K=Kp, g_e=float(dt), g_h=float(dt), B_e=V1.T @ B[:Ne],
                     L_e=np.asarray(L_e).reshape(len(L_e), q), L_h=None, dt=float(dt))
        info = dict(Ne=int(Ne), Nh=int(Nh), t_prep=time.time() - t0, **einfo)
        if cache:
            os.makedirs(CACHE_DIR, exist_ok=True)
            with open(path + ".tmp", "wb") as f:
                pickle.dump((model, info), f, protocol=4)
            os.replace(path + ".tmp", path)
    model = dict(model, amp=np.asarray(scn["amp"], np.float64), wave=np.asarray(scn["wave"], np.float64),
                 n_steps=int(scn["n_steps"]))
    return model, info
