"""Scenario generators for BASELINE.json configs 1-5 and small test variants.

A scenario is a plain dict (all geometry in coarse cell units):

  name, config_id, dim (2|3), n=(nx, ny, nz) coarse cells (nz=1 in 2-D),
  delta [m], eps0, mu0, c0, eps_r (per cell, [nz][ny][nx] or [ny][nx]),
  boxes: [dict(lo, hi, r, q, model, pec_fine)]  refined regions
  pec_sheets: [dict(axis, plane, lo, hi)]        zero-thickness PEC plates
  dt [s], n_steps, precision (32|64), batch B,
  sources: dict(comp [ns], idx [ns, 3], wave [n_steps][ns][B])  J^{n+1/2}
  probes: [dict(terms=[(comp, (i, j, k), weight), ...])]
  init: None | {comp: array [B][storage]}
  basis: dict(recipe, L, M, fmax, p, seed)

Storage index convention (i, j, k) for each component: DESIGN.md §5.
Physical constants: c0 exact, mu0 = 4 pi 1e-7, eps0 = 1/(mu0 c0^2)
(a consistent set; SPEC S:70 lists CODATA eps0 with the classical mu0, which
would make the grid's wave speed differ from c0 in the 10th digit).
"""
from __future__ import annotations

import math

import numpy as np

C0 = 299792458.0
MU0 = 4.0e-7 * math.pi
EPS0 = 1.0 / (MU0 * C0 * C0)

SEED0 = 14067042


def config_ids():
    return (1, 2, 3, 4, 5)


# ---------------------------------------------------------------------------
# waveforms (input samples, fp64)
# ---------------------------------------------------------------------------

def gaussian_tau(f20db):
    """Gaussian g = exp(-(t-t0)^2/(2 tau^2)): |G(f)| = exp(-(2 pi f tau)^2/2)
    is 20 dB below DC at f20db (S:71 convention)."""
    return math.sqrt(2.0 * math.log(10.0)) / (2.0 * math.pi * f20db)


def gaussian_derivative_tau(f20db):
    """Gaussian derivative: |G(f)| ~ x exp(-x^2/2), x = 2 pi f tau, peaks at x=1;
    tau such that f20db is 20 dB below the peak (x > 1 root of
    x exp(-(x^2-1)/2) = 0.1), found by bisection."""
    lo, hi = 1.0, 10.0
    g = lambda x: x * math.exp(-(x * x - 1.0) / 2.0) - 0.1
    for _ in range(200):
        mid = 0.5 * (lo + hi)
        if g(mid) > 0:
            lo = mid
        else:
            hi = mid
    x = 0.5 * (lo + hi)
    return x / (2.0 * math.pi * f20db)


def _times(dt, n_steps):
    # u^{n+1} = J^{n+1/2}: step n (0-based) injects J at (n + 1/2) dt
    return (np.arange(n_steps, dtype=np.float64) + 0.5) * dt


def _gauss(t, tau):
    t0 = 4.0 * tau
    return np.exp(-((t - t0) ** 2) / (2.0 * tau * tau))


def _gauss_deriv(t, tau):
    t0 = 4.0 * tau
    return -(t - t0) / tau * np.exp(-((t - t0) ** 2) / (2.0 * tau * tau))


def _mod_gauss(t, fc, tau):
    t0 = 4.0 * tau
    return np.sin(2.0 * math.pi * fc * (t - t0)) * np.exp(-((t - t0) ** 2) / (2.0 * tau * tau))


def cfl_coarse(dim, delta, c=C0):
    """The scenario's time-step reference: Eq. (1) for the uniform coarse cell in
    vacuum (the fastest medium present)."""
    return delta / (c * math.sqrt(dim))


# ---------------------------------------------------------------------------
# 2-D hybrid cavity family (configs 1, 2 and test variants)
# ---------------------------------------------------------------------------

def _pick_nodes(rng, nx, ny, boxes, count, margin=2, exclude=()):
    """Seeded interior Ez nodes at Chebyshev distance >= margin from every box."""
    out = []
    taken = set(exclude)
    while len(out) < count:
        i = int(rng.integers(1, nx))
        j = int(rng.integers(1, ny))
        ok = True
        for b in boxes:
            if (b["lo"][0] - margin < i < b["hi"][0] + margin) and \
               (b["lo"][1] - margin < j < b["hi"][1] + margin):
                ok = False
        if ok and (i, j) not in taken:
            taken.add((i, j))
            out.append((i, j))
    return out


def cavity2d(name, config_id, nx, ny, delta, box_lo, box_hi, r, q, dt_factor, n_steps,
             precision, n_rect=0, n_probes=1, pulse="gauss_deriv", f20db=30e9,
             basis=None, seed=None):
    rng = np.random.default_rng(SEED0 + config_id if seed is None else seed)
    eps = np.ones((ny, nx))
    for _ in range(n_rect):
        er = float(rng.uniform(1.0, 4.0))
        w = int(rng.integers(4, 33))
        h = int(rng.integers(4, 33))
        x0 = int(rng.integers(0, nx - w + 1))
        y0 = int(rng.integers(0, ny - h + 1))
        eps[y0:y0 + h, x0:x0 + w] = er          # later draws overwrite
    boxes = [dict(lo=(box_lo[0], box_lo[1], 0), hi=(box_hi[0], box_hi[1], 1), r=(r, r, 1),
                  q=q, model=0, pec_fine=[])]
    src = _pick_nodes(rng, nx, ny, boxes, 1)
    prb = _pick_nodes(rng, nx, ny, boxes, n_probes, exclude=src)
    dt = dt_factor * cfl_coarse(2, delta)
    t = _times(dt, n_steps)
    if pulse == "gauss_deriv":
        w = _gauss_deriv(t, gaussian_derivative_tau(f20db))
    else:
        w = _gauss(t, gaussian_tau(f20db))
    sources = dict(comp=np.array([2]), idx=np.array([[src[0][0], src[0][1], 0]]),
                   wave=w.reshape(n_steps, 1, 1))
    probes = [dict(terms=[(2, (i, j, 0), 1.0)]) for (i, j) in prb]
    if basis is None:
        basis = dict(recipe="A", L=2, M=1.1, fmax=f20db, p=1, seed=SEED0 + config_id)
    return dict(name=name, config_id=config_id, dim=2, n=(nx, ny, 1), delta=delta,
                eps0=EPS0, mu0=MU0, c0=C0, eps_r=eps, boxes=boxes, pec_sheets=[],
                dt=dt, dt_factor=dt_factor, n_steps=n_steps, precision=precision, batch=1,
                sources=sources, probes=probes, init=None, basis=basis)


# ---------------------------------------------------------------------------
# 3-D PEC cavity with random initial E (config 3 and variants)
# ---------------------------------------------------------------------------

def storage_shape3(n):
    nx, ny, nz = n
    return (nz + 1, ny + 1, nx + 1)


def _exists3(n, comp):
    nx, ny, nz = n
    k, j, i = np.indices(storage_shape3(n))
    if comp == 0:
        return (i < nx) & (j > 0) & (j < ny) & (k > 0) & (k < nz)
    if comp == 1:
        return (j < ny) & (i > 0) & (i < nx) & (k > 0) & (k < nz)
    return (k < nz) & (i > 0) & (i < nx) & (j > 0) & (j < ny)


def cavity3d_random(name, config_id, nx, ny, nz, delta, dt_factor, n_steps, precision,
                    eps_r=None, seed=None):
    """E ~ U[-1, 1] on every non-PEC E unknown, H = 0 (survey §8(d) config 3)."""
    rng = np.random.default_rng(SEED0 + config_id if seed is None else seed)
    n = (nx, ny, nz)
    init = {}
    for c in (0, 1, 2):
        a = rng.uniform(-1.0, 1.0, size=storage_shape3(n))
        a[~_exists3(n, c)] = 0.0               # tangential-on-wall entries (and padding) zeroed
        if precision == 32:
            a = a.astype(np.float32).astype(np.float64)   # fp32-rounded start (O12 iv)
        init[c] = a.reshape(1, -1)
    eps = np.ones((nz, ny, nx)) if eps_r is None else eps_r
    dt = dt_factor * cfl_coarse(3, delta)
    probes = [dict(terms=[(2, (nx // 2, ny // 2, nz // 2), 1.0)])]
    return dict(name=name, config_id=config_id, dim=3, n=n, delta=delta, eps0=EPS0, mu0=MU0,
                c0=C0, eps_r=eps, boxes=[], pec_sheets=[], dt=dt, dt_factor=dt_factor,
                n_steps=n_steps, precision=precision, batch=1,
                sources=dict(comp=np.zeros(0, int), idx=np.zeros((0, 3), int),
                             wave=np.zeros((n_steps, 0, 1))),
                probes=probes, init=init, basis=None)


# ---------------------------------------------------------------------------
# registry
# ---------------------------------------------------------------------------

def scenario(which, precision=None, n_steps=None, **kw):
    """Return the scenario dict for a BASELINE config id (1-5) or a named test
    variant.  ``precision`` / ``n_steps`` override the config's defaults."""
    if which == 1:
        s = cavity2d("config1", 1, 40, 20, 1e-3, (16, 6), (24, 14), 4, 32, 0.5, 2000, 64,
                     n_rect=0, n_probes=1, pulse="gauss_deriv", f20db=30e9)
    elif which == 2:
        s = cavity2d("config2", 2, 1024, 1024, 0.5e-3, (480, 480), (544, 544), 8, 256, 0.5,
                     20000, 32, n_rect=32, n_probes=16, pulse="gauss", f20db=30e9,
                     basis=dict(recipe="B", L=2, M=1.1, fmax=30e9, p=4, seed=SEED0 + 2))
    elif which == 3:
        s = cavity3d_random("config3", 3, 256, 256, 256, 1e-3, 0.99, 1000, precision or 32)
    elif which == "tiny2d":
        # several tiles + ragged tail in x and y, one refined box, dielectric blocks
        s = cavity2d("tiny2d", 101, 70, 45, 1e-3, (30, 14), (42, 26), 3, 24, 0.5, 300,
                     precision or 64, n_rect=4, n_probes=3, pulse="gauss_deriv", f20db=30e9)
    elif which == "tiny2d_B":
        s = cavity2d("tiny2d_B", 102, 70, 45, 1e-3, (30, 14), (42, 26), 3, 24, 0.5, 300,
                     precision or 64, n_rect=4, n_probes=3, pulse="gauss", f20db=30e9,
                     basis=dict(recipe="B", L=2, M=1.1, fmax=30e9, p=4, seed=SEED0 + 102))
    elif which == "config1_small":
        s = cavity2d("config1", 1, 40, 20, 1e-3, (16, 6), (24, 14), 4, 32, 0.5, 2000, 64,
                     n_rect=0, n_probes=1, pulse="gauss_deriv", f20db=30e9)
    elif which == "tiny3d":
        s = cavity3d_random("tiny3d", 103, 37, 21, 13, 1e-3, 0.99, 100, precision or 64)
    elif which == "config3_small":
        s = cavity3d_random("config3_small", 3, 64, 48, 40, 1e-3, 0.99, 200, precision or 32)
    else:
        raise KeyError(which)
    if precision is not None and which not in (3, "tiny3d", "config3_small"):
        s["precision"] = precision
    if n_steps is not None and n_steps != s["n_steps"]:
        s["n_steps"] = n_steps
        w = s["sources"]["wave"]
        if w.shape[0] >= n_steps:
            s["sources"]["wave"] = w[:n_steps]
        else:       # beyond the generated record the source is zero (ABI semantics)
            pad = np.zeros((n_steps - w.shape[0],) + w.shape[1:])
            s["sources"]["wave"] = np.concatenate([w, pad], axis=0)
    s.update(kw)
    return s
