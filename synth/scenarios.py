"""Scenario generators for BASELINE.json configs 1-5 and small test variants.

A scenario is a plain dict (all geometry in coarse cell units):

  name, config_id, dim (2|3), n=(nx, ny, nz) coarse cells (nz=1 in 2-D),
  delta [m], eps0, mu0, c0, eps_r (per cell, [nz][ny][nx] or [ny][nx]),
  boxes: [dict(lo, hi, r, q, model, pec_fine)]  refined regions
  pec_sheets: [dict(axis, plane, lo, hi)]        zero-thickness PEC plates
  dt [s], n_steps, precision (32|64), batch B,
  sources: dict(comp [ns], idx [ns, 3], wave [n_steps][n_cols][B], optional
           column [ns] (shared waveform columns) and amp [ns])     J^{n+1/2}
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
# 3-D rectangular waveguide with a thin refined iris (config 4 and a variant)
# ---------------------------------------------------------------------------

def waveguide3d(name, config_id, nx, ny, nz, delta, slab, rx, iris_cells, aperture_y, q, batch,
                src_x, probe, dt_factor, n_steps, precision, seed=None):
    """PEC-walled guide, coarse x-cells [slab[0], slab[1])
    refined r_x over the full cross-section (tensor-graded, conformal in y, z),
    a PEC iris of iris_cells fine cells at the slab centre with a centred
    aperture of aperture_y cells (full height); B excitations: a Jz sheet with
    the TE10 profile sin(pi y / b) at x = src_x, modulated Gaussians with seeded
    centre frequencies f_c ~ U[0.5, 2] x the TE10 cutoff c/(2b), -20 dB at
    +-f_c/4; one Ez probe per member."""
    rng = np.random.default_rng(SEED0 + config_id if seed is None else seed)
    nfx = (slab[1] - slab[0]) * rx
    fx0 = nfx // 2 - iris_cells // 2
    a0 = (ny - aperture_y) // 2
    a1 = a0 + aperture_y
    iris = [dict(lo=(fx0, 0, 0), hi=(fx0 + iris_cells, a0, nz)),
            dict(lo=(fx0, a1, 0), hi=(fx0 + iris_cells, ny, nz))]
    boxes = [dict(lo=(slab[0], 0, 0), hi=(slab[1], ny, nz), r=(rx, 1, 1), q=q, model=0, pec_fine=iris)]
    fcut = C0 / (2 * ny * delta)
    fc = rng.uniform(0.5, 2.0, size=batch) * fcut
    dt = dt_factor * cfl_coarse(3, delta)
    t = _times(dt, n_steps)
    wave = np.zeros((n_steps, 1, batch))
    for b in range(batch):
        wave[:, 0, b] = _mod_gauss(t, fc[b], gaussian_tau(fc[b] / 4.0))
    idx = [(src_x, j, k) for j in range(1, ny) for k in range(nz)]
    amp = np.array([math.sin(math.pi * j / ny) for (_, j, _) in idx])
    sources = dict(comp=np.full(len(idx), 2), idx=np.array(idx), column=np.zeros(len(idx), np.int32),
                   amp=amp, wave=wave)
    probes = [dict(terms=[(2, probe, 1.0)])]
    basis = dict(recipe="B", points="zero", p=8, seed=SEED0 + config_id)
    return dict(name=name, config_id=config_id, dim=3, n=(nx, ny, nz), delta=delta, eps0=EPS0, mu0=MU0,
                c0=C0, eps_r=np.ones((nz, ny, nx)), boxes=boxes, pec_sheets=[], dt=dt, dt_factor=dt_factor,
                n_steps=n_steps, precision=precision, batch=batch, sources=sources, probes=probes,
                init=None, basis=basis, fc=fc)


# ---------------------------------------------------------------------------
# 3-D microstrip-filter-shaped domain (config 5 and a small variant)
# ---------------------------------------------------------------------------

def _stub_positions(rng, n, lo, hi, width, spacing):
    """n stub x-starts in [lo, hi - width] with pairwise spacing >= spacing:
    the slack beyond the minimum spacing is split at random (seeded)."""
    span = (hi - width) - lo
    slack = span - (n - 1) * spacing
    if slack < 0:
        raise ValueError("stubs do not fit")
    cuts = np.sort(rng.integers(0, slack + 1, size=n))
    return [int(lo + q * spacing + c) for q, c in enumerate(cuts)]


def microstrip3d(name, config_id, nx, ny, nz, delta, n_stub_side, line_x, line_w, sub_k, eps_sub,
                 stub_w, stub_len, region_xy, region_z, rz, q, dt_factor, n_steps, precision,
                 f20db=30e9, seed=None, spacing=10):
    """PEC box, substrate eps_r in z-cells [0, sub_k),
    zero-thickness PEC strips at z = sub_k (a through-line of width line_w,
    y-centred, x in [line_x[0], line_x[1]], and n_stub_side open stubs of width
    stub_w on each side), one refined region (r_z) around every stub tip.
    Regions of one side are exact translated copies -> two shared models."""
    rng = np.random.default_rng(SEED0 + config_id if seed is None else seed)
    eps = np.ones((nz, ny, nx))
    eps[:sub_k] = eps_sub
    y0 = (ny - line_w) // 2
    y1 = y0 + line_w
    zs = sub_k
    sheets = [dict(axis=2, pos=zs, lo=(line_x[0], y0), hi=(line_x[1], y1))]
    boxes = []
    for side, model in ((+1, 0), (-1, 1)):
        xs = _stub_positions(rng, n_stub_side, line_x[0] + 4, line_x[1] - 4, stub_w, spacing)
        lens = rng.integers(stub_len[0], stub_len[1] + 1, size=n_stub_side)
        for sx, L in zip(xs, lens):
            L = int(L)
            if side > 0:
                tip = y1 + L
                sheets.append(dict(axis=2, pos=zs, lo=(sx, y1), hi=(sx + stub_w, tip)))
            else:
                tip = y0 - L
                sheets.append(dict(axis=2, pos=zs, lo=(sx, tip), hi=(sx + stub_w, y0)))
            bx0 = sx - (region_xy - stub_w) // 2
            by0 = tip - region_xy // 2
            boxes.append(dict(lo=(bx0, by0, region_z[0]), hi=(bx0 + region_xy, by0 + region_xy, region_z[1]),
                              r=(1, 1, rz), q=q, model=model, pec_fine=[]))
    dt = dt_factor * cfl_coarse(3, delta)
    t = _times(dt, n_steps)
    w = _gauss(t, gaussian_tau(f20db))
    src_idx = [(line_x[0], j, k) for j in range(y0, y1) for k in range(0, zs)]
    sources = dict(comp=np.full(len(src_idx), 2), idx=np.array(src_idx),
                   column=np.zeros(len(src_idx), np.int32), wave=w.reshape(n_steps, 1, 1))
    jc = (y0 + y1) // 2
    probes = [dict(terms=[(2, (xp, jc, k), delta) for k in range(zs)]) for xp in (line_x[0], line_x[1])]
    basis = dict(recipe="B", L=2, M=1.1, fmax=f20db, p=4, seed=SEED0 + config_id)
    return dict(name=name, config_id=config_id, dim=3, n=(nx, ny, nz), delta=delta, eps0=EPS0, mu0=MU0,
                c0=C0, eps_r=eps, boxes=boxes, pec_sheets=sheets, dt=dt, dt_factor=dt_factor,
                n_steps=n_steps, precision=precision, batch=1, sources=sources, probes=probes,
                init=None, basis=basis)


# ---------------------------------------------------------------------------
# registry
# ---------------------------------------------------------------------------

# ---------------------------------------------------------------------------
# whole-domain reduced model of a 2-D PEC cavity, batched over excitation
# waveforms (stands in for the cavity of P:399-440, Table I)
# ---------------------------------------------------------------------------

def rom_cavity2d(name, config_id, nx, ny, delta, s_factor, q, batch, n_probes=4, fmax=0.5e9,
                 n_steps=None, seed=None):
    """Vacuum PEC cavity of nx x ny cells, one Ez point source, ``n_probes`` Ez
    probes (seeded nodes).  dt = s_factor x the Eq. (1) limit (the CFL
    extension factor s of P:312-315); the step count covers the physical time
    of the paper's 10,000 steps at s = 0.99 (reading A-15).  The batch members
    differ in their time signature: member 0 is the paper's Gaussian pulse
    (-20 dB at fmax), the others are modulated Gaussians with seeded centre
    frequencies in (0.1, 0.8) fmax, bandwidths and amplitudes."""
    rng = np.random.default_rng(SEED0 + config_id if seed is None else seed)
    src = _pick_nodes(rng, nx, ny, [], 1, margin=0)
    prb = _pick_nodes(rng, nx, ny, [], n_probes, margin=0, exclude=src)
    dt = s_factor * cfl_coarse(2, delta)
    if n_steps is None:
        n_steps = int(math.ceil(10000 * 0.99 / s_factor))
    t = _times(dt, n_steps)
    wave = np.zeros((n_steps, batch))
    wave[:, 0] = _gauss(t, gaussian_tau(fmax))
    for b in range(1, batch):
        fc = float(rng.uniform(0.1, 0.8)) * fmax
        tau = gaussian_tau(float(rng.uniform(0.15, 0.4)) * fmax)
        wave[:, b] = _mod_gauss(t, fc, tau)
    amp = rng.uniform(0.5, 1.5, size=(1, batch))
    amp[0, 0] = 1.0
    return dict(name=name, config_id=config_id, dim=2, n=(nx, ny, 1), delta=delta, eps0=EPS0, mu0=MU0, c0=C0,
                eps_r=np.ones((ny, nx)), boxes=[], pec_sheets=[], dt=dt, dt_factor=s_factor, s_factor=s_factor,
                n_steps=n_steps, precision=64, batch=batch, q=q,
                sources=dict(comp=np.array([2]), idx=np.array([[src[0][0], src[0][1], 0]])),
                amp=amp, wave=wave, probes=[dict(terms=[(2, (i, j, 0), 1.0)]) for (i, j) in prb], init=None,
                basis=dict(recipe="A", L=2, M=1.1, fmax=fmax))


# ---------------------------------------------------------------------------
# lossy media and matched absorbers ("4th-order
# matched absorber", 5 cells)
# ---------------------------------------------------------------------------

def absorber_profile(n_cells, axis_len, delta, eps, mu, order=4, thick=5, r0=1e-4):
    """Per-cell conductivity along one axis: a graded layer of ``thick`` cells at
    both ends, sigma_e(x) = sigma_max (depth / L)^order sampled at cell centres,
    sigma_max = -(order + 1) ln(r0) / (2 eta L) (normal-incidence reflection r0
    of the continuous profile), matched magnetic loss sigma_m = sigma_e mu/eps."""
    L = thick * delta
    eta = math.sqrt(mu / eps)
    smax = -(order + 1) * math.log(r0) / (2.0 * eta * L)
    se = np.zeros(n_cells)
    for i in range(thick):
        depth = (thick - i - 0.5) * delta
        v = smax * (depth / L) ** order
        se[i] = v
        se[n_cells - 1 - i] = v
    return se, se * mu / eps


def lossy_box(name, config_id, dim, nx, ny, nz, delta, dt_factor, n_steps, precision, batch=1, axes=(0,),
              eps_slab=2.5, seed=None):
    """PEC box with 5-cell 4th-order matched absorbers on the ends of ``axes``
    (the paper's waveguide / microstrip terminations), a
    lossy dielectric slab (eps_r, sigma_e > 0, unmatched) in the middle, a
    Gaussian-derivative Ez point source and seeded probes."""
    rng = np.random.default_rng(SEED0 + config_id if seed is None else seed)
    shape = (nz, ny, nx) if dim == 3 else (1, ny, nx)
    eps = np.ones(shape)
    se = np.zeros(shape)
    sm = np.zeros(shape)
    x0, x1 = nx // 2 - 2, nx // 2 + 3
    eps[:, :, x0:x1] = eps_slab
    se[:, :, x0:x1] = 0.02                      # a lossy dielectric (S/m), no magnetic loss
    for ax in axes:
        n_ax = (nx, ny, nz)[ax]
        pe, pm = absorber_profile(n_ax, n_ax * delta, delta, EPS0, MU0)
        sh = [1, 1, 1]
        sh[2 - ax] = n_ax
        se = se + pe.reshape(sh)
        sm = sm + pm.reshape(sh)
    dt = dt_factor * cfl_coarse(dim, delta)
    t = _times(dt, n_steps)
    tau = gaussian_derivative_tau(0.25 * C0 / (10 * delta) * 4)
    w = _gauss_deriv(t, tau)
    i0, j0, k0 = nx // 3, ny // 2, (nz // 2 if dim == 3 else 0)
    amps = np.linspace(1.0, -1.4, batch)
    wave = w[:, None, None] * amps[None, None, :]
    prb = []
    for _ in range(3):
        prb.append((int(rng.integers(2, nx - 1)), int(rng.integers(2, ny - 1)), int(rng.integers(1, nz - 1)) if dim == 3 else 0))
    n3 = (nx, ny, nz) if dim == 3 else (nx, ny, 1)
    return dict(name=name, config_id=config_id, dim=dim, n=n3, delta=delta, eps0=EPS0, mu0=MU0, c0=C0,
                eps_r=eps if dim == 3 else eps[0], sigma_e=se if dim == 3 else se[0], sigma_m=sm if dim == 3 else sm[0],
                boxes=[], pec_sheets=[], dt=dt, dt_factor=dt_factor, n_steps=n_steps, precision=precision, batch=batch,
                sources=dict(comp=np.array([2]), idx=np.array([[i0, j0, k0]]), wave=wave),
                probes=[dict(terms=[(2, p, 1.0)]) for p in prb], init=None, basis=None)


def iris_guide2d(name, config_id, precision, irises=True, n_steps=20000, dt_factor=0.99):
    """The 2-D iris waveguide of P:515-517 from its description: 5 cm x 50 cm,
    40 x 400 cells of 1.25 mm (x along the guide), eps_r = 2.5, PEC side walls,
    five PEC irises 50 cells apart (2 nodes thick with a 16-cell centred aperture:
    the printed "length 1.25 cm, aperture 1 cm" is opaque below 9 GHz when read
    as a 10-cell-long 8-cell-wide channel, so the stand-in uses thin inductive
    irises that form a band-pass filter inside the 3 GHz band),
    5-cell 4th-order matched absorbers at both ends, a Gaussian current line
    source (-20 dB at 3 GHz) near one end and a line probe (sum of Ez across the
    guide) near the other.  ``irises=False``: the empty guide (S21 reference)."""
    nx, ny, delta = 400, 40, 1.25e-3
    eps_r = 2.5
    pe, pm = absorber_profile(nx, nx * delta, delta, eps_r * EPS0, MU0)
    se = np.tile(pe, (ny, 1))
    sm = np.tile(pm, (ny, 1))
    dt = dt_factor * cfl_coarse(2, delta) * math.sqrt(eps_r)       # Eq. (1) with the guide's wave speed
    t = _times(dt, n_steps)
    w = _gauss(t, gaussian_tau(3e9))
    js = np.arange(1, ny)
    xs, xp = 20, 380
    sources = dict(comp=np.full(len(js), 2), idx=np.array([[xs, j, 0] for j in js]),
                   column=np.zeros(len(js), np.int32), wave=w.reshape(n_steps, 1, 1))
    probes = [dict(terms=[(2, (xp, int(j), 0), delta) for j in js]),
              dict(terms=[(2, (xs + 20, int(j), 0), delta) for j in js])]
    blocks = []
    if irises:
        for q in range(5):
            x0 = 95 + 50 * q
            blocks.append(dict(lo=(x0, 0), hi=(x0 + 1, 12)))
            blocks.append(dict(lo=(x0, 28), hi=(x0 + 1, ny)))
    return dict(name=name, config_id=config_id, dim=2, n=(nx, ny, 1), delta=delta, eps0=EPS0, mu0=MU0, c0=C0,
                eps_r=np.full((ny, nx), eps_r), sigma_e=se, sigma_m=sm, boxes=[], pec_sheets=[], pec_blocks=blocks,
                dt=dt, dt_factor=dt_factor, n_steps=n_steps, precision=precision, batch=1, sources=sources,
                probes=probes, init=None, basis=None)


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
    elif which == 4:
        s = waveguide3d("config4", 4, 512, 128, 128, 0.5e-3, (255, 257), 10, 2, 48, 1024, 16, 32,
                        (480, 64, 64), 0.8, 10000, precision or 32)
    elif which == "tiny4":
        s = waveguide3d("tiny4", 104, 48, 12, 10, 0.5e-3, (23, 25), 4, 2, 4, 24, 4, 5, (40, 6, 5),
                        0.8, 300, precision or 64)
    elif which == 5:
        s = microstrip3d("config5", 5, 400, 200, 40, 0.25e-3, 32, (20, 380), 9, 4, 3.38, 4, (10, 60),
                         8, (3, 5), 10, 128, 0.6, 50000, precision or 32)
    elif which == "tiny5":
        # config-5 structure on a small domain: 2 stubs per side, r_z = 4, q = 16
        s = microstrip3d("tiny5", 105, 60, 48, 10, 0.25e-3, 2, (6, 54), 5, 3, 3.38, 3, (6, 12),
                         6, (2, 4), 4, 16, 0.6, 300, precision or 64, spacing=12)
    elif which == "micro4":
        # config-4 structure small enough for a dense eigen-decomposition of the
        # whole reduced-hybrid update matrix (brute-force stability, ~2 K unknowns)
        s = waveguide3d("micro4", 106, 12, 5, 4, 0.5e-3, (5, 7), 4, 2, 1, 8, 1, 2, (10, 2, 2),
                        0.8, 100, precision or 64)
    elif which == "micro5":
        # config-5 structure (PEC strips through z-refined regions, two models)
        s = microstrip3d("micro5", 107, 14, 12, 4, 0.25e-3, 1, (2, 12), 2, 2, 3.38, 2, (2, 2),
                         4, (1, 3), 4, 8, 0.6, 100, precision or 64, spacing=4)
    elif which == "lossy3d":
        s = lossy_box("lossy3d", 301, 3, 70, 23, 19, 1e-3, 0.95, 400, precision or 64, axes=(0,))
    elif which == "lossy3d_b16":
        s = lossy_box("lossy3d_b16", 302, 3, 30, 11, 9, 1e-3, 0.95, 300, precision or 32, batch=16, axes=(0, 1))
    elif which == "lossy256":
        # config 3's grid with matched absorbers on the x and y ends and a lossy slab (throughput of the lossy stencil)
        s = lossy_box("lossy256", 304, 3, 256, 256, 256, 1e-3, 0.95, 1000, precision or 32, axes=(0, 1))
    elif which == "iris_guide":
        s = iris_guide2d("iris_guide", 305, precision or 32, irises=True)
    elif which == "iris_guide_empty":
        s = iris_guide2d("iris_guide_empty", 305, precision or 32, irises=False)
    elif which == "lossy2d":
        s = lossy_box("lossy2d", 303, 2, 90, 61, 1, 1e-3, 0.95, 500, precision or 64, axes=(0, 1))
    elif which == "rom2d":
        # the paper's 2-D cavity (Table I: 101 cells of 1 cm, order 80, 5 points,
        # M = 1.1, f_max = 0.5 GHz) at s = 4.95, 64 excitation waveforms
        s = rom_cavity2d("rom2d", 201, 101, 101, 0.01, kw.pop("s_factor", 4.95), kw.pop("q", 80),
                         kw.pop("batch", 64))
    elif which == "rom2d_small":
        s = rom_cavity2d("rom2d_small", 202, 24, 18, 0.01, kw.pop("s_factor", 2.5), kw.pop("q", 20),
                         kw.pop("batch", 11), n_probes=3, fmax=4e9, n_steps=400)
    elif which == "config3_small":
        s = cavity3d_random("config3_small", 3, 64, 48, 40, 1e-3, 0.99, 200, precision or 32)
    else:
        raise KeyError(which)
    if precision is not None and which not in (3, "tiny3d", "config3_small", 4, "tiny4", 5, "tiny5", "micro4",
                                               "micro5"):
        s["precision"] = precision
    if n_steps is not None and n_steps != s["n_steps"]:
        s["n_steps"] = n_steps
        holder = s["sources"] if "wave" in s["sources"] else s     # reduced-model scenarios keep wave at top level
        w = holder["wave"]
        if w.shape[0] >= n_steps:
            holder["wave"] = w[:n_steps]
        else:       # beyond the generated record the source is zero (ABI semantics)
            pad = np.zeros((n_steps - w.shape[0],) + w.shape[1:])
            holder["wave"] = np.concatenate([w, pad], axis=0)
    s.update(kw)
    return s
