"""Physics checks used to pin the oracle (not parity targets).

* analytic PEC-cavity resonances ("Analytical resonant frequencies ...
  used as accuracy metric"; P:311 the cube's 0.21199 / 0.25963 GHz),
* the exact resonances of the *discrete* lossless leap-frog: a mode whose
  scaled-curl singular value is sigma rotates by theta = 2 arcsin(dt sigma / 2)
  per step (survey F4), i.e. f = arcsin(dt sigma / 2) / (pi dt),
* spectral peak picking on probe series (S:444-461 conventions: rectangular
  window, zero padding, parabolic refinement).
"""
from __future__ import annotations

import itertools

import numpy as np


def cavity_modes(lengths, c, eps_r=1.0, count=10, dim=3, mmax=12):
    """f = c/(2 sqrt(eps_r)) sqrt(sum (m_i/L_i)^2).  2-D Ez (TM):
    m, n >= 1.  3-D: at least two indices non-zero.  Ascending, deduplicated."""
    vals = set()
    for ms in itertools.product(range(mmax + 1), repeat=len(lengths)):
        nz = sum(1 for m in ms if m > 0)
        if dim == 2 and nz < 2:
            continue
        if dim == 3 and nz < 2:
            continue
        f = c / (2.0 * np.sqrt(eps_r)) * np.sqrt(sum((m / L) ** 2 for m, L in zip(ms, lengths)))
        vals.add(round(f, 3))
    return np.array(sorted(vals)[:count])


def discrete_frequency(sigma, dt):
    """Frequency of a lossless leap-frog mode with scaled-curl singular value
    sigma: the update eigenvalues are exp(+-j theta), theta = 2 arcsin(dt sigma/2)
    (survey F4), f = theta / (2 pi dt)."""
    return np.arcsin(np.clip(dt * np.asarray(sigma) / 2.0, -1, 1)) / (np.pi * dt)


def spectrum(series, dt, pad_factor=4, window=None):
    n = len(series)
    nfft = 1 << int(np.ceil(np.log2(pad_factor * n)))
    x = np.asarray(series, dtype=np.float64)
    if window == "hann":            # suppresses the sidelobes of undamped modes
        x = x * np.hanning(n)
    X = np.fft.rfft(x, nfft)
    f = np.fft.rfftfreq(nfft, dt)
    return f, np.abs(X)


def find_peaks(f, mag, prominence=0.05, fmin=0.0, fmax=np.inf, max_count=20):
    """Local maxima above prominence * global max within [fmin, fmax], refined by
    a parabola through three bins."""
    sel = (f >= fmin) & (f <= fmax)
    top = mag[sel].max()
    out = []
    for i in range(1, len(mag) - 1):
        if not sel[i]:
            continue
        if mag[i] > mag[i - 1] and mag[i] >= mag[i + 1] and mag[i] >= prominence * top:
            a, b, c = np.log(mag[i - 1] + 1e-300), np.log(mag[i] + 1e-300), np.log(mag[i + 1] + 1e-300)
            den = a - 2 * b + c
            p = 0.5 * (a - c) / den if den != 0 else 0.0
            out.append(f[i] + p * (f[1] - f[0]))
    return np.array(out[:max_count])
