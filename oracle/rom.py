"""Oracle of the whole-domain reduced model (TEST INFRASTRUCTURE ONLY: imported
by tests/, __graft_entry__.smoke() and bench.py's CPU legs, never by the
product path).

The paper's reduced system, Eq. (12),

    (R~ + F~) x~^{n+1} = (R~ - F~) x~^n + B~ u^{n+1},     x~ = [e~; h~],

with the blocks of Eq. (13)

    R~ = [[D~e/dt, -K~/2], [-K~^T/2, D~m/dt]]   F~ = [[D~se/2, K~/2], [-K~^T/2, D~sm/2]],

is advanced by block forward substitution: R~ + F~ is block lower triangular
(P:79-96), so

    (D~e/dt + D~se/2) e~'            = (D~e/dt - D~se/2) e~ - K~ h~ + B~_e u
    (D~m/dt + D~sm/2) h~'            = (D~m/dt - D~sm/2) h~ + K~^T e~'

(the leap-frog of P:211), each left-hand block solved by a Cholesky
factorisation (dense D~ of Eq. (14); no precomputed inverses).  u^{n+1} =
J^{n+1/2} for step n (reading R2(i)); probes are rows of V applied to the
reduced state (Eq. (10)), E after the E half, H after the H half
(reading R12).  All columns of a batch are advanced together by plain matrix
products: they are independent.

Pins (tests/test_oracle_rom.py): the closed-form rotation of a single mode
(survey F4: theta = 2 arcsin(dt sigma / 2)), conservation of x~^T R~ x~ (F3),
the identity basis reproducing the full FDTD recursion of matrix_form, the
late-time bound of E7, and the resonances of the paper's 2-D cavity
within 1 % of the analytic modes.
"""
from __future__ import annotations

import numpy as np
import scipy.linalg as sla


def _dense(D, q):
    if D is None:
        return np.eye(q)
    D = np.asarray(D, np.float64)
    return np.diag(D) if D.ndim == 1 else D


def blocks(model):
    """The dense blocks of Eq. (13) from a model dict: K [q_e][q_h], optional
    De, Dm, Dse, Dsm (dense, diagonal vectors, or None = I / 0), dt."""
    K = np.asarray(model["K"], np.float64)
    qe, qh = K.shape
    De, Dm = _dense(model.get("De"), qe), _dense(model.get("Dm"), qh)
    Dse = np.zeros((qe, qe)) if model.get("Dse") is None else _dense(model["Dse"], qe)
    Dsm = np.zeros((qh, qh)) if model.get("Dsm") is None else _dense(model["Dsm"], qh)
    return K, De, Dm, Dse, Dsm


def RF(model):
    """R~ and F~ of Eq. (13) as dense matrices."""
    K, De, Dm, Dse, Dsm = blocks(model)
    dt = float(model["dt"])
    R = np.block([[De / dt, -0.5 * K], [-0.5 * K.T, Dm / dt]])
    F = np.block([[0.5 * Dse, 0.5 * K], [-0.5 * K.T, 0.5 * Dsm]])
    return R, F


def run(model, amp, wave, n_steps, state=None, start_step=0):
    """Advance Eq. (12) for ``n_steps`` steps.  amp [n_in][B], wave [n_wave][B]:
    u^{n+1}[:, b] = amp[:, b] wave[n][b] (zero beyond the record).  Returns
    (e~ [q_e][B], h~ [q_h][B], probes [n_steps][n_out_e + n_out_h][B])."""
    K, De, Dm, Dse, Dsm = blocks(model)
    dt = float(model["dt"])
    qe, qh = K.shape
    amp = np.asarray(amp, np.float64).reshape(-1, np.asarray(wave).shape[1] if np.ndim(wave) == 2 else 1)
    wave = np.asarray(wave, np.float64).reshape(-1, amp.shape[1])
    Bn = amp.shape[1]
    Be = np.asarray(model["B_e"], np.float64).reshape(qe, -1)
    Le = None if model.get("L_e") is None else np.asarray(model["L_e"], np.float64).reshape(-1, qe)
    Lh = None if model.get("L_h") is None else np.asarray(model["L_h"], np.float64).reshape(-1, qh)
    cE = sla.cho_factor(De / dt + 0.5 * Dse)
    cH = sla.cho_factor(Dm / dt + 0.5 * Dsm)
    ME = De / dt - 0.5 * Dse
    MH = Dm / dt - 0.5 * Dsm
    e = np.zeros((qe, Bn)) if state is None else np.array(state[0], np.float64).reshape(qe, Bn)
    h = np.zeros((qh, Bn)) if state is None else np.array(state[1], np.float64).reshape(qh, Bn)
    n_out = (0 if Le is None else Le.shape[0]) + (0 if Lh is None else Lh.shape[0])
    probes = np.zeros((n_steps, n_out, Bn))
    for s in range(n_steps):
        n = start_step + s
        u = amp * wave[n][None, :] if n < wave.shape[0] else np.zeros_like(amp)
        e = sla.cho_solve(cE, ME @ e - K @ h + Be @ u)
        k = 0
        if Le is not None:
            probes[s, :Le.shape[0]] = Le @ e
            k = Le.shape[0]
        h = sla.cho_solve(cH, MH @ h + K.T @ e)
        if Lh is not None:
            probes[s, k:] = Lh @ h
    return e, h, probes


def energy(model, e, h):
    """x~^T R~ x~ per batch column (conserved when lossless, survey F3)."""
    R, _ = RF(model)
    x = np.vstack([e, h])
    return np.einsum("ib,ij,jb->b", x, R, x)
