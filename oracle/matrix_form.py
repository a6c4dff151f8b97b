"""Eqs. (4)-(6): the compact form (R+F) x^{n+1} = (R-F) x^n + B u^{n+1}.

R = [[D_eps/dt, -K/2], [-K^T/2, D_mu/dt]]        F = [[D_se/2, K/2], [-K^T/2, D_sm/2]]
x^n = [E^n ; H^{n+1/2}].

Two ways of advancing it are written here:

* ``step_literal`` forms R+F and R-F explicitly and solves with a sparse
  triangular solve (R+F is block lower-triangular) - the definition.
* ``step_leapfrog`` is the same recursion after subtracting (R+F) x^n from both
  sides:   (R+F)(x^{n+1} - x^n) = -2 F x^n + B u^{n+1},
  solved by block forward substitution with the inverse diagonal blocks
  G_E = (D_eps/dt + D_se/2)^{-1},  G_H = (D_mu/dt + D_sm/2)^{-1}:
      E^{n+1} = E^n + G_E (-K H^n - D_se E^n + B_E u)
      H^{n+1} = H^n + G_H ( K^T E^{n+1} - D_sm H^n + B_H u)
  which is the leap-frog of P:211.  G_E, G_H may be given directly (vectors or
  dense blocks) so that the problem's coefficients enter bit-for-bit
  (reading R8, survey F13).

u follows Eq. (4)'s u^{n+1} = [J^{n+1/2}; M^{n+1}] for the full and the reduced
system alike (reading R2(i); P:110 vs P:178).
"""
from __future__ import annotations

import numpy as np
import scipy.sparse as sp
import scipy.sparse.linalg as spla


def build_RF(De, Dm, K, Dse, Dsm, dt):
    """R and F of Eq. (5) as sparse matrices.  De/Dm may be vectors
    (diagonal) or dense matrices (reduced model, Eq. (13))."""
    def blk(D):
        return sp.diags(D) if np.ndim(D) == 1 else sp.csr_matrix(D)
    K = sp.csr_matrix(K)
    R = sp.bmat([[blk(De) / dt, -0.5 * K], [-0.5 * K.T, blk(Dm) / dt]]).tocsr()
    F = sp.bmat([[0.5 * blk(Dse), 0.5 * K], [-0.5 * K.T, 0.5 * blk(Dsm)]]).tocsr()
    return R, F


def step_literal(x, R, F, Bu):
    """Solve (R+F) x^{n+1} = (R-F) x^n + B u^{n+1} (Eq. (4)) directly."""
    A = (R + F).tocsr()
    rhs = (R - F) @ x + Bu
    if A.shape[0] <= 3000:
        return np.linalg.solve(A.toarray(), rhs)
    return spla.spsolve_triangular(A, rhs, lower=True)


def step_leapfrog(E, H, GE, GH, KE, KH, Dse=None, Dsm=None, su_E=None, su_H=None):
    """One step of (R+F)(x^{n+1}-x^n) = -2F x^n + B u^{n+1} by forward substitution.

    GE, GH : inverse diagonal blocks of R+F (vectors, or callables for dense
             blocks); KE: operator of the E rows (K), KH: operator of the H rows
             (K^T in the paper; passed separately so row-scaled H equations can
             be used, reading R8).  su_E = G_E B_E u, su_H = G_H B_H u
             (source increments, already multiplied by the block inverse).
    """
    def apply(G, v):
        return G(v) if callable(G) else G * v
    rE = -(KE @ H)
    if Dse is not None:
        rE = rE - Dse * E
    E1 = E + apply(GE, rE)
    if su_E is not None:
        E1 = E1 + su_E
    rH = KH @ E1
    if Dsm is not None:
        rH = rH - Dsm * H
    H1 = H + apply(GH, rH)
    if su_H is not None:
        H1 = H1 + su_H
    return E1, H1


def energy(x, R):
    """x^T R x, conserved by the lossless recursion (survey F3)."""
    return float(x @ (R @ x))


def update_matrix(R, F):
    """Dense one-step map (R+F)^{-1}(R-F) whose eigenvalues are the poles of (4)
    (P:140)."""
    A = (R + F).toarray()
    Bm = (R - F).toarray()
    return np.linalg.solve(A, Bm)


def update_eigenvalues(R, F):
    return np.linalg.eigvals(update_matrix(R, F))
