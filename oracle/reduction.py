"""SPRIM-style projection (Eqs. (9)-(16)) and the quantities used to
check a basis: expansion points (Eq. (19)) and transfer functions.

The oracle does not generate Krylov bases (they are not unique across
implementations, survey §8(c)); it verifies the bases the preprocessing emits
through properties the paper fixes: orthonormality, moment matching at
the expansion points, congruence/structure.
"""
from __future__ import annotations

import numpy as np
import scipy.sparse as sp
import scipy.sparse.linalg as spla


def expansion_points(M, L, fmax, dt):
    """z_l = M exp(j 2 pi (l/L) fmax dt), l = -L..L (Eq. (19)).  L = 0
    would divide by zero; the single point z = M is used (reading R5(ii))."""
    if L == 0:
        return np.array([complex(M)])
    l = np.arange(-L, L + 1)
    return M * np.exp(1j * 2 * np.pi * (l / L) * fmax * dt)


def project(V1, V2, De, Dm, K, Dse=None, Dsm=None, B=None):
    """Eqs. (14)-(16): D~ = V^T D V, K~ = V1^T K V2, B~ = V^T B."""
    def dproj(V, D):
        return V.T @ (D[:, None] * V) if np.ndim(D) == 1 else V.T @ (D @ V)
    out = dict(De=dproj(V1, De), Dm=dproj(V2, Dm), K=V1.T @ (K @ V2))
    if Dse is not None:
        out["Dse"] = dproj(V1, Dse)
    if Dsm is not None:
        out["Dsm"] = dproj(V2, Dsm)
    if B is not None:
        Ne = V1.shape[0]
        Bd = B.toarray() if sp.issparse(B) else np.asarray(B)
        out["B"] = np.vstack([V1.T @ Bd[:Ne], V2.T @ Bd[Ne:]])
    return out


def shifted_operator(R, F, z):
    """z (R+F) - (R-F): the resolvent of recursion (4) in the z domain.  The
    printed P:358 has (R-F) + z(R+F); reading R5(i) / survey F6 adopts this
    sign, the one consistent with 'z = 1 corresponds to static conditions'
    (P:349)."""
    return (z * (R + F) - (R - F)).tocsc() if sp.issparse(R) else z * (R + F) - (R - F)


def transfer(R, F, B, C, z):
    """C^T (z(R+F) - (R-F))^{-1} B at complex z (state response to u)."""
    A = shifted_operator(R, F, z)
    Bd = B.toarray() if sp.issparse(B) else np.asarray(B)
    if sp.issparse(A):
        X = spla.spsolve(A, Bd.astype(complex))
        X = X.reshape(A.shape[0], -1)
    else:
        X = np.linalg.solve(A, Bd.astype(complex))
    Cd = C.toarray() if sp.issparse(C) else np.asarray(C)
    return Cd.T @ X


def random_orthonormal(n, k, rng):
    Q, _ = np.linalg.qr(rng.standard_normal((n, k)))
    return Q


def d_orthonormal(V, D):
    """Re-orthonormalise the columns of V in the <.,.>_D inner product (V^T D V = I),
    a congruence within the same subspace (reading R5(vi))."""
    G = V.T @ ((D[:, None] * V) if np.ndim(D) == 1 else D @ V)
    Lc = np.linalg.cholesky(G)
    return np.linalg.solve(Lc, V.T).T
