"""Stability: Eq. (1) CFL, the singular-value criterion (25)-(26), and the
§III-A perturbation, plus the hybrid split enforcement (DESIGN.md
reading R7, not in the paper).

All plain dense fp64 linear algebra (numpy.linalg.svd / eigh).
"""
from __future__ import annotations

import numpy as np
import scipy.sparse as sp


def cfl_dt(d, c):
    """Eq. (1): dt <= 1 / (c sqrt(1/dx^2 + 1/dy^2 + 1/dz^2)).

    ``d`` lists the spacings of the active axes only (inactive axes contribute
    zero).  ``c`` may be an array of per-cell wave speeds; the per-cell
    minimum is taken (reading R3(i))."""
    s = np.sqrt(sum(1.0 / float(v) ** 2 for v in d))
    return float(np.min(1.0 / (np.asarray(c, dtype=np.float64) * s)))


def _sym_power(D, p):
    """D^p for a positive diagonal (vector) or symmetric positive-definite
    matrix, via the symmetric eigen-decomposition (any square root gives the same
    perturbed K, survey F5)."""
    if np.ndim(D) == 1:
        return np.asarray(D, dtype=np.float64) ** p
    w, Q = np.linalg.eigh(D)
    if np.min(w) <= 0:
        raise ValueError("D is not positive definite")
    return (Q * w ** p) @ Q.T


def _left(Dp, M):
    return Dp[:, None] * M if np.ndim(Dp) == 1 else Dp @ M


def _right(M, Dp):
    return M * Dp[None, :] if np.ndim(Dp) == 1 else M @ Dp


def scaled_curl(De, K, Dm):
    """D_eps^{-1/2} K D_mu^{-1/2}, dense."""
    K = K.toarray() if sp.issparse(K) else np.asarray(K, dtype=np.float64)
    return _right(_left(_sym_power(De, -0.5), K), _sym_power(Dm, -0.5))


def singular_values(De, K, Dm):
    """sigma_i of D_eps^{-1/2} K D_mu^{-1/2}, descending."""
    return np.linalg.svd(scaled_curl(De, K, Dm), compute_uv=False)


def exact_dt_max(De, K, Dm):
    """The exact stability limit 2 / sigma_max implied by (26): R > 0
    iff every sigma_i < 2/dt.  Equals 2/sqrt(rho(D_mu^-1 K^T D_eps^-1 K))."""
    return 2.0 / float(singular_values(De, K, Dm)[0])


def is_R_positive_definite(R) -> bool:
    """Condition (8) checked by a dense Cholesky (small systems only)."""
    try:
        np.linalg.cholesky(R.toarray() if sp.issparse(R) else R)
        return True
    except np.linalg.LinAlgError:
        return False


def enforce(De, K, Dm, dt, gamma=0.9999):
    """§III-A three-step procedure.

    1. SVD  D_eps^{-1/2} K D_mu^{-1/2} = U S W^T
    2. sigma'_i = sigma_i if sigma_i < gamma 2/dt else gamma 2/dt
    3. K' = D_eps^{1/2} U S' W^T D_mu^{1/2}

    Works for rectangular K (the full-system demo of P:316-318 has N_e != N_h).
    Returns (K', report) with report = dict(sigma, sigma_new, n_clipped).
    """
    A = scaled_curl(De, K, Dm)
    U, s, Wt = np.linalg.svd(A, full_matrices=False)
    lim = gamma * 2.0 / dt
    s_new = np.where(s < lim, s, lim)
    Kp = _right(_left(_sym_power(De, 0.5), (U * s_new) @ Wt), _sym_power(Dm, 0.5))
    return Kp, dict(sigma=s, sigma_new=s_new, n_clipped=int(np.sum(s >= lim)), limit=lim)


def split_alpha(dt, dt_coarse):
    """Share of the interface-E mass given to the local block (reading R7):
    alpha = (1 - (dt/dt_c)^2) / 2, valid for dt < dt_c."""
    a = 0.5 * (1.0 - (dt / dt_coarse) ** 2)
    if not (0.0 < a < 0.5):
        raise ValueError(f"split enforcement needs dt < coarse CFL (alpha={a})")
    return a


def enforce_hybrid_block(Dt_e, Kt_rr, S_E, Dt_m, De_if, alpha, dt, gamma=0.9999):
    """Reading R7: clip the local block of the reduced hybrid.

    L = blockdiag(Dt_e, alpha D_eps,if)^{-1/2} [K_rr ; S_E] Dt_m^{-1/2}, a
    (q + n_if) x q matrix, goes through the §III-A procedure as a whole; the
    perturbed rows are written back to K'_rr and S'_E.  With n_if = 0 this is
    exactly §III-A.
    """
    q = Kt_rr.shape[0]
    M = np.vstack([np.asarray(Kt_rr), np.asarray(S_E)])
    if np.ndim(Dt_e) == 1:
        Dl = np.concatenate([np.asarray(Dt_e), alpha * np.asarray(De_if)])
    else:
        n_if = S_E.shape[0]
        Dl = np.zeros((q + n_if, q + n_if))
        Dl[:q, :q] = Dt_e
        Dl[q:, q:] = np.diag(alpha * np.asarray(De_if))
    Mp, rep = enforce(Dl, M, Dt_m, dt, gamma)
    return Mp[:q], Mp[q:], rep


def coarse_piece_sigma_max(De_c, Dm_c, K_cc, if_rows, alpha):
    """sigma_max of blockdiag(D_eps,c with (1-alpha) on the interface rows)^{-1/2}
    K_cc D_mu,c^{-1/2}: the coarse half of the split must satisfy (26) too."""
    De = np.asarray(De_c, dtype=np.float64).copy()
    De[if_rows] *= (1.0 - alpha)
    A = sp.diags(De ** -0.5) @ sp.csr_matrix(K_cc) @ sp.diags(np.asarray(Dm_c) ** -0.5)
    if A.shape[0] * A.shape[1] <= 4.0e6:
        return float(np.linalg.svd(A.toarray(), compute_uv=False)[0])
    import scipy.sparse.linalg as spla
    return float(spla.svds(A.tocsc(), k=1, return_singular_vectors=False, tol=1e-10)[0])
