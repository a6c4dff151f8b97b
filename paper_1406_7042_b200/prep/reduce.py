"""Offline model-order reduction of the refined boxes (host preprocessing).

* expansion points, Eq. (19)
* shifted solves [z(R+F) - (R-F)] x = b with the 2x2 block Schur elimination
  of P:373-392 (A11, A22 diagonal) and a sparse LU of the Schur complement
  ("one LU decomposition in 2-D"); sign per reading R5(i)
* multi-point block Arnoldi (readings R5(iv),(v),(vii)):
  MGS with one re-orthogonalisation per point, realified columns split into
  E and H parts, deflation at 1e-8, truncation to q each
* D-orthonormalisation (R5(vi)), projection (14)-(16)
* stability enforcement: §III-A applied to the local block of
  the hybrid (reading R7).
"""
from __future__ import annotations

import math

import numpy as np
import scipy.sparse as sp
import scipy.sparse.linalg as spla

GAMMA = 0.9999


def expansion_points(M, L, fmax, dt):
    """Representatives of z_l = M exp(j 2 pi (l/L) fmax dt), l = -L..L: l = 0..L
    (conjugate points give conjugate Krylov vectors, no new real information)."""
    if fmax * dt >= 0.5:
        raise ValueError("f_max * dt must be < 1/2 (aliasing)")
    if L == 0:
        return [complex(M, 0.0)]
    return [M * complex(math.cos(2 * math.pi * l / L * fmax * dt), math.sin(2 * math.pi * l / L * fmax * dt))
            for l in range(0, L + 1)]


class ShiftedSolver:
    """Solves [z(R+F) - (R-F)] x = b for the lossless system with blocks
    A11 = (z-1) De/dt, A12 = K, A21 = -z K^T, A22 = (z-1) Dm/dt."""

    def __init__(self, De, Dm, K, dt, z):
        z = complex(z)
        self.real = z.imag == 0.0
        self.z = z.real if self.real else z
        self.dt = dt
        dtype = np.float64 if self.real else np.complex128
        self.K = K.tocsr().astype(dtype)
        self.KT = K.T.tocsr().astype(dtype)
        self.a11 = (self.z - 1.0) * De / dt
        self.a22 = (self.z - 1.0) * Dm / dt
        if self.z == 0:
            # the z = 0 fast path of P:371: R - F is block upper triangular,
            # so the solve is a back substitution (no factorisation)
            self.lu = None
        else:
            # Schur complement A11 - A12 A22^-1 A21 = A11 + z K A22^-1 K^T
            Sc = sp.diags(self.a11) + self.z * (self.K @ sp.diags(1.0 / self.a22) @ self.KT)
            self.lu = spla.splu(Sc.tocsc())

    def solve(self, b1, b2):
        rhs = b1 - self.K @ (b2 / self.a22[:, None])
        x1 = rhs / self.a11[:, None] if self.lu is None else self.lu.solve(rhs)
        x2 = (b2 + self.z * (self.KT @ x1)) / self.a22[:, None]
        return x1, x2


class _Basis:
    """Growing orthonormal vector set (real or complex), preallocated with one
    vector per ROW so that the active part is contiguous; new blocks are
    orthogonalised by block classical Gram-Schmidt applied twice (CGS2,
    numerically equivalent to MGS with re-orthogonalisation) followed by MGS
    within the block, with deflation of vectors whose norm drops below tol x
    their original norm (R5(vii))."""

    def __init__(self, n, cap, dtype, tol):
        self.Vt = np.zeros((cap, n), dtype)
        self.k = 0
        self.tol = tol
        self.cplx = np.issubdtype(np.dtype(dtype), np.complexfloating)

    def _proj(self, A, W):            # W -= A^H (A W), A rows = basis vectors, W cols
        # A^H W computed as conj(A conj(W)) so the large basis is never copied
        G = np.conj(A @ np.conj(W)) if self.cplx else A @ W
        W -= A.T @ G
        return W

    def add(self, X, limit=None):
        cap = self.Vt.shape[0]
        limit = cap if limit is None else min(limit, cap)
        out = []
        if self.k >= limit or X.shape[1] == 0:
            return out
        nrm0 = np.linalg.norm(X, axis=0)
        W = np.array(X, dtype=self.Vt.dtype, copy=True)
        for _ in range(2):
            if self.k:
                W = self._proj(self.Vt[:self.k], W)
        start = self.k
        for j in range(W.shape[1]):
            if self.k >= limit:
                break
            w = W[:, j:j + 1].copy()
            for _ in range(2):
                if self.k > start:
                    w = self._proj(self.Vt[start:self.k], w)
            nrm = np.linalg.norm(w)
            if nrm0[j] > 0 and nrm > self.tol * nrm0[j]:
                self.Vt[self.k] = w[:, 0] / nrm
                out.append(self.k)
                self.k += 1
        return out

    @property
    def cols(self):
        return self.Vt[:self.k].T


def krylov_basis(De, Dm, K, dt, B, keep_e, keep_h, q, points, max_iter=None, window_bytes=4e9):
    """Multi-point block Arnoldi on (R+F)/(R-F) of the lossless system (De, Dm, K)
    started at A(z)^{-1} B; the rows keep_e / keep_h of each realified Krylov
    block feed the V1 / V2 pools (round-robin over the points, R5(iv)).
    Returns (V1, V2) with q columns each."""
    Ne, Nh = K.shape
    max_iter = max_iter or 4 * q
    P1 = _Basis(len(keep_e), q, np.float64, 1e-8)
    P2 = _Basis(len(keep_h), q, np.float64, 1e-8)
    solvers = [ShiftedSolver(De, Dm, K, dt, z) for z in points]
    cap = 2 * max_iter * B.shape[1] // max(len(points), 1) + 4 * B.shape[1]
    cap = min(cap, 4 * q + 4 * B.shape[1])
    # large systems keep only a window of recent Krylov blocks per point for
    # the re-orthogonalisation (partial reorthogonalisation); the V pools are
    # always fully orthogonalised
    if (Ne + Nh) * cap * 16 > window_bytes:
        cap = max(4 * B.shape[1], int(window_bytes // ((Ne + Nh) * 16)) // B.shape[1] * B.shape[1])
        windowed = True
    else:
        windowed = False
    Qs, nxt = [], []
    for s in solvers:
        dt_ = np.float64 if s.real else np.complex128
        x1, x2 = s.solve(B[:Ne].astype(dt_), B[Ne:].astype(dt_))
        Qs.append(_Basis(Ne + Nh, cap, dt_, 1e-10))
        nxt.append(np.vstack([x1, x2]))
    it = 0
    while not (P1.k >= q and P2.k >= q) and it < max_iter:
        progressed = False
        for pi, s in enumerate(solvers):
            Q, X = Qs[pi], nxt[pi]
            if windowed and Q.k + X.shape[1] > Q.Vt.shape[0]:
                keep = Q.Vt.shape[0] // 2               # slide the window
                Q.Vt[:keep] = Q.Vt[Q.k - keep:Q.k]
                Q.k = keep
            if X.shape[1] == 0 or Q.k >= Q.Vt.shape[0]:
                continue
            idx = Q.add(X)
            if not idx:
                nxt[pi] = X[:, :0]
                continue
            progressed = True
            Wb = Q.Vt[idx].T
            real = Wb if s.real else np.hstack([Wb.real, Wb.imag])
            P1.add(real[:Ne][keep_e], q)
            P2.add(real[Ne:][keep_h], q)
            # next block: A^{-1} (R+F) W,   (R+F) = [[De/dt, 0], [-K^T, Dm/dt]]
            wE, wH = Wb[:Ne], Wb[Ne:]
            b1 = (De / dt)[:, None] * wE
            b2 = -(s.KT @ wE) + (Dm / dt)[:, None] * wH
            x1, x2 = s.solve(b1, b2)
            nxt[pi] = np.vstack([x1, x2])
            if P1.k >= q and P2.k >= q:
                break
        if not progressed:
            break
        it += 1
    if not (P1.k >= q and P2.k >= q):
        raise RuntimeError(f"Krylov basis stalled at {P1.k}/{P2.k} of {q} columns")
    return P1.cols.copy(), P2.cols.copy()


def d_orthonormalise(V, D):
    """Columns made orthonormal in <x, y>_D = x^T diag(D) y (same span)."""
    G = V.T @ (D[:, None] * V)
    L = np.linalg.cholesky(0.5 * (G + G.T))
    return np.linalg.solve(L, V.T).T


def project(V1, V2, Kff, Kcf):
    """K~_rr = V1^T K_ff V2, S_E = K_cf V2 (Eqs. (14)-(16) with the partial
    projection of reading R6)."""
    return V1.T @ (Kff @ V2), np.asarray(Kcf @ V2)


def enforce_block(Kt, SE, De_if, alpha, dt, gamma=GAMMA):
    """Reading R7: §III-A on L = blockdiag(I, alpha D_eps,if)^{-1/2} [K~; S_E]
    (D~ = I after D-orthonormalisation).  Returns (K~', S_E', info)."""
    q = Kt.shape[0]
    d = np.concatenate([np.ones(q), alpha * np.asarray(De_if)])
    sc = 1.0 / np.sqrt(d)
    L = sc[:, None] * np.vstack([Kt, SE])
    U, s, Wt = np.linalg.svd(L, full_matrices=False)
    lim = gamma * 2.0 / dt
    s2 = np.minimum(s, lim)
    Lp = (U * s2) @ Wt
    M = np.sqrt(d)[:, None] * Lp
    return M[:q], M[q:], dict(sigma_max=float(s[0]), sigma_max_new=float(s2[0]),
                              n_clipped=int(np.sum(s >= lim)), limit=lim)
