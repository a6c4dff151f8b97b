"""Eq. (3) assembly on uniform Yee grids, plain fp64.

The paper states the matrix form (3) with
  * D_eps, D_mu   diagonal permittivity / permeability per unknown,
  * D_sig_e/m     diagonal conductivities,
  * K             "the discretization of the curl operators ... terms in the form
                  (+-1/dx, +-1/dy, +-1/dz)",
  * B             1's at source locations,
arranged so that   (D_eps/dt) dE = -K H + B u   and   (D_mu/dt) dH = K^T E
(rows of (3)).  K is built here from the E equations, i.e. from
Ampere's law eps dE/dt = curl H - J, so K = -(discrete curl acting on H).  The
H equations are built *independently* from Faraday's law mu dH/dt = -curl E,
and ``assemble`` returns that operator too, so the tests can check the
paper's claim that the H rows carry K^T of the same matrix (reading R1(i):
Eq. (2b)'s printed curl sign is inconsistent with (3); see tests/test_oracle_yee).

Unknown naming follows the storage convention used everywhere in this repo
(DESIGN.md §5): a component array indexed [k][j][i] holds
  Ex(i+1/2, j, k)   Ey(i, j+1/2, k)   Ez(i, j, k+1/2)
  Hx(i, j+1/2, k+1/2)   Hy(i+1/2, j, k+1/2)   Hz(i+1/2, j+1/2, k)
and in 2-D (the paper's TM case with Ez) [j][i] holds
  Ez(i, j)   Hx(i, j+1/2)   Hy(i+1/2, j).
Component ids: Ex=0 Ey=1 Ez=2 Hx=3 Hy=4 Hz=5 (2-D uses 2, 3, 4).

PEC walls eliminate tangential E and normal H unknowns (reading
R1(ii)).  Unknown order: all E then all H, component-major, then lexicographic
(k, j, i) with i fastest.  Materials: owning cell, no averaging:
the unknown at storage index (i, j, k) takes the cell (min(i,nx-1),
min(j,ny-1), min(k,nz-1)).
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np
import scipy.sparse as sp

E_COMPS_3D = (0, 1, 2)
H_COMPS_3D = (3, 4, 5)
E_COMPS_2D = (2,)
H_COMPS_2D = (3, 4)
COMP_NAMES = ("Ex", "Ey", "Ez", "Hx", "Hy", "Hz")

# curl H at each E component: list of (H comp, (di, dj, dk), sign, axis of the
# difference).  Straight transcription of (curl H)_x = dHz/dy - dHy/dz etc. on
# the staggered grid.
_CURL_H_3D = {
    0: [(5, (0, 0, 0), +1, 1), (5, (0, -1, 0), -1, 1),
        (4, (0, 0, 0), -1, 2), (4, (0, 0, -1), +1, 2)],
    1: [(3, (0, 0, 0), +1, 2), (3, (0, 0, -1), -1, 2),
        (5, (0, 0, 0), -1, 0), (5, (-1, 0, 0), +1, 0)],
    2: [(4, (0, 0, 0), +1, 0), (4, (-1, 0, 0), -1, 0),
        (3, (0, 0, 0), -1, 1), (3, (0, -1, 0), +1, 1)],
}
# -curl E at each H component (Faraday: mu dH/dt = -curl E).
_MCURL_E_3D = {
    3: [(2, (0, 1, 0), -1, 1), (2, (0, 0, 0), +1, 1),
        (1, (0, 0, 1), +1, 2), (1, (0, 0, 0), -1, 2)],
    4: [(0, (0, 0, 1), -1, 2), (0, (0, 0, 0), +1, 2),
        (2, (1, 0, 0), +1, 0), (2, (0, 0, 0), -1, 0)],
    5: [(1, (1, 0, 0), -1, 0), (1, (0, 0, 0), +1, 0),
        (0, (0, 1, 0), +1, 1), (0, (0, 0, 0), -1, 1)],
}
# 2-D Ez polarisation: eps dEz/dt = dHy/dx - dHx/dy ; mu dHx/dt = -dEz/dy ;
# mu dHy/dt = +dEz/dx.
_CURL_H_2D = {
    2: [(4, (0, 0, 0), +1, 0), (4, (-1, 0, 0), -1, 0),
        (3, (0, 0, 0), -1, 1), (3, (0, -1, 0), +1, 1)],
}
_MCURL_E_2D = {
    3: [(2, (0, 1, 0), -1, 1), (2, (0, 0, 0), +1, 1)],
    4: [(2, (1, 0, 0), +1, 0), (2, (0, 0, 0), -1, 0)],
}


def storage_shape(dim: int, n) -> tuple:
    """Shape of one component array: (nz+1, ny+1, nx+1) in 3-D, (ny+1, nx+1) in 2-D."""
    nx, ny, nz = n
    return (nz + 1, ny + 1, nx + 1) if dim == 3 else (ny + 1, nx + 1)


def exists_mask(dim: int, n, comp: int) -> np.ndarray:
    """True where storage index (i, j, k) holds a real unknown of ``comp``."""
    nx, ny, nz = n
    shp = storage_shape(dim, n)
    m = np.ones(shp, dtype=bool)
    if dim == 3:
        k, j, i = np.indices(shp)
        lim = {0: (i < nx), 1: (j < ny), 2: (k < nz),
               3: (j < ny) & (k < nz), 4: (i < nx) & (k < nz), 5: (i < nx) & (j < ny)}
        return m & lim[comp]
    j, i = np.indices(shp)
    lim = {2: np.ones(shp, bool), 3: (j < ny), 4: (i < nx)}
    return m & lim[comp]


def wall_pec_mask(dim: int, n, comp: int) -> np.ndarray:
    """True where a PEC wall eliminates the unknown: tangential E, normal H."""
    nx, ny, nz = n
    shp = storage_shape(dim, n)
    if dim == 3:
        k, j, i = np.indices(shp)
        xw, yw, zw = (i == 0) | (i == nx), (j == 0) | (j == ny), (k == 0) | (k == nz)
        table = {0: yw | zw, 1: xw | zw, 2: xw | yw, 3: xw, 4: yw, 5: zw}
        return table[comp]
    j, i = np.indices(shp)
    xw, yw = (i == 0) | (i == nx), (j == 0) | (j == ny)
    return {2: xw | yw, 3: xw, 4: yw}[comp]


def owning_cell(dim: int, n, shape=None):
    """Owning-cell index arrays: clamp storage index into the cell range."""
    nx, ny, nz = n
    shp = storage_shape(dim, n) if shape is None else shape
    if dim == 3:
        k, j, i = np.indices(shp)
        return np.minimum(k, nz - 1), np.minimum(j, ny - 1), np.minimum(i, nx - 1)
    j, i = np.indices(shp)
    return np.minimum(j, ny - 1), np.minimum(i, nx - 1)


@dataclass
class YeeSystem:
    """Matrices of Eq. (3) for one grid, plus the unknown index maps."""
    dim: int
    n: tuple
    d: tuple
    e_comps: tuple
    h_comps: tuple
    index: dict            # comp -> int array (storage shape), -1 where eliminated
    K: sp.csr_matrix       # N_e x N_h, from Ampere (E rows)
    L: sp.csr_matrix       # N_h x N_e, from Faraday (H rows); paper: L == K^T
    De: np.ndarray
    Dm: np.ndarray
    Dse: np.ndarray
    Dsm: np.ndarray
    eps_unknown: np.ndarray = field(default=None)
    mu_unknown: np.ndarray = field(default=None)

    @property
    def Ne(self):
        return self.K.shape[0]

    @property
    def Nh(self):
        return self.K.shape[1]

    def unknown_of(self, comp: int, idx) -> int:
        return int(self.index[comp][tuple(idx)])

    def to_storage(self, x: np.ndarray) -> dict:
        """Scatter an E-then-H state vector into per-component storage arrays."""
        out = {}
        off_e = 0
        for c in self.e_comps + self.h_comps:
            shp = storage_shape(self.dim, self.n)
            a = np.zeros(shp)
            m = self.index[c] >= 0
            base = 0 if c in self.e_comps else self.Ne
            a[m] = x[base + self.index[c][m]]
            out[c] = a
        return out

    def from_storage(self, arrays: dict) -> np.ndarray:
        x = np.zeros(self.Ne + self.Nh)
        for c in self.e_comps + self.h_comps:
            m = self.index[c] >= 0
            base = 0 if c in self.e_comps else self.Ne
            x[base + self.index[c][m]] = arrays[c][m]
        return x


def _number(dim, n, comps, eliminate_pec):
    """Assign consecutive unknown numbers, component-major, (k,j,i) lexicographic."""
    index, count = {}, 0
    for c in comps:
        m = exists_mask(dim, n, c)
        if eliminate_pec:
            m &= ~wall_pec_mask(dim, n, c)
        idx = -np.ones(m.shape, dtype=np.int64)
        idx[m] = count + np.arange(int(m.sum()))
        count += int(m.sum())
        index[c] = idx
    return index, count


def _operator(dim, n, d, row_index, col_index, terms, nrows, ncols):
    """Sparse operator sum_terms sign/d_axis * col[(idx + offset)], rows in row_index."""
    rows, cols, vals = [], [], []
    shp = storage_shape(dim, n)
    for rc, tl in terms.items():
        ridx = row_index[rc]
        sel = ridx >= 0
        pos = np.nonzero(sel)                     # tuple of index arrays (k,j,i) or (j,i)
        for (cc, off, sign, axis) in tl:
            # offset in storage order: off = (di, dj, dk)
            if dim == 3:
                q = (pos[0] + off[2], pos[1] + off[1], pos[2] + off[0])
            else:
                q = (pos[0] + off[1], pos[1] + off[0])
            ok = np.ones(pos[0].shape, bool)
            for ax_len, qa in zip(shp, q):
                ok &= (qa >= 0) & (qa < ax_len)
            qc = tuple(qa[ok] for qa in q)
            cidx = col_index[cc][qc]
            good = cidx >= 0                       # eliminated (PEC) partners drop out
            r = ridx[tuple(pa[ok] for pa in pos)][good]
            rows.append(r)
            cols.append(cidx[good])
            vals.append(np.full(r.shape, sign / d[axis]))
    rows = np.concatenate(rows)
    cols = np.concatenate(cols)
    vals = np.concatenate(vals)
    return sp.csr_matrix((vals, (rows, cols)), shape=(nrows, ncols))


def assemble(dim: int, n, d, eps0: float, mu0: float, eps_r=None, mu_r=None,
             sig_e=None, sig_m=None, eliminate_pec: bool = True) -> YeeSystem:
    """Assemble Eq. (3) on a uniform nx*ny(*nz) grid of cells with spacings d.

    n = (nx, ny, nz) (nz ignored in 2-D), d = (dx, dy, dz).  Per-cell material
    arrays have shape (nz, ny, nx) (3-D) or (ny, nx) (2-D); None = vacuum /
    lossless.  Returns the physical-units matrices of P:100-105:
    D_eps = eps per unknown, K entries +-1/d_axis.
    """
    n = tuple(int(v) for v in n)
    e_comps = E_COMPS_3D if dim == 3 else E_COMPS_2D
    h_comps = H_COMPS_3D if dim == 3 else H_COMPS_2D
    curl_h = _CURL_H_3D if dim == 3 else _CURL_H_2D
    mcurl_e = _MCURL_E_3D if dim == 3 else _MCURL_E_2D
    e_index, Ne = _number(dim, n, e_comps, eliminate_pec)
    h_index, Nh = _number(dim, n, h_comps, eliminate_pec)
    # E rows: D_eps dE/dt = curl H - J = -K H + B u  =>  K = -curl_H
    C = _operator(dim, n, d, e_index, h_index, curl_h, Ne, Nh)
    K = (-C).tocsr()
    # H rows: D_mu dH/dt = -curl E  (paper: = K^T E)
    L = _operator(dim, n, d, h_index, e_index, mcurl_e, Nh, Ne)
    cell_shape = (n[2], n[1], n[0]) if dim == 3 else (n[1], n[0])

    def per_unknown(cell_vals, index, comps, default):
        out = np.empty(sum(int((index[c] >= 0).sum()) for c in comps))
        if cell_vals is None:
            out[:] = default
            return out
        cell_vals = np.asarray(cell_vals, dtype=np.float64).reshape(cell_shape)
        own = owning_cell(dim, n)
        for c in comps:
            m = index[c] >= 0
            out[index[c][m]] = cell_vals[tuple(o[m] for o in own)]
        return out

    eps_u = per_unknown(eps_r, e_index, e_comps, 1.0) * eps0
    mu_u = per_unknown(mu_r, h_index, h_comps, 1.0) * mu0
    Dse = per_unknown(sig_e, e_index, e_comps, 0.0)
    Dsm = per_unknown(sig_m, h_index, h_comps, 0.0)
    index = dict(e_index)
    index.update(h_index)
    return YeeSystem(dim, n, tuple(float(v) for v in d), e_comps, h_comps, index,
                     K, L.tocsr(), eps_u.copy(), mu_u.copy(), Dse, Dsm, eps_u, mu_u)


def incidence(sys: YeeSystem) -> sp.csr_matrix:
    """K with the 1/d_axis factors removed (entries exactly +-1): K_inc.

    For a uniform cubic grid K = K_inc / delta, the form used by the
    F13 shared-input rule (reading R8)."""
    K = sys.K.tocoo()
    return sp.csr_matrix((np.sign(K.data), (K.row, K.col)), shape=K.shape)


def line_1d(nz: int, dz: float, eps: float, mu: float, eliminate_ends: bool = True):
    """1-D Yee line of Eqs. (2a)/(2b): E_k at k*dz, H_{k+1/2}.

    K follows the curl term of (2a): row E_k has +1/dz at H_{k+1/2} and -1/dz at
    H_{k-1/2}.  With ``eliminate_ends`` the PEC end nodes E_0, E_nz are removed
    (N_e = nz-1, N_h = nz); otherwise all nz+1 E nodes are kept (S:109's
    3-node / 2-H example uses nz = 2 without elimination).
    """
    k0, k1 = (1, nz) if eliminate_ends else (0, nz + 1)
    e_nodes = np.arange(k0, k1)
    Ne, Nh = len(e_nodes), nz
    K = sp.lil_matrix((Ne, Nh))
    for r, k in enumerate(e_nodes):
        if k < nz:
            K[r, k] += 1.0 / dz          # H_{k+1/2}
        if k > 0:
            K[r, k - 1] -= 1.0 / dz      # H_{k-1/2}
    return K.tocsr(), np.full(Ne, eps), np.full(Nh, mu)
