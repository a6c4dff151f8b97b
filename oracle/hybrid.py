"""Coarse grid + refined boxes assembled as ONE system of form (3).

Not in the paper: the paper always reduces the whole FDTD system
and SPEC excludes subgridding (S:9).  The north star replaces the finely
meshed region of a coarse grid by a reduced model, which needs the unreduced
"coarse + fine" system to project.  Reading R4 (survey §8(c) O4):

1. Two independent finite-integration grids in symmetric volume form:
   D_eps,i = eps * (dual volume of edge i clipped to the grid's own domain),
   D_mu,j  = mu * A_j * Ltilde_j,  K_ij = +-L_i Ltilde_j  with Ltilde_j the
   dual edge of face j clipped to the domain.  On a uniform grid this is the
   paper's form times delta^dim.
2. The coarse domain is every coarse cell outside the boxes; each box is a
   fine grid (ratio r per axis) filling the box.
3. Constraint x_full = T x: fine tangential E on the box surface = P (coarse
   surface E) (copy where points coincide, linear interpolation across hanging
   positions, piecewise constant along the edge direction); fine normal H on
   the surface = the coarse face value.
4. K_h = T_E^T K T_H,  D_mu,h = T_H^T D_mu T_H (diagonal),
   D_eps,h = rowsum-lump(T_E^T D_eps T_E).

The result has the structure of (3), so conditions (7)/(8) apply.
Everything is returned in the *scaled* units used by the problem description
(volume form / delta^(dim-1)): a uniform coarse unknown has K = +-1,
D_eps = eps*delta, D_mu = mu*delta, so G_E = dt/D_eps = dt/(eps delta) = cb.

This module is written for clarity on small grids (loops over surface
unknowns); it is the oracle's independent check of the preprocessing library.
2-D (Ez/Hx/Hy) and 3-D grids are both supported.
"""
from __future__ import annotations

from dataclasses import dataclass, field
from fractions import Fraction

import numpy as np
import scipy.sparse as sp


@dataclass
class Box:
    """A refined region: coarse cells lo[a] <= c < hi[a] on each axis a, ratio r[a]."""
    lo: tuple
    hi: tuple
    r: tuple


@dataclass
class HybridSystem:
    dim: int
    n: tuple                    # coarse cells (nx, ny, nz)
    delta: float
    e_keys: list                # ('c', comp, (i,j,k)) or ('f', b, comp, (a,b,c))
    h_keys: list
    e_tag: np.ndarray           # 0 coarse regular, 1 coarse surface (interface), 2 fine
    h_tag: np.ndarray
    e_box: np.ndarray           # box id of fine unknowns, -1 for coarse
    h_box: np.ndarray
    K: sp.csr_matrix            # scaled units
    De: np.ndarray
    Dm: np.ndarray
    e_index: dict = field(default_factory=dict)
    h_index: dict = field(default_factory=dict)

    @property
    def Ne(self):
        return len(self.e_keys)

    @property
    def Nh(self):
        return len(self.h_keys)


# ----------------------------------------------------------------------------
# one FIT grid (uniform spacing h per axis) with a cell-domain mask
# ----------------------------------------------------------------------------

def _edges_2d(nx, ny):
    """2-D Ez 'edges' (z-directed, one per node) and H 'faces' (segments)."""
    E = [(2, (i, j, 0)) for j in range(ny + 1) for i in range(nx + 1)]
    H = [(3, (i, j, 0)) for j in range(ny) for i in range(nx + 1)] + \
        [(4, (i, j, 0)) for j in range(ny + 1) for i in range(nx)]
    return E, H


def _edges_3d(nx, ny, nz):
    E, H = [], []
    for k in range(nz + 1):
        for j in range(ny + 1):
            for i in range(nx + 1):
                if i < nx:
                    E.append((0, (i, j, k)))
                if j < ny:
                    E.append((1, (i, j, k)))
                if k < nz:
                    E.append((2, (i, j, k)))
                if j < ny and k < nz:
                    H.append((3, (i, j, k)))
                if i < nx and k < nz:
                    H.append((4, (i, j, k)))
                if i < nx and j < ny:
                    H.append((5, (i, j, k)))
    return E, H


def _edge_cells(dim, comp, idx):
    """Cells around an E unknown (4 around an edge; 4 around a 2-D node)."""
    i, j, k = idx
    if dim == 2:
        return [(i - 1, j - 1, 0), (i, j - 1, 0), (i - 1, j, 0), (i, j, 0)]
    if comp == 0:
        return [(i, j - 1, k - 1), (i, j, k - 1), (i, j - 1, k), (i, j, k)]
    if comp == 1:
        return [(i - 1, j, k - 1), (i, j, k - 1), (i - 1, j, k), (i, j, k)]
    return [(i - 1, j - 1, k), (i, j - 1, k), (i - 1, j, k), (i, j, k)]


def _face_cells(dim, comp, idx):
    """The two cells sharing an H face; the normal axis."""
    i, j, k = idx
    if comp == 3:
        return [(i - 1, j, k), (i, j, k)], 0
    if comp == 4:
        return [(i, j - 1, k), (i, j, k)], 1
    return [(i, j, k - 1), (i, j, k)], 2


def _face_edges(dim, comp, idx):
    """E unknowns on the boundary of H face (comp, idx) with the K sign of the
    paper form (K = -curl_H, see oracle.yee): list of (E comp, idx, sign)."""
    i, j, k = idx
    if dim == 2:
        if comp == 3:   # Hx(i, j+1/2): Ez(i,j) +, Ez(i,j+1) -
            return [(2, (i, j, 0), +1), (2, (i, j + 1, 0), -1)]
        return [(2, (i, j, 0), -1), (2, (i + 1, j, 0), +1)]   # Hy(i+1/2, j)
    # 3-D: K = -curl_H; entries read off oracle.yee._CURL_H_3D with sign flipped.
    if comp == 3:   # Hx[k][j][i] appears in Ey(+, k) / Ey(-, k+1) and Ez(-, j)/(+, j+1)
        return [(1, (i, j, k), -1), (1, (i, j, k + 1), +1),
                (2, (i, j, k), +1), (2, (i, j + 1, k), -1)]
    if comp == 4:   # Hy[k][j][i]
        return [(2, (i, j, k), -1), (2, (i + 1, j, k), +1),
                (0, (i, j, k), +1), (0, (i, j, k + 1), -1)]
    return [(0, (i, j, k), -1), (0, (i, j + 1, k), +1),
            (1, (i, j, k), +1), (1, (i + 1, j, k), -1)]


def _in_cells(c, n):
    return all(0 <= c[a] < n[a] for a in range(3))


class _Grid:
    """One uniform FIT grid: n cells, spacings h (3-tuple; 2-D uses h[2] = 1)."""

    def __init__(self, dim, n, h, domain, eps_of_cell, mu_of_cell, pec_e, pec_h):
        self.dim, self.n, self.h = dim, n, h
        self.domain = domain                 # callable(cell) -> bool
        self.E, self.H = (_edges_2d(n[0], n[1]) if dim == 2 else _edges_3d(*n))
        self.De, self.Dm, self.Lt = {}, {}, {}
        vol = h[0] * h[1] * h[2]
        for comp, idx in self.E:
            if pec_e(comp, idx):
                continue
            cells = [c for c in _edge_cells(dim, comp, idx) if _in_cells(c, n) and domain(c)]
            if not cells:
                continue
            own = tuple(min(idx[a], n[a] - 1) for a in range(3))
            # D_eps = eps(owning cell) * edge length * clipped dual-face area
            #       = eps * sum over in-domain adjacent cells of vol/4
            self.De[(comp, idx)] = eps_of_cell(own) * len(cells) * vol / 4.0
        for comp, idx in self.H:
            if pec_h(comp, idx):
                continue
            cells, ax = _face_cells(dim, comp, idx)
            cells = [c for c in cells if _in_cells(c, n) and domain(c)]
            if not cells:
                continue
            Lt = len(cells) * h[ax] / 2.0
            area = vol / h[ax]
            own = tuple(min(idx[a], n[a] - 1) for a in range(3))
            self.Lt[(comp, idx)] = Lt
            self.Dm[(comp, idx)] = mu_of_cell(own) * area * Lt
        # K entries: +-L_edge * Ltilde_face
        self.K = []
        for (comp, idx), Lt in self.Lt.items():
            for (ec, eidx, sgn) in _face_edges(dim, comp, idx):
                if (ec, eidx) in self.De:
                    L = h[ec] if dim == 3 else 1.0
                    self.K.append(((ec, eidx), (comp, idx), sgn * L * Lt))


# ----------------------------------------------------------------------------
# the hybrid assembly
# ----------------------------------------------------------------------------

def _axes(dim):
    return (0, 1) if dim == 2 else (0, 1, 2)


def _on_wall(dim, n, pos_c):
    """Which coarse-grid walls a coarse-unit position lies on (per axis)."""
    return [pos_c[a] == 0 or pos_c[a] == n[a] for a in _axes(dim)]


def _edge_axis(dim, comp):
    return 2 if dim == 2 else comp


def _pec_e_coarse(dim, n, pec_e_extra):
    def f(comp, idx):
        ax = _edge_axis(dim, comp)
        for a in _axes(dim):
            if a != ax and (idx[a] == 0 or idx[a] == n[a]):
                return True
        return pec_e_extra(('c', comp, idx)) if pec_e_extra else False
    return f


def _pec_h_coarse(dim, n):
    def f(comp, idx):
        ax = comp - 3
        return idx[ax] == 0 or idx[ax] == n[ax]
    return f


def assemble(dim, n, delta, eps_cell, boxes, eps0, mu0, mu_cell=None, pec_e_extra=None):
    """Assemble the hybrid of reading R4.

    n: coarse cells (nx, ny, nz) (nz = 1 in 2-D); eps_cell: relative
    permittivity per coarse cell, array [nz][ny][nx] ([ny][nx] in 2-D);
    boxes: list of Box.  pec_e_extra(key) -> bool marks interior PEC E
    unknowns (key = ('c', comp, idx) or ('f', b, comp, fine idx)).
    """
    n = tuple(int(v) for v in n) + ((1,) if len(n) == 2 else ())
    eps_cell = np.asarray(eps_cell, dtype=np.float64)
    if dim == 2:
        eps_cell = eps_cell.reshape(1, n[1], n[0])
    mu_cell = np.ones_like(eps_cell) if mu_cell is None else np.asarray(mu_cell).reshape(eps_cell.shape)

    def in_box(c, b):
        return all(b.lo[a] <= c[a] < b.hi[a] for a in _axes(dim))

    def coarse_domain(c):
        return not any(in_box(c, b) for b in boxes)

    hz = delta if dim == 3 else 1.0
    coarse = _Grid(dim, n, (delta, delta, hz), coarse_domain,
                   lambda c: eps0 * eps_cell[c[2], c[1], c[0]],
                   lambda c: mu0 * mu_cell[c[2], c[1], c[0]],
                   _pec_e_coarse(dim, n, pec_e_extra), _pec_h_coarse(dim, n))

    fines = []
    for bi, b in enumerate(boxes):
        r = tuple(b.r) + ((1,) if len(b.r) == 2 else ())
        nf = tuple((b.hi[a] - b.lo[a]) * r[a] for a in _axes(dim)) + ((1,) if dim == 2 else ())
        hf = tuple(delta / r[a] for a in _axes(dim)) + ((1.0,) if dim == 2 else ())

        def parent(c, b=b, r=r):
            return tuple(b.lo[a] + c[a] // r[a] for a in _axes(dim)) + ((0,) if dim == 2 else ())

        def pos_c(idx, b=b, r=r):     # coarse-unit position of a fine node index
            return tuple(Fraction(b.lo[a]) + Fraction(idx[a], r[a]) for a in _axes(dim))

        def pec_e(comp, idx, bi=bi, pos_c=pos_c):
            ax = _edge_axis(dim, comp)
            p = pos_c(idx)
            for a in _axes(dim):
                if a != ax and (p[a] == 0 or p[a] == n[a]):
                    return True
            return pec_e_extra(('f', bi, comp, idx)) if pec_e_extra else False

        def pec_h(comp, idx, pos_c=pos_c):
            ax = comp - 3
            p = pos_c(idx)
            return p[ax] == 0 or p[ax] == n[ax]

        g = _Grid(dim, nf, hf, lambda c: True,
                  lambda c, parent=parent: eps0 * eps_cell[parent(c)[2], parent(c)[1], parent(c)[0]],
                  lambda c, parent=parent: mu0 * mu_cell[parent(c)[2], parent(c)[1], parent(c)[0]],
                  pec_e, pec_h)
        fines.append((b, r, nf, g, pos_c))

    # ---- hybrid unknown lists -------------------------------------------------
    e_keys, e_tag, e_box = [], [], []
    h_keys, h_tag, h_box = [], [], []
    e_index, h_index = {}, {}

    def on_box_surface_e(comp, idx):
        """Coarse E unknown lies on some box surface (its dual is clipped)."""
        cells = [c for c in _edge_cells(dim, comp, idx) if _in_cells(c, n)]
        return any(not coarse_domain(c) for c in cells)

    for key in coarse.De:
        comp, idx = key
        e_index[('c', comp, idx)] = len(e_keys)
        e_keys.append(('c', comp, idx))
        e_tag.append(1 if on_box_surface_e(comp, idx) else 0)
        e_box.append(-1)
    for key in coarse.Dm:
        comp, idx = key
        cells, _ = _face_cells(dim, comp, idx)
        surf = any(_in_cells(c, n) and not coarse_domain(c) for c in cells)
        h_index[('c', comp, idx)] = len(h_keys)
        h_keys.append(('c', comp, idx))
        h_tag.append(1 if surf else 0)
        h_box.append(-1)

    # fine unknowns: classify surface (constrained) vs interior
    TE, TH = {}, {}
    for bi, (b, r, nf, g, pos_c) in enumerate(fines):
        for (comp, idx) in g.De:
            ax = _edge_axis(dim, comp)
            on_surf = any(a != ax and (idx[a] == 0 or idx[a] == nf[a]) for a in _axes(dim))
            key = ('f', bi, comp, idx)
            if not on_surf:
                e_index[key] = len(e_keys)
                e_keys.append(key)
                e_tag.append(2)
                e_box.append(bi)
                continue
            TE[key] = _interp_row(dim, n, comp, pos_c(idx), ax, coarse.De)
        for (comp, idx) in g.Dm:
            ax = comp - 3
            key = ('f', bi, comp, idx)
            if idx[ax] == 0 or idx[ax] == nf[ax]:
                # normal H on the surface -> copy of the coarse face containing it
                p = pos_c(idx)
                cidx = tuple(int(p[a]) if a == ax else int(np.floor(p[a])) for a in _axes(dim))
                cidx = cidx + ((0,) if dim == 2 else ())
                ck = (comp, cidx)
                TH[key] = ck if ck in coarse.Dm else None
                continue
            h_index[key] = len(h_keys)
            h_keys.append(key)
            h_tag.append(2)
            h_box.append(bi)

    Ne, Nh = len(e_keys), len(h_keys)
    De = np.zeros(Ne)
    Dm = np.zeros(Nh)
    rows, cols, vals = [], [], []

    for (comp, idx), v in coarse.De.items():
        De[e_index[('c', comp, idx)]] += v
    for (comp, idx), v in coarse.Dm.items():
        Dm[h_index[('c', comp, idx)]] += v
    for (ek, hk, v) in coarse.K:
        rows.append(e_index[('c',) + ek])
        cols.append(h_index[('c',) + hk])
        vals.append(v)

    def e_map(key):
        if key in e_index:
            return [(e_index[key], 1.0)]
        return [(e_index[('c',) + ck], w) for ck, w in TE[key]]

    def h_map(key):
        if key in h_index:
            return [(h_index[key], 1.0)]
        ck = TH[key]
        return [] if ck is None else [(h_index[('c',) + ck], 1.0)]

    for bi, (b, r, nf, g, pos_c) in enumerate(fines):
        for (comp, idx), v in g.De.items():
            key = ('f', bi, comp, idx)
            if key in e_index:
                De[e_index[key]] += v
            else:
                row = TE[key]
                s = sum(w for _, w in row)
                for ck, w in row:          # rowsum-lump of T_E^T D_eps T_E
                    De[e_index[('c',) + ck]] += w * v * s
        for (comp, idx), v in g.Dm.items():
            for hi_, w in h_map(('f', bi, comp, idx)):
                Dm[hi_] += w * w * v
        for (ek, hk, v) in g.K:
            for ei_, we in e_map(('f', bi) + ek):
                for hi_, wh in h_map(('f', bi) + hk):
                    rows.append(ei_)
                    cols.append(hi_)
                    vals.append(we * wh * v)

    scale = delta ** (dim - 1)       # volume form -> scaled units
    K = sp.csr_matrix((np.array(vals) / scale, (rows, cols)), shape=(Ne, Nh))
    K.sum_duplicates()
    K.eliminate_zeros()
    hs = HybridSystem(dim, n, delta, e_keys, h_keys, np.array(e_tag), np.array(h_tag),
                      np.array(e_box), np.array(h_box), K, De / scale, Dm / scale,
                      e_index, h_index)
    return hs


def _interp_row(dim, n, comp, p, ax, coarse_De):
    """P row of a fine surface E unknown at coarse-unit position p, directed
    along axis ax: piecewise constant along ax, multilinear across the other
    axes between the enclosing coarse lines (reading R4 step 3).  PEC coarse
    partners (absent from coarse_De) drop out."""
    axes = [a for a in _axes(dim) if a != ax]
    terms = [((), 1.0)]
    for a in axes:
        lo = int(np.floor(p[a]))
        t = p[a] - lo
        new = []
        for part, w in terms:
            if t == 0:
                new.append((part + ((a, lo),), w))
            else:
                new.append((part + ((a, lo),), w * float(1 - t)))
                new.append((part + ((a, lo + 1),), w * float(t)))
        terms = new
    out = []
    along = int(np.floor(p[ax])) if dim == 3 else 0
    for part, w in terms:
        idx = [0, 0, 0]
        for a, v in part:
            idx[a] = v
        if dim == 3:
            idx[ax] = along
        key = (comp, tuple(idx))
        if key in coarse_De and w != 0.0:
            out.append((key, w))
    return out


# ----------------------------------------------------------------------------
# helpers on the assembled hybrid
# ----------------------------------------------------------------------------

def blocks(hs: HybridSystem, box: int = None):
    """Partition into coarse (c) and fine (f) sets: returns index arrays and
    the sub-matrices K_cc, K_cf, K_fc, K_ff (survey O6)."""
    ec = np.nonzero(hs.e_tag < 2)[0]
    hc = np.nonzero(hs.h_tag < 2)[0]
    if box is None:
        ef = np.nonzero(hs.e_tag == 2)[0]
        hf = np.nonzero(hs.h_tag == 2)[0]
    else:
        ef = np.nonzero((hs.e_tag == 2) & (hs.e_box == box))[0]
        hf = np.nonzero((hs.h_tag == 2) & (hs.h_box == box))[0]
    K = hs.K
    return dict(ec=ec, hc=hc, ef=ef, hf=hf,
                Kcc=K[ec][:, hc], Kcf=K[ec][:, hf], Kfc=K[ef][:, hc], Kff=K[ef][:, hf])


def coarse_storage_index(key):
    """('c', comp, (i,j,k)) -> (comp, (i,j,k))."""
    return key[1], key[2]


def project(hs: HybridSystem, V1f, V2f):
    """Reading R6 / survey O6: V1 = blockdiag(I_c, V1_f), V2 = blockdiag(I_c, V2_f)
    applied to the hybrid, Eqs. (14)-(16):

      K~ = [[K_cc, S_E], [0, K~_rr]],  S_E = K_cf V2_f,  K~_rr = V1_f^T K_ff V2_f,
      D~_eps,f = V1_f^T D_eps,f V1_f,  D~_mu,f = V2_f^T D_mu,f V2_f.

    Returns dict with the blocks and index sets.  (K_fc = 0 is asserted: fine E
    never sees coarse H under reading R4.)"""
    b = blocks(hs)
    if b["Kfc"].nnz and abs(b["Kfc"]).max() != 0.0:
        raise AssertionError("K_fc must vanish (reading R4)")
    Kff = b["Kff"].toarray() if sp.issparse(b["Kff"]) else b["Kff"]
    out = dict(b)
    out["Kt_rr"] = V1f.T @ (Kff @ V2f)
    out["S_E"] = b["Kcf"] @ V2f                       # rows: coarse E (mostly zero)
    De_f = hs.De[b["ef"]]
    Dm_f = hs.Dm[b["hf"]]
    out["Dt_e"] = V1f.T @ (De_f[:, None] * V1f)
    out["Dt_m"] = V2f.T @ (Dm_f[:, None] * V2f)
    out["De_c"] = hs.De[b["ec"]]
    out["Dm_c"] = hs.Dm[b["hc"]]
    # interface rows = coarse E rows coupled to the fine H (surface E, tag 1)
    out["if_rows"] = np.nonzero(hs.e_tag[b["ec"]] == 1)[0]
    return out


def reduced_system(pr, Kt_rr=None, S_E_if=None):
    """The reduced hybrid as one system of form (3) (for brute-force checks):
    D_eps = blockdiag(D_eps,c, D~_eps,f), D_mu = blockdiag(D_mu,c, D~_mu,f),
    K = [[K_cc, S_E], [0, K~_rr]].  Optional perturbed blocks (after enforcement)
    replace K~_rr and the interface rows of S_E."""
    Kt = pr["Kt_rr"] if Kt_rr is None else Kt_rr
    SE = np.asarray(pr["S_E"].toarray() if sp.issparse(pr["S_E"]) else pr["S_E"]).copy()
    if S_E_if is not None:
        SE[pr["if_rows"]] = S_E_if
    K = sp.bmat([[pr["Kcc"], sp.csr_matrix(SE)],
                 [None, sp.csr_matrix(Kt)]]).tocsr()
    Ne_c, Nh_c = pr["Kcc"].shape
    De = sp.block_diag([sp.diags(pr["De_c"]), sp.csr_matrix(pr["Dt_e"])]).toarray()
    Dm = sp.block_diag([sp.diags(pr["Dm_c"]), sp.csr_matrix(pr["Dt_m"])]).toarray()
    return De, Dm, K


def sheet_pec(sheets, boxes, dim=3):
    """Predicate for oracle.hybrid.assemble(pec_e_extra=...): an E edge is PEC if
    it lies in a zero-thickness plate (closed rectangle in a plane z = pos).
    Plates are given in coarse units; fine edges are tested at their exact
    rational positions."""
    def test(key):
        if key[0] == "c":
            _, comp, (i, j, k) = key
            lo, r = (0, 0, 0), (1, 1, 1)
        else:
            _, b, comp, (i, j, k) = key
            lo, r = tuple(boxes[b]["lo"]), tuple(boxes[b]["r"])
        if comp not in (0, 1):
            return False
        x = Fraction(lo[0]) + Fraction(i, r[0])
        y = Fraction(lo[1]) + Fraction(j, r[1])
        z = Fraction(lo[2]) + Fraction(k, r[2])
        for sh in sheets:
            (x0, y0), (x1, y1) = sh["lo"], sh["hi"]
            if z != sh["pos"]:
                continue
            if comp == 0 and x0 <= x and x + Fraction(1, r[0]) <= x1 and y0 <= y <= y1:
                return True
            if comp == 1 and x0 <= x <= x1 and y0 <= y and y + Fraction(1, r[1]) <= y1:
                return True
        return False
    return test


def block_pec(boxes):
    """Predicate for solid PEC blocks given in a box's fine node indices (closed
    box): an E edge is PEC when both of its end nodes lie in the block."""
    def test(key):
        if key[0] != "f":
            return False
        _, b, comp, idx = key
        for blk in boxes[b].get("pec_fine") or []:
            lo, hi = blk["lo"], blk["hi"]
            ok = True
            for a in range(3):
                lo_a = idx[a]
                hi_a = idx[a] + (1 if a == comp else 0)
                if not (lo[a] <= lo_a and hi_a <= hi[a]):
                    ok = False
                    break
            if ok:
                return True
        return False
    return test
