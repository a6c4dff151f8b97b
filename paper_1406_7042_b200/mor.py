"""Thin ctypes binding of the device-side offline reduction of libfdtd
(include/fdtd_mor.h): argument marshalling only, the shifted
solves (block Schur + batched CGS) and the multi-point block Arnoldi
 run in the CUDA library (csrc/mor.cu).  No CPU fallback: raises
when the library or an sm_100 GPU is missing.
"""
from __future__ import annotations

import ctypes as C

import numpy as np
import scipy.sparse as sp

from . import fdtd as _f

_f64p = C.POINTER(C.c_double)
_i64p = C.POINTER(C.c_int64)
_i32p = C.POINTER(C.c_int32)


class MorSystem(C.Structure):
    _fields_ = [("n_e", C.c_int64), ("n_h", C.c_int64), ("K_rowptr", _i64p), ("K_col", _i32p), ("K_val", _f64p),
                ("De", _f64p), ("Dm", _f64p), ("dt", C.c_double)]


class MorBasisRequest(C.Structure):
    _fields_ = [("n_points", C.c_int32), ("z_re", _f64p), ("z_im", _f64p), ("n_b", C.c_int32), ("B", _f64p),
                ("n_keep_e", C.c_int64), ("keep_e", _i64p), ("n_keep_h", C.c_int64), ("keep_h", _i64p),
                ("q", C.c_int32), ("max_iter", C.c_int32), ("solve_tol", C.c_double), ("solve_max_iter", C.c_int32),
                ("tol_krylov", C.c_double), ("tol_pool", C.c_double), ("window_bytes", C.c_double)]


MOR_SYMBOLS = ("mor_create", "mor_shifted_solve", "mor_krylov_basis", "mor_launch_count", "mor_destroy")
STATS = ("sweeps", "solve_columns", "cgs_iterations", "worst_residue", "t_solve", "t_orth", "krylov_vectors",
         "window_slid")
_ready = False


def _lib():
    global _ready
    lib = _f.load_library()
    if not _ready:
        lib.mor_create.argtypes = [C.POINTER(MorSystem), C.c_void_p, C.POINTER(C.c_void_p)]
        lib.mor_create.restype = C.c_int
        lib.mor_shifted_solve.argtypes = [C.c_void_p, C.c_double, C.c_double, C.c_int32, _f64p, _f64p, C.c_double,
                                          C.c_int32, _f64p, _f64p, _i32p, _f64p]
        lib.mor_shifted_solve.restype = C.c_int
        lib.mor_krylov_basis.argtypes = [C.c_void_p, C.POINTER(MorBasisRequest), _f64p, _f64p, _f64p, C.c_int32]
        lib.mor_krylov_basis.restype = C.c_int
        lib.mor_launch_count.argtypes = [C.c_void_p]
        lib.mor_launch_count.restype = C.c_int64
        lib.mor_destroy.argtypes = [C.c_void_p]
        lib.mor_destroy.restype = None
        _ready = True
    return lib


def _a(x, dtype=np.float64):
    return np.ascontiguousarray(np.asarray(x, dtype))


def _stream_ptr(stream):
    import torch
    st = stream if stream is not None else torch.cuda.current_stream()
    return C.c_void_p(st.cuda_stream)


class Mor:
    """One system to reduce (mor_t): diagonal masses De, Dm, curl K (n_e x n_h), dt."""

    def __init__(self, De, Dm, K, dt, stream=None):
        lib = _lib()
        self.lib = lib
        K = sp.csr_matrix(K)
        K.sort_indices()
        self.ne, self.nh = K.shape
        rp, ci, val = _a(K.indptr, np.int64), _a(K.indices, np.int32), _a(K.data)
        De, Dm = _a(De).ravel(), _a(Dm).ravel()
        if De.size != self.ne or Dm.size != self.nh:
            raise ValueError("De / Dm do not match K")
        s = MorSystem(self.ne, self.nh, rp.ctypes.data_as(_i64p), ci.ctypes.data_as(_i32p), val.ctypes.data_as(_f64p),
                      De.ctypes.data_as(_f64p), Dm.ctypes.data_as(_f64p), float(dt))
        h = C.c_void_p()
        _f._check(lib.mor_create(C.byref(s), _stream_ptr(stream), C.byref(h)))
        self.h = h

    def shifted_solve(self, z, b, tol=1e-4, max_iter=2000):
        """x = A(z)^-1 b for the columns of b [(n_e + n_h), nrhs]; returns (x, iters, resid)."""
        z = complex(z)
        b = np.asarray(b)
        if b.ndim == 1:
            b = b[:, None]
        N = self.ne + self.nh
        if b.shape[0] != N:
            raise ValueError("b must have n_e + n_h rows")
        m = b.shape[1]
        cplx = np.iscomplexobj(b) or z.imag != 0.0
        bre = _a(b.real.T)
        bim = _a(b.imag.T) if np.iscomplexobj(b) else None
        xre = np.zeros((m, N))
        xim = np.zeros((m, N)) if cplx else None
        iters = np.zeros(m, np.int32)
        resid = np.zeros(m)
        _f._check(self.lib.mor_shifted_solve(
            self.h, z.real, z.imag, m, bre.ctypes.data_as(_f64p), bim.ctypes.data_as(_f64p) if bim is not None else None,
            float(tol), int(max_iter), xre.ctypes.data_as(_f64p), xim.ctypes.data_as(_f64p) if cplx else None,
            iters.ctypes.data_as(_i32p), resid.ctypes.data_as(_f64p)))
        x = (xre + 1j * xim).T if cplx else xre.T
        return x, iters, resid

    def krylov_basis(self, B, keep_e, keep_h, q, points, max_iter=None, solve_tol=1e-4, solve_max_iter=2000,
                     tol_krylov=1e-10, tol_pool=1e-8, window_bytes=0.0):
        """(V1 [n_keep_e, q], V2 [n_keep_h, q], stats) -- same contract as
        prep.reduce.krylov_basis."""
        B = np.asarray(B, np.float64)
        if B.ndim == 1:
            B = B[:, None]
        Bt = _a(B.T)
        pts = [complex(z) for z in points]
        zre, zim = _a([z.real for z in pts]), _a([z.imag for z in pts])
        ke, kh = _a(keep_e, np.int64), _a(keep_h, np.int64)
        r = MorBasisRequest(len(pts), zre.ctypes.data_as(_f64p), zim.ctypes.data_as(_f64p), Bt.shape[0],
                            Bt.ctypes.data_as(_f64p), ke.size, ke.ctypes.data_as(_i64p), kh.size,
                            kh.ctypes.data_as(_i64p), int(q), int(max_iter or 0), float(solve_tol),
                            int(solve_max_iter), float(tol_krylov), float(tol_pool), float(window_bytes))
        V1 = np.zeros((q, ke.size))
        V2 = np.zeros((q, kh.size))
        st = np.zeros(len(STATS))
        _f._check(self.lib.mor_krylov_basis(self.h, C.byref(r), V1.ctypes.data_as(_f64p), V2.ctypes.data_as(_f64p),
                                            st.ctypes.data_as(_f64p), len(STATS)))
        return V1.T, V2.T, dict(zip(STATS, st.tolist()))          # (views: no 8 GB transposed copies at config 4's size)

    def launch_count(self):
        return int(self.lib.mor_launch_count(self.h))

    def close(self):
        if getattr(self, "h", None):
            self.lib.mor_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def krylov_basis(De, Dm, K, dt, B, keep_e, keep_h, q, points, **kw):
    """Drop-in device replacement of prep.reduce.krylov_basis (returns V1, V2)."""
    m = Mor(De, Dm, K, dt)
    try:
        V1, V2, st = m.krylov_basis(B, keep_e, keep_h, q, points, **kw)
    finally:
        m.close()
    krylov_basis.last_stats = st
    return V1, V2
