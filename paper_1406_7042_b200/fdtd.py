"""Thin ctypes binding of libfdtd (include/fdtd.h): argument marshalling only.

Every step of the hot path runs in the CUDA library; this module converts a
problem description into the C descriptors and raises on error
codes with ``fdtd_last_error()`` as the message.  PyTorch supplies the CUDA
stream and, optionally, its caching allocator.  There is no CPU fallback: if
the shared library is missing or the device is not an sm_100 GPU, this raises.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libfdtd.so")

FDTD_OK, FDTD_EINVAL, FDTD_ESTAMP, FDTD_ENOMEM, FDTD_ECUDA, FDTD_ENOTSUP, FDTD_EDIVERGED = range(7)
ERROR_NAMES = {1: "EINVAL", 2: "ESTAMP", 3: "ENOMEM", 4: "ECUDA", 5: "ENOTSUP", 6: "EDIVERGED"}


class FdtdError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"FDTD_{ERROR_NAMES.get(code, code)}: {msg}")
        self.code = code


class DivergenceError(FdtdError):
    pass


_i32p = C.POINTER(C.c_int32)
_i64p = C.POINTER(C.c_int64)
_f64p = C.POINTER(C.c_double)
_u8p = C.POINTER(C.c_uint8)
ALLOC_FN = C.CFUNCTYPE(C.c_void_p, C.c_size_t, C.c_void_p)
FREE_FN = C.CFUNCTYPE(None, C.c_void_p, C.c_void_p)


class Grid(C.Structure):
    _fields_ = [("dim", C.c_int32), ("nx", C.c_int32), ("ny", C.c_int32), ("nz", C.c_int32),
                ("dx", C.c_double), ("dy", C.c_double), ("dz", C.c_double),
                ("batch", C.c_int32), ("precision", C.c_int32), ("dt", C.c_double)]


class Materials(C.Structure):
    _fields_ = [("n_mat", C.c_int32), ("mat_id", _u8p), ("coef", _f64p), ("if_mask", _u8p),
                ("uniform_coef", C.c_double * 6), ("coef_a", _f64p)]


class Interface(C.Structure):
    _fields_ = [("n_rows", C.c_int64), ("unknown", _i64p), ("c", _f64p), ("rowptr", _i64p),
                ("col", _i64p), ("val", _f64p), ("block", _i32p), ("inst", _i32p), ("local", _i32p)]


class ReducedBlock(C.Structure):
    _fields_ = [("qe", C.c_int32), ("qh", C.c_int32), ("n_inst", C.c_int32), ("n_if", C.c_int32),
                ("K", _f64p), ("S_E", _f64p), ("g_e", _f64p), ("g_h", _f64p),
                ("g_e_scalar", C.c_double), ("g_h_scalar", C.c_double)]


class Sources(C.Structure):
    _fields_ = [("n_src", C.c_int64), ("unknown", _i64p), ("coef", _f64p), ("column", _i32p),
                ("n_cols", C.c_int64), ("n_wave", C.c_int64), ("wave", _f64p)]


class Probes(C.Structure):
    _fields_ = [("n_probe", C.c_int64), ("kind", _i32p), ("rowptr", _i64p), ("index", _i64p),
                ("weight", _f64p), ("block", _i32p), ("inst", _i32p)]


class Exec(C.Structure):
    _fields_ = [("stream", C.c_void_p), ("alloc", ALLOC_FN), ("free", FREE_FN), ("alloc_ctx", C.c_void_p),
                ("check_every", C.c_int32), ("graph_steps", C.c_int32), ("probe_capacity", C.c_int64),
                ("reduced_form", C.c_int32)]


_lib = None


def load_library(path: str = LIB_PATH):
    """Load libfdtd.so (fails loudly when it has not been built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise FileNotFoundError(f"{path} not found: build it with `python -c 'import __graft_entry__ as g; g.build()'`")
    lib = C.CDLL(path)
    lib.fdtd_create.argtypes = [C.POINTER(Grid), C.POINTER(Materials), C.POINTER(Interface),
                                C.POINTER(ReducedBlock), C.c_int32, C.POINTER(Sources),
                                C.POINTER(Probes), C.POINTER(Exec), C.POINTER(C.c_void_p)]
    lib.fdtd_create.restype = C.c_int
    lib.fdtd_step.argtypes = [C.c_void_p, C.c_int64]
    lib.fdtd_step.restype = C.c_int
    lib.fdtd_probe.argtypes = [C.c_void_p, _f64p, C.c_int64, _i64p]
    lib.fdtd_probe.restype = C.c_int
    lib.fdtd_get_state.argtypes = [C.c_void_p, C.c_int32, _f64p, C.c_int64]
    lib.fdtd_get_state.restype = C.c_int
    lib.fdtd_set_state.argtypes = [C.c_void_p, C.c_int32, _f64p, C.c_int64]
    lib.fdtd_set_state.restype = C.c_int
    lib.fdtd_sync.argtypes = [C.c_void_p]
    lib.fdtd_sync.restype = C.c_int
    lib.fdtd_launch_count.argtypes = [C.c_void_p]
    lib.fdtd_launch_count.restype = C.c_int64
    lib.fdtd_path.argtypes = [C.c_void_p]
    lib.fdtd_path.restype = C.c_int32
    lib.fdtd_profile.argtypes = [C.c_void_p, C.c_int32]
    lib.fdtd_profile.restype = C.c_int
    lib.fdtd_phase_times.argtypes = [C.c_void_p, _f64p, C.c_int32]
    lib.fdtd_phase_times.restype = C.c_int
    lib.fdtd_plane_device.argtypes = [C.c_void_p, C.c_int32, C.c_int32, C.c_void_p, C.c_int32]
    lib.fdtd_plane_device.restype = C.c_int
    lib.fdtd_destroy.argtypes = [C.c_void_p]
    lib.fdtd_destroy.restype = None
    lib.fdtd_last_error.argtypes = []
    lib.fdtd_last_error.restype = C.c_char_p
    lib.fdtd_version.argtypes = []
    lib.fdtd_version.restype = C.c_int
    _lib = lib
    return lib


EXPORTED_SYMBOLS = ("fdtd_create", "fdtd_step", "fdtd_probe", "fdtd_get_state", "fdtd_set_state",
                    "fdtd_sync", "fdtd_launch_count", "fdtd_path", "fdtd_profile", "fdtd_phase_times", "fdtd_plane_device",
                    "fdtd_destroy",
                    "fdtd_last_error", "fdtd_version")
PHASES = ("stencil", "reduced", "reduced_grid")


def _check(code):
    if code != FDTD_OK:
        msg = _lib.fdtd_last_error().decode()
        if code == FDTD_EDIVERGED:
            raise DivergenceError(code, msg)
        raise FdtdError(code, msg)


def _arr(a, dtype):
    return np.ascontiguousarray(np.asarray(a, dtype=dtype))


def _ptr(a, ctype):
    return a.ctypes.data_as(C.POINTER(ctype)) if a is not None and a.size else None


def storage_shape(dim, n):
    nx, ny, nz = n
    return (nz + 1, ny + 1, nx + 1) if dim == 3 else (ny + 1, nx + 1)


class Sim:
    """One simulation handle (fdtd_t).  ``problem``: DESIGN.md §6 dict;
    ``precision`` 32/64 overrides problem['precision']."""

    def __init__(self, problem, precision=None, stream=None, use_torch_allocator=True,
                 check_every=100, graph_steps=32, probe_capacity=0, reduced_form="auto"):
        lib = load_library()
        self.lib = lib
        self.problem = problem
        dim = int(problem["dim"])
        n = tuple(int(v) for v in problem["n"])
        if len(n) == 2:
            n = n + (1,)
        self.dim, self.n = dim, n
        self.B = int(problem.get("batch", 1))
        self.S = int(np.prod(storage_shape(dim, n)))
        prec = int(precision or problem.get("precision", 64))
        d = float(problem["delta"])
        keep = []                               # arrays alive for the call
        g = Grid(dim, n[0], n[1], n[2] if dim == 3 else 1, d, d, d, self.B, prec, float(problem["dt"]))
        mat = Materials()
        if problem.get("mat_id") is not None:
            mid = _arr(problem["mat_id"], np.uint8).ravel()
            coef = _arr(problem["mat_coef"], np.float64)
            ifm = _arr(problem["mat_ifmask"], np.uint8)
            keep += [mid, coef, ifm]
            mat.n_mat = coef.shape[0]
            mat.mat_id, mat.coef, mat.if_mask = _ptr(mid, C.c_uint8), _ptr(coef, C.c_double), _ptr(ifm, C.c_uint8)
            if problem.get("mat_ca") is not None:        # lossy media: ca / da per material (fdtd.h coef_a)
                ca = _arr(problem["mat_ca"], np.float64)
                assert ca.shape == coef.shape
                keep.append(ca)
                mat.coef_a = _ptr(ca, C.c_double)
        else:
            mat.n_mat = 0
            uc = _arr(problem["uniform_coef"], np.float64)
            for c in range(6):
                mat.uniform_coef[c] = float(uc[c])
        itf = Interface()
        it = problem.get("interface")
        if it is not None and len(it["unknown"]):
            a = {k: _arr(it[k], np.int64) for k in ("unknown", "rowptr", "col")}
            a.update({k: _arr(it[k], np.float64) for k in ("c", "val")})
            a.update({k: _arr(it[k], np.int32) for k in ("block", "inst", "local")})
            keep.append(a)
            itf.n_rows = len(a["unknown"])
            itf.unknown, itf.rowptr, itf.col = (_ptr(a[k], C.c_int64) for k in ("unknown", "rowptr", "col"))
            itf.c, itf.val = _ptr(a["c"], C.c_double), _ptr(a["val"], C.c_double)
            itf.block, itf.inst, itf.local = (_ptr(a[k], C.c_int32) for k in ("block", "inst", "local"))
        blocks = problem.get("blocks") or []
        nb = len(blocks)
        BA = (ReducedBlock * max(nb, 1))()
        self.block_shapes = []
        for i, b in enumerate(blocks):
            qe = int(b.get("qe", b.get("q")))
            qh = int(b.get("qh", b.get("q")))
            K = _arr(b["K"], np.float64).reshape(qe, qh)
            SE = _arr(b["S_E"], np.float64).reshape(-1, qh)
            keep += [K, SE]
            BA[i].qe, BA[i].qh, BA[i].n_inst, BA[i].n_if = qe, qh, int(b["n_inst"]), SE.shape[0]
            BA[i].K, BA[i].S_E = _ptr(K, C.c_double), _ptr(SE, C.c_double)
            for side, q in (("g_e", qe), ("g_h", qh)):
                v = np.asarray(b[side], np.float64)
                if v.ndim == 0:
                    setattr(BA[i], side + "_scalar", float(v))
                else:
                    v = _arr(v, np.float64)
                    keep.append(v)
                    setattr(BA[i], side, _ptr(v, C.c_double))
            self.block_shapes.append((qe, qh, int(b["n_inst"])))
        src = Sources()
        s = problem.get("sources")
        if s is not None and len(s["unknown"]):
            u = _arr(s["unknown"], np.int64)
            cf = _arr(s["coef"], np.float64)
            wv = _arr(s["wave"], np.float64)
            if wv.ndim == 2:
                wv = wv[:, :, None]
            if wv.shape[2] != self.B:
                wv = np.ascontiguousarray(np.broadcast_to(wv, (wv.shape[0], wv.shape[1], self.B)))
            keep += [u, cf, wv]
            src.n_src, src.unknown, src.coef = len(u), _ptr(u, C.c_int64), _ptr(cf, C.c_double)
            if s.get("column") is not None:
                col = _arr(s["column"], np.int32)
                keep.append(col)
                src.column = _ptr(col, C.c_int32)
            src.n_cols = wv.shape[1]
            src.n_wave, src.wave = wv.shape[0], _ptr(wv, C.c_double)
        prb = Probes()
        plist = problem.get("probes") or []
        self.n_probe = len(plist)
        if plist:
            kind, rp, idx, w, blk, inst = [], [0], [], [], [], []
            for p in plist:
                k = int(p["kind"])
                kind.append(k)
                if k == 0:
                    idx += [int(v) for v in p["unknowns"]]
                    w += [float(v) for v in p["weights"]]
                    blk.append(0); inst.append(0)
                else:
                    vr = np.asarray(p["vrow"], np.float64)
                    nzi = np.nonzero(vr)[0]
                    idx += [int(v) for v in nzi]
                    w += [float(vr[v]) for v in nzi]
                    blk.append(int(p["block"])); inst.append(int(p["inst"]))
                rp.append(len(idx))
            arrs = dict(kind=_arr(kind, np.int32), rowptr=_arr(rp, np.int64), index=_arr(idx, np.int64),
                        weight=_arr(w, np.float64), block=_arr(blk, np.int32), inst=_arr(inst, np.int32))
            keep.append(arrs)
            prb.n_probe = len(kind)
            prb.kind, prb.block, prb.inst = (_ptr(arrs[k], C.c_int32) for k in ("kind", "block", "inst"))
            prb.rowptr, prb.index = _ptr(arrs["rowptr"], C.c_int64), _ptr(arrs["index"], C.c_int64)
            prb.weight = _ptr(arrs["weight"], C.c_double)
        ex = Exec()
        ex.check_every, ex.graph_steps, ex.probe_capacity = int(check_every), int(graph_steps), int(probe_capacity)
        ex.reduced_form = {"auto": 0, "fused": 1, "leapfrog": 2}[reduced_form]
        self._torch_cbs = None
        try:
            import torch
            if torch.cuda.is_available():
                st = stream if stream is not None else torch.cuda.current_stream()
                ex.stream = C.c_void_p(st.cuda_stream)
                self._stream = st
                if use_torch_allocator:
                    dev = torch.cuda.current_device()

                    def _alloc(nbytes, ctx):
                        return torch.cuda.caching_allocator_alloc(int(nbytes), dev, st)

                    def _free(ptr, ctx):
                        if torch is not None and getattr(torch, "cuda", None) is not None:   # interpreter teardown
                            torch.cuda.caching_allocator_delete(ptr)
                    self._torch_cbs = (ALLOC_FN(_alloc), FREE_FN(_free))
                    ex.alloc, ex.free = self._torch_cbs
        except ImportError:
            pass
        h = C.c_void_p()
        _check(lib.fdtd_create(C.byref(g), C.byref(mat), C.byref(itf), BA if nb else None, nb,
                               C.byref(src), C.byref(prb), C.byref(ex), C.byref(h)))
        self.h = h
        self.steps_done = 0

    # -- API mirroring the C calls -------------------------------------------------
    def step(self, n):
        _check(self.lib.fdtd_step(self.h, int(n)))
        self.steps_done += int(n)

    def sync(self):
        _check(self.lib.fdtd_sync(self.h))

    def probe(self):
        """All probe samples since the last call: array [steps][n_probe][B] (fp64)."""
        cap = max(1, self.steps_done * max(self.n_probe, 1) * self.B)
        out = np.zeros(cap)
        wr = C.c_int64()
        _check(self.lib.fdtd_probe(self.h, _ptr(out, C.c_double), cap, C.byref(wr)))
        k = wr.value
        return out[:k].reshape(-1, self.n_probe, self.B) if self.n_probe else out[:0]

    def get_state(self, which):
        if which <= 5:
            n = self.B * self.S
        elif which in (6, 7):
            n = sum((qe if which == 6 else qh) * ni * self.B for qe, qh, ni in self.block_shapes)
        else:
            n = 1
        out = np.zeros(n)
        _check(self.lib.fdtd_get_state(self.h, int(which), _ptr(out, C.c_double), n))
        return out.reshape(self.B, self.S) if which <= 5 else out

    def set_state(self, which, values):
        v = _arr(values, np.float64).ravel()
        _check(self.lib.fdtd_set_state(self.h, int(which), _ptr(v, C.c_double), v.size))

    def profile(self, enable=True):
        _check(self.lib.fdtd_profile(self.h, int(bool(enable))))

    def phase_times(self):
        """{phase: accumulated device ms}, plus 'steps' profiled."""
        out = np.zeros(len(PHASES) + 1)
        _check(self.lib.fdtd_phase_times(self.h, _ptr(out, C.c_double), len(out)))
        d = dict(zip(PHASES, out[:len(PHASES)].tolist()))
        d["steps"] = int(out[-1])
        return d

    def plane_device(self, which, k, dev_ptr, to_state):
        """z-plane k of coarse component ``which`` <-> a device buffer (asynchronous)."""
        _check(self.lib.fdtd_plane_device(self.h, int(which), int(k), C.c_void_p(int(dev_ptr)), 1 if to_state else 0))

    def launch_count(self):
        return int(self.lib.fdtd_launch_count(self.h))

    PATH_BITS = {1: "persistent2d", 2: "tma3d", 4: "fused_gemm", 8: "leapfrog", 16: "tile3d", 32: "tc_gemm",
                 64: "fused_rows"}

    def path(self):
        """Kernel paths taken by step() (fdtd_path bit mask) as a list of names."""
        m = int(self.lib.fdtd_path(self.h))
        return [nm for bit, nm in self.PATH_BITS.items() if m & bit]

    def close(self):
        if getattr(self, "h", None):
            self.lib.fdtd_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
