"""Thin ctypes binding of the whole-domain reduced-model calls of libfdtd
(include/fdtd_rom.h): argument marshalling only, every step runs in the CUDA
library (csrc/rom.cu).  No CPU fallback: raises when the library or an sm_100
GPU is missing.

``model``: dict with K [q_e][q_h], g_e [q_e], g_h [q_h], B_e [q_e][n_in],
optional L_e [n_out_e][q_e], L_h [n_out_h][q_h]; ``amp``
[n_in][batch], ``wave`` [n_wave][batch].
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import fdtd as _f

_f64p = C.POINTER(C.c_double)


class RomModel(C.Structure):
    _fields_ = [("q_e", C.c_int32), ("q_h", C.c_int32), ("n_in", C.c_int32), ("n_out_e", C.c_int32),
                ("n_out_h", C.c_int32), ("K", _f64p), ("g_e", _f64p), ("g_h", _f64p), ("B_e", _f64p),
                ("L_e", _f64p), ("L_h", _f64p)]


class RomExcitation(C.Structure):
    _fields_ = [("batch", C.c_int32), ("amp", _f64p), ("n_wave", C.c_int64), ("wave", _f64p)]


ROM_SYMBOLS = ("rom_create", "rom_step", "rom_probe", "rom_get_state", "rom_set_state", "rom_sync", "rom_info",
               "rom_dmma_peak_tflops", "rom_destroy")
_ready = False


def _lib():
    global _ready
    lib = _f.load_library()
    if not _ready:
        lib.rom_create.argtypes = [C.POINTER(RomModel), C.POINTER(RomExcitation), C.c_void_p, C.c_int32,
                                   C.POINTER(C.c_void_p)]
        lib.rom_create.restype = C.c_int
        lib.rom_step.argtypes = [C.c_void_p, C.c_int64]
        lib.rom_step.restype = C.c_int
        lib.rom_probe.argtypes = [C.c_void_p, _f64p, C.c_int64, C.POINTER(C.c_int64)]
        lib.rom_probe.restype = C.c_int
        lib.rom_get_state.argtypes = [C.c_void_p, C.c_int32, _f64p, C.c_int64]
        lib.rom_get_state.restype = C.c_int
        lib.rom_set_state.argtypes = [C.c_void_p, C.c_int32, _f64p, C.c_int64]
        lib.rom_set_state.restype = C.c_int
        lib.rom_sync.argtypes = [C.c_void_p]
        lib.rom_sync.restype = C.c_int
        lib.rom_info.argtypes = [C.c_void_p, C.POINTER(C.c_int64), C.c_int32]
        lib.rom_info.restype = C.c_int
        lib.rom_dmma_peak_tflops.argtypes = [C.c_void_p]
        lib.rom_dmma_peak_tflops.restype = C.c_double
        lib.rom_destroy.argtypes = [C.c_void_p]
        lib.rom_destroy.restype = None
        _ready = True
    return lib


def _a(x, shape=None):
    a = np.ascontiguousarray(np.asarray(x, np.float64))
    return a if shape is None else a.reshape(shape)


def _p(a):
    return a.ctypes.data_as(_f64p)


def _stream_ptr(stream):
    import torch
    st = stream if stream is not None else torch.cuda.current_stream()
    return C.c_void_p(st.cuda_stream)


def dmma_peak_tflops(stream=None):
    """Measured fp64 tensor-core (mma.sync m8n8k4) throughput of this GPU."""
    return float(_lib().rom_dmma_peak_tflops(_stream_ptr(stream)))


class Rom:
    """One batched reduced-model handle (rom_t)."""

    def __init__(self, model, amp, wave, stream=None, cols_per_cluster=0):
        lib = _lib()
        self.lib = lib
        K = _a(model["K"])
        qe, qh = K.shape
        ge = _a(np.broadcast_to(np.asarray(model["g_e"], np.float64), (qe,)))
        gh = _a(np.broadcast_to(np.asarray(model["g_h"], np.float64), (qh,)))
        Be = _a(model["B_e"]).reshape(qe, -1)
        n_in = Be.shape[1]
        Le = _a(model["L_e"]).reshape(-1, qe) if model.get("L_e") is not None else np.zeros((0, qe))
        Lh = _a(model["L_h"]).reshape(-1, qh) if model.get("L_h") is not None else np.zeros((0, qh))
        amp = _a(amp).reshape(n_in, -1)
        batch = amp.shape[1]
        wave = _a(wave).reshape(-1, batch)
        m = RomModel(qe, qh, n_in, Le.shape[0], Lh.shape[0], _p(K), _p(ge), _p(gh), _p(Be),
                     _p(Le) if Le.size else None, _p(Lh) if Lh.size else None)
        x = RomExcitation(batch, _p(amp), wave.shape[0], _p(wave))
        self._keep = (K, ge, gh, Be, Le, Lh, amp, wave)
        self.qe, self.qh, self.batch = qe, qh, batch
        self.n_out = Le.shape[0] + Lh.shape[0]
        self.steps_pending = 0
        h = C.c_void_p()
        _f._check(lib.rom_create(C.byref(m), C.byref(x), _stream_ptr(stream), int(cols_per_cluster), C.byref(h)))
        self.h = h

    def step(self, n):
        _f._check(self.lib.rom_step(self.h, int(n)))
        self.steps_pending += int(n)

    def sync(self):
        _f._check(self.lib.rom_sync(self.h))

    def probe(self):
        """Probe samples since the last call: [steps][n_out_e + n_out_h][batch]."""
        cap = max(1, self.steps_pending * max(self.n_out, 1) * self.batch)
        out = np.zeros(cap)
        wr = C.c_int64()
        _f._check(self.lib.rom_probe(self.h, _p(out), cap, C.byref(wr)))
        self.steps_pending = 0
        if self.n_out == 0:
            return np.zeros((0, 0, self.batch))
        return out[:wr.value].reshape(-1, self.n_out, self.batch)

    def get_state(self, which):
        n = 1 if which == 2 else self.batch * (self.qe if which == 0 else self.qh)
        out = np.zeros(n)
        _f._check(self.lib.rom_get_state(self.h, int(which), _p(out), n))
        return out if which == 2 else out.reshape(self.batch, -1)

    def set_state(self, which, values):
        v = _a(values).ravel()
        _f._check(self.lib.rom_set_state(self.h, int(which), _p(v), v.size))

    def info(self):
        v = (C.c_int64 * 7)()
        _f._check(self.lib.rom_info(self.h, v, 7))
        return dict(zip(("ctas_per_cluster", "cols_per_cluster", "clusters", "threads", "q_padded", "registers",
                         "launches"), [int(x) for x in v]))

    def close(self):
        if getattr(self, "h", None):
            self.lib.rom_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
