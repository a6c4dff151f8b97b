"""Host-side checks of the C ABI (no GPU needed): the library loads, exports
every symbol include/fdtd.h declares, and validates its arguments."""
import ctypes as C
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _lib():
    from paper_1406_7042_b200 import build, fdtd
    build.build()
    return fdtd, fdtd.load_library()


def test_header_symbols_exported():
    fdtd, lib = _lib()
    hdr = open(os.path.join(ROOT, "include", "fdtd.h")).read()
    declared = set(re.findall(r"\b(fdtd_[a-z_]+)\s*\(", hdr))
    assert declared == set(fdtd.EXPORTED_SYMBOLS)
    for name in declared:
        assert hasattr(lib, name)
    assert lib.fdtd_version() == 100


def _grid(fdtd, **kw):
    g = dict(dim=3, nx=4, ny=4, nz=4, dx=1e-3, dy=1e-3, dz=1e-3, batch=1, precision=32, dt=1e-12)
    g.update(kw)
    return fdtd.Grid(**g)


@pytest.mark.parametrize("kw,code", [
    (dict(dim=4), 1), (dict(nx=0), 1), (dict(dx=-1.0), 1), (dict(precision=16), 1),
    (dict(batch=0), 1), (dict(dim=2, nz=3), 1), (dict(dy=2e-3), 5)])
def test_create_rejects_invalid_grid(kw, code):
    fdtd, lib = _lib()
    g = _grid(fdtd, **kw)
    h = C.c_void_p()
    rc = lib.fdtd_create(C.byref(g), None, None, None, 0, None, None, None, C.byref(h))
    assert rc == code
    assert lib.fdtd_last_error().decode()
    assert not h.value


def test_create_without_gpu_fails_loudly():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    fdtd, lib = _lib()
    g = _grid(fdtd)
    h = C.c_void_p()
    rc = lib.fdtd_create(C.byref(g), None, None, None, 0, None, None, None, C.byref(h))
    assert rc in (4, 5)      # FDTD_ECUDA / FDTD_ENOTSUP: no silent CPU fallback
    with pytest.raises(fdtd.FdtdError):
        fdtd.Sim(dict(dim=3, n=(4, 4, 4), delta=1e-3, dt=1e-12, batch=1, precision=32,
                      uniform_coef=np.ones(6)))


def test_null_handle_calls():
    fdtd, lib = _lib()
    assert lib.fdtd_step(None, 1) == 1
    assert lib.fdtd_sync(None) == 1
    assert lib.fdtd_launch_count(None) == 0


def test_rom_header_symbols_exported_and_arguments_checked():
    # include/fdtd_rom.h: every declared symbol is exported; rom_create validates
    # its arguments before touching the device; no CPU fallback
    fdtd, lib = _lib()
    from paper_1406_7042_b200 import rom
    rom._lib()
    hdr = open(os.path.join(ROOT, "include", "fdtd_rom.h")).read()
    declared = set(re.findall(r"\b(rom_[a-z_]+)\s*\(", hdr))
    assert declared == set(rom.ROM_SYMBOLS)
    for name in declared:
        assert hasattr(lib, name)
    K = np.eye(4)
    g = np.ones(4)
    f64 = C.POINTER(C.c_double)
    p = lambda a: a.ctypes.data_as(f64)
    h = C.c_void_p()
    x = rom.RomExcitation(1, None, 0, None)
    for q_e, batch, code in ((0, 1, 1), (300, 1, 1), (4, 0, 1)):
        m = rom.RomModel(q_e, 4, 0, 0, 0, p(K), p(g), p(g), None, None, None)
        x.batch = batch
        assert lib.rom_create(C.byref(m), C.byref(x), None, 0, C.byref(h)) == code
        assert lib.fdtd_last_error().decode() and not h.value
    m = rom.RomModel(4, 4, 0, 0, 0, p(K), p(g), p(g), None, None, None)
    x.batch = 1
    assert lib.rom_create(C.byref(m), C.byref(x), None, 7, C.byref(h)) == 1     # cols_per_cluster
    assert lib.rom_step(None, 1) == 1 and lib.rom_sync(None) == 1
    import torch
    if not torch.cuda.is_available():
        assert lib.rom_create(C.byref(m), C.byref(x), None, 0, C.byref(h)) in (4, 5)


def test_mor_header_symbols_exported_and_arguments_checked():
    # include/fdtd_mor.h: every declared symbol is exported; mor_create validates
    # its arguments before touching the device; no CPU fallback
    fdtd, lib = _lib()
    from paper_1406_7042_b200 import mor
    mor._lib()
    hdr = open(os.path.join(ROOT, "include", "fdtd_mor.h")).read()
    declared = set(re.findall(r"\b(mor_[a-z_]+)\s*\(", hdr))
    assert declared == set(mor.MOR_SYMBOLS)
    for name in declared:
        assert hasattr(lib, name)
    f64, i64, i32 = C.POINTER(C.c_double), C.POINTER(C.c_int64), C.POINTER(C.c_int32)
    rp = np.array([0, 1, 2], np.int64)
    ci = np.array([0, 1], np.int32)
    val = np.array([1.0, -1.0])
    De = np.array([1.0, 2.0])
    Dm = np.array([1.0, 1.0])

    def system(**kw):
        a = dict(n_e=2, n_h=2, rp=rp, ci=ci, val=val, De=De, Dm=Dm, dt=1e-12)
        a.update(kw)
        return mor.MorSystem(a["n_e"], a["n_h"], a["rp"].ctypes.data_as(i64), a["ci"].ctypes.data_as(i32),
                             a["val"].ctypes.data_as(f64), a["De"].ctypes.data_as(f64), a["Dm"].ctypes.data_as(f64),
                             a["dt"])
    h = C.c_void_p()
    for kw, code in ((dict(n_e=0), 1), (dict(dt=0.0), 1), (dict(De=np.array([1.0, -2.0])), 1),
                     (dict(ci=np.array([0, 5], np.int32)), 2), (dict(rp=np.array([0, 2, 1], np.int64)), 1)):
        s = system(**kw)
        assert lib.mor_create(C.byref(s), None, C.byref(h)) == code
        assert lib.fdtd_last_error().decode() and not h.value
    assert lib.mor_shifted_solve(None, 1.1, 0.0, 1, None, None, 1e-4, 10, None, None, None, None) == 1
    assert lib.mor_krylov_basis(None, None, None, None, None, 0) == 1
    assert lib.mor_launch_count(None) == 0
    import torch
    if not torch.cuda.is_available():
        s = system()
        assert lib.mor_create(C.byref(s), None, C.byref(h)) in (4, 5)
