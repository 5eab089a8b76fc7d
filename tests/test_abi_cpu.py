"""CPU-side checks of the C-ABI library (-m "not gpu"): it builds, loads,
exports every symbol declared in include/hq.h, and hq_create validates its
inputs.  No compute call is made here; hq_solve on a
machine without a GPU must fail loudly with HQ_E_CUDA (no CPU fallback)."""
import ctypes
import os
import re

import numpy as np
import pytest

from paper_2603_03019_b200 import build as hqbuild

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def hq():
    hqbuild.build()
    from paper_2603_03019_b200 import hq as _hq

    return _hq


def declared_symbols():
    with open(os.path.join(ROOT, "include", "hq.h")) as f:
        src = f.read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(hq_[a-z_]+)\s*\(", src)))


def test_exports_every_declared_symbol(hq):
    lib = ctypes.CDLL(hq.LIB_PATH)
    syms = declared_symbols()
    assert set(syms) >= {"hq_create", "hq_solve", "hq_measures", "hq_destroy", "hq_error_string"}
    for s in syms:
        assert hasattr(lib, s), s
    assert set(hq.EXPORTED) == set(syms)


def test_library_is_sm100a(hq):
    import subprocess

    out = subprocess.run(["cuobjdump", "--list-elf", hq.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def _ok_instance():
    return dict(N=3, J=2, lam=[1.0, 0.5], mu=[1.0, 2.0, 0.5], pref=[[0, 1, 2], [2, 1, 0]])


def test_create_valid(hq):
    d = _ok_instance()
    h = hq.hq_create(d["N"], d["J"], d["lam"], d["mu"], d["pref"])
    assert h
    hq.hq_destroy(h)


@pytest.mark.parametrize("mut,needle", [
    (dict(N=0, J=1, lam=[1.0], mu=np.zeros(0), pref=np.zeros((1, 0), np.int32)), "N must be"),
    (dict(lam=[1.0, -0.5]), "lambda"),
    (dict(lam=[0.0, 0.0]), "sum of lambda"),
    (dict(lam=[np.nan, 1.0]), "lambda"),
    (dict(mu=[1.0, 0.0, 1.0]), "mu"),
    (dict(mu=[1.0, np.inf, 1.0]), "mu"),
    (dict(pref=[[0, 1, 3], [2, 1, 0]]), "out of range"),
    (dict(pref=[[0, 0, 1], [2, 1, 0]]), "duplicated"),
    (dict(pref=[[0, -1, 1], [2, 1, 0]]), "after -1"),
    (dict(pref=[[-1, -1, -1], [2, 1, 0]]), "empty"),
    (dict(pref=[[0, 1, -1], [0, 1, -1]]), "reducible"),
    (dict(lam=[1.0, 0.0], pref=[[0, 1, -1], [2, 1, 0]]), "reducible"),
])
def test_create_rejects(hq, mut, needle):
    d = _ok_instance()
    d.update(mut)
    N, J = d["N"], d["J"]
    with pytest.raises(hq.HQError) as ei:
        hq.hq_create(N, J, d["lam"], d["mu"], d["pref"])
    assert ei.value.status == hq.HQ_E_INVAL
    assert needle in str(ei.value)


def test_create_rejects_n32(hq):
    N = 32
    with pytest.raises(hq.HQError):
        hq.hq_create(N, 1, [1.0], np.ones(N), np.arange(N, dtype=np.int32)[None, :])


def test_solve_without_gpu_fails_loudly(hq):
    import torch

    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    d = _ok_instance()
    h = hq.hq_create(d["N"], d["J"], d["lam"], d["mu"], d["pref"])
    lib = hq.load()
    it = ctypes.c_int(0)
    res = ctypes.c_double(0.0)
    buf = ctypes.create_string_buffer(64)
    st = lib.hq_solve(ctypes.c_void_p(h), 1e-13, 10, ctypes.cast(buf, ctypes.c_void_p), None, ctypes.byref(it),
                      ctypes.byref(res))
    assert st == hq.HQ_E_CUDA
    assert "CUDA" in hq.hq_error_string(h) or "device" in hq.hq_error_string(h)
    hq.hq_destroy(h)


def test_set_buffer_validation(hq):
    """hq_set_buffer: C >= HQ_BUFFER_UNLIMITED; a waiting room needs full lists; the
    tail cannot be read before a solve (no compute call is made)."""
    d = _ok_instance()
    h = hq.hq_create(d["N"], d["J"], d["lam"], d["mu"], d["pref"])
    hq.hq_set_buffer(h, 5)
    hq.hq_set_buffer(h, hq.HQ_BUFFER_UNLIMITED)
    hq.hq_set_buffer(h, 0)
    with pytest.raises(hq.HQError, match="HQ_E_INVAL"):
        hq.hq_set_buffer(h, -2)
    with pytest.raises(hq.HQError, match="HQ_E_ORDER"):
        hq.hq_queue_tail(h, 3)
    hq.hq_destroy(h)
    t = hq.hq_create(3, 2, [1.0, 0.5], [1.0, 2.0, 0.5], [[0, 1, -1], [2, 1, 0]])
    with pytest.raises(hq.HQError, match="full preference lists"):
        hq.hq_set_buffer(t, 3)
    hq.hq_set_buffer(t, 0)
    hq.hq_destroy(t)


def test_batch_solve_validation(hq):
    """hq_batch_solve validates every instance before touching the device."""
    import ctypes

    lib = hq.load()
    lam = np.array([[1.0, 0.5], [0.0, 0.0]])
    mu = np.array([[1.0, 2.0, 0.5], [1.0, 1.0, 1.0]])
    pref = np.array([[[0, 1, 2], [2, 1, 0]]] * 2, dtype=np.int32)
    dp = ctypes.POINTER(ctypes.c_double)
    st = lib.hq_batch_solve(2, 3, 2, lam.ctypes.data_as(dp), mu.ctypes.data_as(dp),
                            pref.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)), 1e-13, 100, ctypes.c_void_p(16),
                            None, None, None, None, None, None, None)
    assert st == hq.HQ_E_INVAL
    assert "instance 1" in lib.hq_batch_error_string().decode()
    st = lib.hq_batch_solve(1, 13, 2, lam.ctypes.data_as(dp), mu.ctypes.data_as(dp),
                            pref.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)), 1e-13, 100, ctypes.c_void_p(16),
                            None, None, None, None, None, None, None)
    assert st == hq.HQ_E_INVAL


def test_batch_solve_without_gpu_fails_loudly(hq):
    import ctypes
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    lib = hq.load()
    lam = np.array([[1.0, 0.5]])
    mu = np.array([[1.0, 2.0, 0.5]])
    pref = np.array([[[0, 1, 2], [2, 1, 0]]], dtype=np.int32)
    dp = ctypes.POINTER(ctypes.c_double)
    st = lib.hq_batch_solve(1, 3, 2, lam.ctypes.data_as(dp), mu.ctypes.data_as(dp),
                            pref.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)), 1e-13, 100, ctypes.c_void_p(16),
                            None, None, None, None, None, None, None)
    assert st == hq.HQ_E_CUDA
