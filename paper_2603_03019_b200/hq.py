"""Thin Python binding of the C-ABI in include/hq.h (argument marshalling only).

Every step of the solve runs in the CUDA kernels of libhq.so.  PyTorch is used
for device memory (the pi / measure tensors) and streams.  There is no CPU
fallback: if libhq.so is missing or CUDA is unavailable the calls raise.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("HQ_LIB") or os.path.join(_PKG, "libhq.so")   # HQ_LIB: A/B variant builds (tools/ab.py)

HQ_OK = 0
HQ_NOT_CONVERGED = 1
HQ_E_INVAL = -1
HQ_E_NOMEM = -2
HQ_E_CUDA = -3
HQ_E_NUMERIC = -4
HQ_E_ORDER = -5
HQ_STATS_LEN = 20
STATUS_NAMES = {0: "HQ_OK", 1: "HQ_NOT_CONVERGED", -1: "HQ_E_INVAL", -2: "HQ_E_NOMEM", -3: "HQ_E_CUDA",
                -4: "HQ_E_NUMERIC", -5: "HQ_E_ORDER"}
EXPORTED = ["hq_create", "hq_solve", "hq_measures", "hq_destroy", "hq_error_string", "hq_stats", "hq_version",
            "hq_debug_copy", "hq_set_buffer", "hq_queue_tail", "hq_batch_solve", "hq_batch_error_string", "hq_response_times"]
HQ_BUFFER_UNLIMITED = -1

_dptr = ctypes.POINTER(ctypes.c_double)
_lib = None
_dims = {}   # handle -> (N, J), recorded by hq_create for the binding's size checks


class HQError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"{STATUS_NAMES.get(status, status)}: {msg}")
        self.status = status


def load():
    """Load libhq.so (raises if it has not been built: no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} not found: build it with `python -m paper_2603_03019_b200.build` "
                          "(there is no CPU fallback)")
    lib = ctypes.CDLL(LIB_PATH)
    lib.hq_create.restype = ctypes.c_int
    lib.hq_create.argtypes = [ctypes.c_int, ctypes.c_int, _dptr, _dptr, ctypes.POINTER(ctypes.c_int32),
                              ctypes.POINTER(ctypes.c_void_p)]
    lib.hq_solve.restype = ctypes.c_int
    lib.hq_solve.argtypes = [ctypes.c_void_p, ctypes.c_double, ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p,
                             ctypes.POINTER(ctypes.c_int), _dptr]
    lib.hq_measures.restype = ctypes.c_int
    lib.hq_measures.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, _dptr,
                                ctypes.c_void_p]
    lib.hq_destroy.restype = None
    lib.hq_destroy.argtypes = [ctypes.c_void_p]
    lib.hq_error_string.restype = ctypes.c_char_p
    lib.hq_error_string.argtypes = [ctypes.c_void_p]
    lib.hq_stats.restype = ctypes.c_int
    lib.hq_stats.argtypes = [ctypes.c_void_p, _dptr]
    lib.hq_version.restype = ctypes.c_char_p
    lib.hq_version.argtypes = []
    lib.hq_debug_copy.restype = ctypes.c_int
    lib.hq_debug_copy.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p, ctypes.c_size_t]
    lib.hq_set_buffer.restype = ctypes.c_int
    lib.hq_set_buffer.argtypes = [ctypes.c_void_p, ctypes.c_int]
    lib.hq_queue_tail.restype = ctypes.c_int
    lib.hq_queue_tail.argtypes = [ctypes.c_void_p, _dptr, ctypes.c_int, _dptr]
    lib.hq_batch_solve.restype = ctypes.c_int
    lib.hq_batch_solve.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, _dptr, _dptr,
                                   ctypes.POINTER(ctypes.c_int32), ctypes.c_double, ctypes.c_int, ctypes.c_void_p,
                                   ctypes.c_void_p, ctypes.POINTER(ctypes.c_int), _dptr,
                                   ctypes.POINTER(ctypes.c_int), ctypes.c_void_p, ctypes.c_void_p, _dptr]
    lib.hq_response_times.restype = ctypes.c_int
    lib.hq_response_times.argtypes = [ctypes.c_void_p, ctypes.c_void_p, _dptr, ctypes.c_double, _dptr, _dptr,
                                      ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]
    lib.hq_batch_error_string.restype = ctypes.c_char_p
    lib.hq_batch_error_string.argtypes = []
    _lib = lib
    return lib


# ---------------------------------------------------------------- C-ABI names

def hq_create(N, J, lam, mu, pref):
    """hq_create(N, J, lambda[J], mu[N], pref[J][N]) -> handle (int)."""
    lib = load()
    lam = np.ascontiguousarray(lam, dtype=np.float64)
    mu = np.ascontiguousarray(mu, dtype=np.float64)
    pref = np.ascontiguousarray(pref, dtype=np.int32)
    if lam.shape != (J,) or mu.shape != (N,) or pref.shape != (J, N):
        raise HQError(HQ_E_INVAL, "dimension mismatch")
    h = ctypes.c_void_p()
    st = lib.hq_create(int(N), int(J), lam.ctypes.data_as(_dptr), mu.ctypes.data_as(_dptr),
                       pref.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)), ctypes.byref(h))
    if st != HQ_OK:
        raise HQError(st, lib.hq_error_string(None).decode())
    _dims[h.value] = (int(N), int(J))
    return h.value


def _check_size(t, n, what):
    if t.numel() != n:
        raise HQError(HQ_E_INVAL, f"{what} must have {n} elements, got {t.numel()}")


def _stream_ptr(stream):
    import torch

    if stream is None:
        stream = torch.cuda.current_stream()
    return ctypes.c_void_p(stream.cuda_stream)


def hq_solve(h, tol, max_iter, pi, stream=None):
    """hq_solve on a caller-owned float64 CUDA tensor pi[2^N].  Returns
    (status, iters, residual); raises on errors (status < 0)."""
    lib = load()
    _check_tensor(pi)
    if h in _dims:
        _check_size(pi, 1 << _dims[h][0], "pi")
    it = ctypes.c_int(0)
    res = ctypes.c_double(0.0)
    st = lib.hq_solve(ctypes.c_void_p(h), float(tol), int(max_iter), ctypes.c_void_p(pi.data_ptr()),
                      _stream_ptr(stream), ctypes.byref(it), ctypes.byref(res))
    if st < 0:
        raise HQError(st, lib.hq_error_string(ctypes.c_void_p(h)).decode())
    return st, it.value, res.value


def hq_measures(h, pi, workload, dispatch, stream=None):
    lib = load()
    for t in (pi, workload, dispatch):
        _check_tensor(t)
    if h in _dims:
        N, J = _dims[h]
        _check_size(pi, 1 << N, "pi")
        _check_size(workload, N, "workload")
        _check_size(dispatch, J * N, "dispatch")
    loss = ctypes.c_double(0.0)
    st = lib.hq_measures(ctypes.c_void_p(h), ctypes.c_void_p(pi.data_ptr()), ctypes.c_void_p(workload.data_ptr()),
                         ctypes.c_void_p(dispatch.data_ptr()), ctypes.byref(loss), _stream_ptr(stream))
    if st != HQ_OK:
        raise HQError(st, lib.hq_error_string(ctypes.c_void_p(h)).decode())
    return loss.value


def hq_set_buffer(h, C):
    """hq_set_buffer(h, C): waiting room of C calls (HQ_BUFFER_UNLIMITED: unlimited)."""
    lib = load()
    st = lib.hq_set_buffer(ctypes.c_void_p(h), int(C))
    if st != HQ_OK:
        raise HQError(st, lib.hq_error_string(ctypes.c_void_p(h)).decode())


def hq_queue_tail(h, n):
    """(P~{1..n} as a numpy array, sum_c P~{c}) of the last solve."""
    lib = load()
    tail = np.zeros(max(int(n), 1))
    mass = ctypes.c_double(0.0)
    st = lib.hq_queue_tail(ctypes.c_void_p(h), tail.ctypes.data_as(_dptr), int(n), ctypes.byref(mass))
    if st != HQ_OK:
        raise HQError(st, lib.hq_error_string(ctypes.c_void_p(h)).decode())
    return tail[: int(n)], mass.value


def hq_batch_solve(lam, mu, pref, tol=1e-13, max_iter=10000, pi=None, stream=None, measures=None):
    """hq_batch_solve on stacked instances: lam [B][J], mu [B][N], pref [B][J][N].
    Returns (pi [B][2^N] CUDA float64 tensor, iters[B], residual[B], status[B]); with a
    dict ``measures`` it is filled with workload [B][N], dispatch [B][J][N] (CUDA) and
    loss [B] (numpy).  Raises on HQ_E_INVAL / HQ_E_CUDA."""
    import torch

    lib = load()
    lam = np.ascontiguousarray(lam, dtype=np.float64)
    mu = np.ascontiguousarray(mu, dtype=np.float64)
    pref = np.ascontiguousarray(pref, dtype=np.int32)
    B, J = lam.shape
    N = mu.shape[1]
    if mu.shape != (B, N) or pref.shape != (B, J, N):
        raise HQError(HQ_E_INVAL, "dimension mismatch")
    if pi is None:
        pi = torch.empty((B, 1 << N), dtype=torch.float64, device="cuda")
    _check_tensor(pi)
    _check_size(pi, B << N, "pi")
    it = np.zeros(B, dtype=np.int32)
    res = np.zeros(B)
    sts = np.zeros(B, dtype=np.int32)
    w = d = None
    loss = np.zeros(B)
    if measures is not None:
        w = torch.empty((B, N), dtype=torch.float64, device=pi.device)
        d = torch.empty((B, J, N), dtype=torch.float64, device=pi.device)
        measures.update(workload=w, dispatch=d, loss=loss)
    st = lib.hq_batch_solve(B, N, J, lam.ctypes.data_as(_dptr), mu.ctypes.data_as(_dptr),
                            pref.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)), float(tol), int(max_iter),
                            ctypes.c_void_p(pi.data_ptr()), _stream_ptr(stream),
                            it.ctypes.data_as(ctypes.POINTER(ctypes.c_int)), res.ctypes.data_as(_dptr),
                            sts.ctypes.data_as(ctypes.POINTER(ctypes.c_int)),
                            ctypes.c_void_p(w.data_ptr()) if w is not None else None,
                            ctypes.c_void_p(d.data_ptr()) if d is not None else None,
                            loss.ctypes.data_as(_dptr) if measures is not None else None)
    if st in (HQ_E_INVAL, HQ_E_CUDA, HQ_E_NOMEM):
        raise HQError(st, lib.hq_batch_error_string().decode())
    return pi, it, res, sts


def hq_response_times(h, dispatch, tau, T_bar, mrt_j=None, f_j=None, stream=None):
    """(MRT, F(T_bar)); fills the optional CUDA tensors mrt_j[J], f_j[J]."""
    lib = load()
    _check_tensor(dispatch)
    tau = np.ascontiguousarray(tau, dtype=np.float64)
    if h in _dims:
        N, J = _dims[h]
        _check_size(dispatch, J * N, "dispatch")
        if tau.shape != (J, N):
            raise HQError(HQ_E_INVAL, f"tau must have shape ({J}, {N}), got {tau.shape}")
        for t in (mrt_j, f_j):
            if t is not None:
                _check_size(t, J, "per-atom output")
    mrt = ctypes.c_double(0.0)
    frac = ctypes.c_double(0.0)
    ptr = lambda t: ctypes.c_void_p(t.data_ptr()) if t is not None else None  # noqa: E731
    for t in (mrt_j, f_j):
        if t is not None:
            _check_tensor(t)
    st = lib.hq_response_times(ctypes.c_void_p(h), ctypes.c_void_p(dispatch.data_ptr()), tau.ctypes.data_as(_dptr),
                               float(T_bar), ctypes.byref(mrt), ctypes.byref(frac), ptr(mrt_j), ptr(f_j),
                               _stream_ptr(stream))
    if st != HQ_OK:
        raise HQError(st, lib.hq_error_string(ctypes.c_void_p(h)).decode())
    return mrt.value, frac.value


def hq_destroy(h):
    if h:
        _dims.pop(h, None)
        load().hq_destroy(ctypes.c_void_p(h))


def hq_error_string(h=None):
    return load().hq_error_string(ctypes.c_void_p(h) if h else None).decode()


def hq_stats(h):
    out = np.zeros(HQ_STATS_LEN)
    load().hq_stats(ctypes.c_void_p(h), out.ctypes.data_as(_dptr))
    return out


def hq_debug_copy(h, which, nbytes, dtype):
    """Copy an internal device array (see include/hq.h) into a numpy array."""
    out = np.zeros(nbytes // np.dtype(dtype).itemsize, dtype=dtype)
    st = load().hq_debug_copy(ctypes.c_void_p(h), int(which), out.ctypes.data, out.nbytes)
    if st != HQ_OK:
        raise HQError(st, "hq_debug_copy failed")
    return out


def hq_version():
    return load().hq_version().decode()


def _check_tensor(t):
    import torch

    if not (isinstance(t, torch.Tensor) and t.is_cuda and t.dtype == torch.float64 and t.is_contiguous()):
        raise HQError(HQ_E_INVAL, "expected a contiguous float64 CUDA tensor")


# ---------------------------------------------------------------- convenience

class Solver:
    """Owns one hq handle.  ``solve`` returns pi (CUDA float64 tensor)."""

    def __init__(self, lam, mu, pref):
        pref = np.asarray(pref, dtype=np.int32)
        self.J, self.N = pref.shape
        self.h = hq_create(self.N, self.J, lam, mu, pref)

    @classmethod
    def from_instance(cls, inst):
        return cls(inst.lam, inst.mu, inst.pref)

    def solve(self, tol=1e-13, max_iter=10000, pi=None, stream=None):
        import torch

        if pi is None:
            pi = torch.empty(1 << self.N, dtype=torch.float64, device="cuda")
        st, it, res = hq_solve(self.h, tol, max_iter, pi, stream)
        return dict(pi=pi, status=st, iters=it, residual=res)

    def response_times(self, dispatch, tau, T_bar, stream=None):
        import torch

        mj = torch.empty(self.J, dtype=torch.float64, device=dispatch.device)
        fj = torch.empty(self.J, dtype=torch.float64, device=dispatch.device)
        mrt, f = hq_response_times(self.h, dispatch.contiguous(), tau, T_bar, mj, fj, stream)
        return dict(mrt=mrt, frac_within=f, mrt_j=mj, frac_within_j=fj)

    def set_buffer(self, C):
        hq_set_buffer(self.h, C)

    def queue_tail(self, n):
        return hq_queue_tail(self.h, n)

    def measures(self, pi, stream=None):
        import torch

        w = torch.empty(self.N, dtype=torch.float64, device=pi.device)
        d = torch.empty(self.J * self.N, dtype=torch.float64, device=pi.device)
        loss = hq_measures(self.h, pi, w, d, stream)
        return dict(workload=w, dispatch=d.view(self.J, self.N), loss=loss)

    def stats(self):
        s = hq_stats(self.h)
        keys = ["sweeps", "halfsweeps", "state_updates", "launches", "residual_evals", "trie_nodes", "sum_pi_minus_1",
                "solve_ms", "sweep_ms", "sweep_launches", "residual_ms", "precompute_ms", "program_bytes", "path",
                "max_program_block", "program_nwv", "solve_kernel_ms", "device_loop", "chunk_bits",
                "group_lag"]
        return {k: float(s[i]) for i, k in enumerate(keys)}

    def close(self):
        if self.h:
            hq_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()
