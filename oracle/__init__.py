"""CPU oracle for the spatial hypercube queueing model (arXiv 2603.03019).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and the
``cpu_baseline`` / ``--impl reference`` legs of ``bench.py`` may import this
package.  The product path (``paper_2603_03019_b200``) never imports it, and
it never imports the product path: the two share no code, header, table or
constant generator.  The only module both use is ``hqinst`` (seeded input
generator, no method arithmetic).

Contents
  hq_oracle.c  plain C (+OpenMP over independent states) implementation of
               Algorithm 1, Algorithm 3 rates
               (PAPER.md:541-567), Eq. bnd_stationary, the
               relative balance residual and the performance measures.
  dense.py     the plain definition: dense generator matrix and an LU solve of
               pi Q = 0, sum pi = 1, for N <= 12.

Pins (tests/test_oracle_*.py, ``-m "not gpu"``): hand-derived N = 1 and N = 2
values, the Erlang-B layer masses for homogeneous service rates, the
ordered-hunt closed form for per-unit workloads and loss, brute force (the
dense LU) on tiny instances, rate conservation and the exact flow identities.
Parity status per function is listed in DESIGN.md §3.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "hq_oracle.c")
_LIB_PATH = os.path.join(_HERE, "liboracle.so")
_lock = threading.Lock()
_lib = None

_dptr = ctypes.POINTER(ctypes.c_double)
_iptr = ctypes.POINTER(ctypes.c_int32)
_u64ptr = ctypes.POINTER(ctypes.c_uint64)


def build(force: bool = False) -> str:
    """Compile hq_oracle.c into liboracle.so (gcc, -O2, OpenMP, no fast-math)."""
    if force or not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < os.path.getmtime(_SRC):
        tmp = _LIB_PATH + f".tmp{os.getpid()}"
        cmd = ["gcc", "-O2", "-fopenmp", "-fno-fast-math", "-ffp-contract=off", "-shared", "-fPIC",
               "-std=c11", "-Wall", "-o", tmp, _SRC, "-lm"]
        subprocess.run(cmd, check=True)
        os.replace(tmp, _LIB_PATH)   # new inode: a process that has the old library loaded keeps it
    return _LIB_PATH


def _load():
    global _lib
    with _lock:
        if _lib is None:
            build()
            lib = ctypes.CDLL(_LIB_PATH)
            lib.oracle_solve.restype = ctypes.c_int
            lib.oracle_solve.argtypes = [ctypes.c_int, ctypes.c_int, _dptr, _dptr, _iptr, ctypes.c_double,
                                         ctypes.c_int, ctypes.c_int, _dptr, ctypes.POINTER(ctypes.c_int), _dptr,
                                         _dptr, _dptr, _dptr]
            lib.oracle_residual.restype = ctypes.c_double
            lib.oracle_residual.argtypes = [ctypes.c_int, ctypes.c_int, _dptr, _dptr, _iptr, _dptr]
            lib.oracle_measures.restype = ctypes.c_int
            lib.oracle_measures.argtypes = [ctypes.c_int, ctypes.c_int, _dptr, _dptr, _iptr, _dptr, _dptr, _dptr,
                                            _dptr]
            lib.oracle_dispatch_rates.restype = ctypes.c_int
            lib.oracle_dispatch_rates.argtypes = [ctypes.c_int, ctypes.c_int, _dptr, _iptr, ctypes.c_uint64, _dptr]
            lib.oracle_out_rates.restype = ctypes.c_int
            lib.oracle_out_rates.argtypes = [ctypes.c_int, ctypes.c_int, _dptr, _iptr, ctypes.c_uint64, _dptr,
                                             _dptr]
            lib.oracle_state_balance.restype = ctypes.c_int
            lib.oracle_state_balance.argtypes = [ctypes.c_int, ctypes.c_int, _dptr, _dptr, _iptr, _u64ptr,
                                                 ctypes.c_int64, _dptr, _dptr]
            lib.oracle_residual_stream.restype = ctypes.c_double
            lib.oracle_residual_stream.argtypes = [ctypes.c_int, ctypes.c_int, _dptr, _dptr, _iptr, _dptr,
                                                   ctypes.c_int, _dptr, _dptr]
            lib.oracle_tree_rates.restype = ctypes.c_double
            lib.oracle_tree_rates.argtypes = [ctypes.c_int, ctypes.c_int, _dptr, _iptr, ctypes.c_uint64, _dptr]
            lib.oracle_lambda_m.restype = ctypes.c_double
            lib.oracle_lambda_m.argtypes = [ctypes.c_int, ctypes.c_int, _dptr, _iptr, ctypes.c_uint64]
            lib.oracle_num_threads.restype = ctypes.c_int
            _lib = lib
    return _lib


def _d(a):
    return a.ctypes.data_as(_dptr)


def _arrays(inst):
    lam = np.ascontiguousarray(inst.lam, dtype=np.float64)
    mu = np.ascontiguousarray(inst.mu, dtype=np.float64)
    pref = np.ascontiguousarray(inst.pref, dtype=np.int32)
    return lam, mu, pref


def num_threads() -> int:
    return int(_load().oracle_num_threads())


def solve(inst, tol: float = 1e-13, max_iter: int = 5000, use_table=None, trace: bool = False):
    """Algorithm 1 to relative residual <= tol.  Returns a dict with pi
    (natural index), iters, residual, status, layer_lambda, layer_mu and (if
    trace) the residual after every sweep."""
    lib = _load()
    lam, mu, pref = _arrays(inst)
    N, J = inst.N, inst.J
    if use_table is None:
        use_table = (1 << N) * N * 8 <= 48 * (1 << 30)
    pi = np.zeros(1 << N)
    it = ctypes.c_int(0)
    res = ctypes.c_double(0.0)
    tr = np.full(max_iter, np.nan) if trace else None
    ll = np.zeros(N + 1)
    lm = np.zeros(N + 1)
    st = lib.oracle_solve(N, J, _d(lam), _d(mu), pref.ctypes.data_as(_iptr), tol, max_iter, int(bool(use_table)),
                          _d(pi), ctypes.byref(it), ctypes.byref(res), _d(tr) if trace else None, _d(ll), _d(lm))
    if st < 0:
        raise RuntimeError(f"oracle_solve failed with status {st}")
    out = dict(pi=pi, iters=it.value, residual=res.value, status=st, layer_lambda=ll, layer_mu=lm)
    if trace:
        out["trace"] = tr[: it.value]
    return out


def residual(inst, pi) -> float:
    lib = _load()
    lam, mu, pref = _arrays(inst)
    pi = np.ascontiguousarray(pi, dtype=np.float64)
    assert pi.shape == (1 << inst.N,)
    return float(lib.oracle_residual(inst.N, inst.J, _d(lam), _d(mu), pref.ctypes.data_as(_iptr), _d(pi)))


def residual_stream(inst, pi, block_bits: int = 16):
    """r(pi) like ``residual`` with O(2^N / 2^block_bits) scratch (rates through the
    prefix tree of the lists; fixed-order block sums).  Returns (r, num, den)."""
    lib = _load()
    lam, mu, pref = _arrays(inst)
    pi = np.ascontiguousarray(pi, dtype=np.float64)
    assert pi.shape == (1 << inst.N,)
    num = ctypes.c_double(0.0)
    den = ctypes.c_double(0.0)
    r = lib.oracle_residual_stream(inst.N, inst.J, _d(lam), _d(mu), pref.ctypes.data_as(_iptr), _d(pi),
                                   int(block_bits), ctypes.byref(num), ctypes.byref(den))
    return float(r), num.value, den.value


def tree_rates(inst, m: int):
    """(W[N], lambda_m) of state m through the oracle's prefix tree."""
    lib = _load()
    lam, _, pref = _arrays(inst)
    W = np.zeros(inst.N)
    lm = lib.oracle_tree_rates(inst.N, inst.J, _d(lam), pref.ctypes.data_as(_iptr), int(m), _d(W))
    return W, float(lm)


def lambda_m(inst, m: int) -> float:
    """lambda_m by list scans (Table 1)."""
    lib = _load()
    lam, _, pref = _arrays(inst)
    return float(lib.oracle_lambda_m(inst.N, inst.J, _d(lam), pref.ctypes.data_as(_iptr), int(m)))


def measures(inst, pi):
    """(workload[N], dispatch[J,N], loss) by definition."""
    lib = _load()
    lam, mu, pref = _arrays(inst)
    pi = np.ascontiguousarray(pi, dtype=np.float64)
    work = np.zeros(inst.N)
    disp = np.zeros((inst.J, inst.N))
    loss = np.zeros(1)
    lib.oracle_measures(inst.N, inst.J, _d(lam), _d(mu), pref.ctypes.data_as(_iptr), _d(pi), _d(work), _d(disp),
                        _d(loss))
    return work, disp, float(loss[0])


def dispatch_rates(inst, m: int) -> np.ndarray:
    """Algorithm 3 for state m: W[i] = lambda_{m\\i -> m} for busy i."""
    lib = _load()
    lam, _, pref = _arrays(inst)
    W = np.zeros(inst.N)
    lib.oracle_dispatch_rates(inst.N, inst.J, _d(lam), pref.ctypes.data_as(_iptr), int(m), _d(W))
    return W


def out_rates(inst, l: int):
    """Eq. tran_rates from the source: (out[i] for free i, lost rate)."""
    lib = _load()
    lam, _, pref = _arrays(inst)
    out = np.zeros(inst.N)
    lost = np.zeros(1)
    lib.oracle_out_rates(inst.N, inst.J, _d(lam), pref.ctypes.data_as(_iptr), int(l), _d(out), _d(lost))
    return out, float(lost[0])


def state_balance(inst, states, nbr):
    """Balance at chosen states.  nbr[s] = [pi(m_s), pi(m_s ^ 1), ..., pi(m_s ^ 2^(N-1))].
    Returns (outflow[s], inflow[s])."""
    lib = _load()
    lam, mu, pref = _arrays(inst)
    states = np.ascontiguousarray(states, dtype=np.uint64)
    nbr = np.ascontiguousarray(nbr, dtype=np.float64)
    assert nbr.shape == (states.shape[0], inst.N + 1)
    out = np.zeros(2 * states.shape[0])
    lib.oracle_state_balance(inst.N, inst.J, _d(lam), _d(mu), pref.ctypes.data_as(_iptr),
                             states.ctypes.data_as(_u64ptr), states.shape[0], _d(nbr), _d(out))
    return out[0::2], out[1::2]
