"""GPU parity of the waiting-room extension (include/hq.h
hq_set_buffer / hq_queue_tail) against oracle/buffer.py, through the C-ABI.

The oracle side is the Proposition "Reformulation, Finite Buffer"
applied to the Algorithm-1 CPU oracle, pinned to brute force and closed forms in
tests/test_oracle_buffer.py; at N = 24 (cfg3) the committed oracle fixture of the loss
system is extended by the same birth-death tail."""
import os

import numpy as np
import pytest
import torch

import hqinst
import oracle
from oracle import buffer

pytestmark = pytest.mark.gpu

TOL = 1e-13
U = buffer.UNLIMITED


def gpu_solve_buffer(hq, inst, C, tol=TOL):
    s = hq.Solver.from_instance(inst)
    s.set_buffer(C)
    r = s.solve(tol=tol, max_iter=20000)
    m = s.measures(r["pi"])
    n = 50 if C == U else C
    tail, mass = s.queue_tail(n)
    out = dict(pi=r["pi"].cpu().numpy(), status=r["status"], residual=r["residual"], tail=tail, mass=mass,
               workload=m["workload"].cpu().numpy(), dispatch=m["dispatch"].cpu().numpy(), loss=m["loss"])
    s.close()
    return out


@pytest.mark.parametrize("C", [1, 7, 64, U])
@pytest.mark.parametrize("which", ["cfg1", "n12"])
def test_buffer_parity(hq, which, C):
    inst = hqinst.config_instance(1) if which == "cfg1" else hqinst.generate(12, 40, seed=12, rho=0.75)
    g = gpu_solve_buffer(hq, inst, C)
    assert g["status"] == 0 and g["residual"] <= TOL
    pi_loss = oracle.solve(inst, tol=1e-14, max_iter=20000)["pi"]
    pi, tail = buffer.tail_from_loss(pi_loss, inst.lam.sum(), inst.mu, C)
    assert np.abs(g["pi"] - pi).sum() <= 1e-10
    assert np.abs(g["pi"] - pi).max() <= 1e-12
    n = len(g["tail"])
    np.testing.assert_allclose(g["tail"], tail[:n], rtol=0, atol=1e-12)
    assert abs(g["mass"] - tail.sum()) <= 1e-12
    assert abs(g["pi"].sum() + g["mass"] - 1.0) <= 1e-12
    w, d, loss = buffer.measures_buffer(inst.lam, inst.mu, inst.pref, pi, tail, C)
    assert np.abs(g["workload"] - w).max() <= 1e-10
    assert np.abs(g["dispatch"] - d).max() <= 1e-10
    assert abs(g["loss"] - loss) <= 1e-10


def test_buffer_zero_is_loss_system(hq):
    inst = hqinst.config_instance(1)
    a = gpu_solve_buffer(hq, inst, 0)
    s = hq.Solver.from_instance(inst)
    r = s.solve(tol=TOL)
    m = s.measures(r["pi"])
    assert np.array_equal(a["pi"], r["pi"].cpu().numpy())
    assert a["loss"] == m["loss"] and a["mass"] == 0.0
    s.close()


def test_buffer_unstable_unlimited_rejected(hq):
    inst = hqinst.generate(9, 20, seed=3, rho=1.2)
    s = hq.Solver.from_instance(inst)
    s.set_buffer(hq.HQ_BUFFER_UNLIMITED)
    with pytest.raises(hq.HQError, match="HQ_E_INVAL"):
        s.solve(tol=TOL)
    s.set_buffer(5)   # a finite buffer is stable at any load
    r = s.solve(tol=TOL)
    assert r["status"] == 0
    s.close()


@pytest.mark.parametrize("C", [20, U])
def test_buffer_cfg3_against_fixture(hq, C):
    """N = 24: the loss-system oracle fixture extended by the birth-death tail."""
    inst = hqinst.config_instance(3)
    f = np.load(os.path.join(os.path.dirname(__file__), "golden", "oracle_cfg3.npz"))
    assert str(f["sha256"]) == inst.sha256()
    g = gpu_solve_buffer(hq, inst, C)
    assert g["status"] == 0 and g["residual"] <= TOL
    N = inst.N
    r = inst.lam.sum() / inst.mu.sum()
    pN = float(f["masses"][N])
    cs = np.arange(1, (20 if C != U else 2000) + 1)
    geo = (r ** cs).sum()
    sc = 1.0 / (1.0 + pN * geo)          # Proposition: P{B_m} = sc * pi_loss(m)
    got = g["pi"][f["states"].astype(np.int64)]
    assert np.abs(got - sc * f["pi_states"]).max() <= 1e-12
    np.testing.assert_allclose(g["tail"], sc * pN * r ** cs[: len(g["tail"])], rtol=0, atol=1e-13)
    Lam = inst.lam.sum()
    assert abs(g["dispatch"].sum() - 1.0) <= 1e-12
    np.testing.assert_allclose(inst.mu * g["workload"], Lam * (1.0 - g["loss"]) * g["dispatch"].sum(axis=0),
                               rtol=1e-10, atol=1e-12)


@pytest.mark.parametrize("N", [3, 5, 8])
def test_buffer_small_paths(hq, N):
    """The two-pass path (N <= 8) takes the same waiting room as the tiled path."""
    inst = hqinst.generate(N, 6, seed=N, rho=0.8)
    for C in (2, U):
        g = gpu_solve_buffer(hq, inst, C)
        pi_d, tail_d = buffer.stationary_buffer(inst.lam, inst.mu, inst.pref, 300 if C == U else C)
        assert np.abs(g["pi"] - pi_d).max() <= 1e-12
        n = len(g["tail"])
        np.testing.assert_allclose(g["tail"], tail_d[:n], rtol=0, atol=1e-12)
