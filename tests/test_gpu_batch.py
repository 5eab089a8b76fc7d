"""GPU parity of the batched small-instance solver (include/hq.h
hq_batch_solve) against the CPU oracle (Algorithm 1 + Eq. bnd_stationary), through the C-ABI.
Bar as for the single-instance path: r <= 1e-13, pi within 1e-10 L1 and 1e-12 max-abs."""
import numpy as np
import pytest
import torch

import hqinst
import oracle
from oracle import dense

pytestmark = pytest.mark.gpu
TOL = 1e-13


def stack(insts):
    lam = np.stack([i.lam for i in insts])
    mu = np.stack([i.mu for i in insts])
    pref = np.stack([i.pref for i in insts]).astype(np.int32)
    return lam, mu, pref


def check_against_oracle(insts, pi, it, res, st):
    for b, inst in enumerate(insts):
        assert st[b] == 0 and res[b] <= TOL, (b, st[b], res[b])
        o = oracle.solve(inst, tol=1e-14, max_iter=20000)["pi"]
        g = pi[b].cpu().numpy()
        assert np.abs(g - o).sum() <= 1e-10, b
        assert np.abs(g - o).max() <= 1e-12, b


def test_batch_mixed_n9(hq):
    insts = []
    for k, rho in enumerate([0.1, 0.3, 0.5, 0.7, 0.9, 0.95]):
        for L in (None, 4):
            insts.append(hqinst.generate(9, 30, seed=100 + k, rho=rho, L=L, clustered=bool(k % 2)))
    meas = {}
    pi, it, res, st = hq.hq_batch_solve(*stack(insts), tol=TOL, measures=meas)
    check_against_oracle(insts, pi, it, res, st)
    for b, inst in enumerate(insts):   # measures vs the oracle's, on the GPU pi
        w, d, loss = oracle.measures(inst, pi[b].cpu().numpy())
        assert np.abs(meas["workload"][b].cpu().numpy() - w).max() <= 1e-12
        assert np.abs(meas["dispatch"][b].cpu().numpy() - d).max() <= 1e-12
        assert abs(meas["loss"][b] - loss) <= 1e-12


def test_batch_rho_sweep_n11(hq):
    """The paper's pattern: one geometry, the load swept over 9 values."""
    base = hqinst.generate(11, 71, seed=7, rho=0.5, mu_lo=0.8, mu_hi=1.2)
    insts = []
    for rho in np.linspace(0.1, 0.9, 9):
        lam = base.lam * (rho * base.mu.sum() / base.lam.sum())
        insts.append(hqinst.from_arrays(lam, base.mu, base.pref, rho=float(rho)))
    pi, it, res, st = hq.hq_batch_solve(*stack(insts), tol=TOL)
    check_against_oracle(insts, pi, it, res, st)


def test_batch_n12_and_tiny(hq):
    insts = [hqinst.generate(12, 20, seed=s, rho=0.6) for s in (1, 2, 3)]
    pi, it, res, st = hq.hq_batch_solve(*stack(insts), tol=TOL)
    check_against_oracle(insts, pi, it, res, st)
    for N in (1, 2, 3):
        insts = [hqinst.generate(N, 3, seed=s, rho=0.7) for s in range(4)]
        pi, it, res, st = hq.hq_batch_solve(*stack(insts), tol=TOL)
        for b, inst in enumerate(insts):
            lu = dense.stationary(inst.lam, inst.mu, inst.pref)
            assert np.abs(pi[b].cpu().numpy() - lu).max() <= 1e-13


def test_batch_independent_of_composition_and_matches_hq_solve(hq):
    insts = [hqinst.generate(10, 25, seed=s, rho=0.4 + 0.1 * s) for s in range(5)]
    pi, _, _, _ = hq.hq_batch_solve(*stack(insts), tol=TOL)
    one, _, _, _ = hq.hq_batch_solve(*stack(insts[3:4]), tol=TOL)
    assert torch.equal(pi[3], one[0])   # bitwise: an instance's result does not depend on its batch
    s = hq.Solver.from_instance(insts[3])
    r = s.solve(tol=TOL)
    assert (r["pi"] - pi[3]).abs().max().item() <= 1e-12
    s.close()


def test_batch_not_converged_status(hq):
    insts = [hqinst.generate(9, 30, seed=1, rho=0.9)]
    pi, it, res, st = hq.hq_batch_solve(*stack(insts), tol=TOL, max_iter=3)
    assert st[0] == hq.HQ_NOT_CONVERGED and it[0] == 3 and res[0] > TOL


def test_batch_more_instances_than_ctas(hq):
    """B larger than the resident grid: every CTA loops over several instances."""
    insts = [hqinst.generate(4, 5, seed=s, rho=0.2 + 0.7 * (s % 10) / 10) for s in range(3000)]
    pi, it, res, st = hq.hq_batch_solve(*stack(insts), tol=TOL)
    assert (st == 0).all() and (res <= TOL).all()
    for b in range(0, 3000, 211):
        lu = dense.stationary(insts[b].lam, insts[b].mu, insts[b].pref)
        assert np.abs(pi[b].cpu().numpy() - lu).max() <= 1e-13
