"""GPU parity: the CUDA path (through the C-ABI) against the CPU oracle.

Bar (BASELINE.json north_star): both run to relative residual 1e-13, pi within
1e-10 L1 and 1e-12 max-abs, measures within 1e-10.
"""
import numpy as np
import pytest
import torch

import hqinst
import oracle
from oracle import dense

pytestmark = pytest.mark.gpu

TOL = 1e-13
PI_L1 = 1e-10
PI_MAX = 1e-12
MEAS = 1e-10


def gpu_solve(hq, inst, tol=TOL, max_iter=20000):
    s = hq.Solver.from_instance(inst)
    r = s.solve(tol=tol, max_iter=max_iter)
    pi = r["pi"].cpu().numpy()
    m = s.measures(r["pi"])
    out = dict(pi=pi, iters=r["iters"], residual=r["residual"], status=r["status"],
               workload=m["workload"].cpu().numpy(), dispatch=m["dispatch"].cpu().numpy(), loss=m["loss"],
               stats=s.stats())
    s.close()
    return out


def check_parity(g, o, inst):
    assert g["status"] == 0, g
    assert g["residual"] <= TOL
    d = g["pi"] - o["pi"]
    assert np.abs(d).sum() <= PI_L1, np.abs(d).sum()
    assert np.abs(d).max() <= PI_MAX, np.abs(d).max()
    w, disp, loss = oracle.measures(inst, o["pi"])
    assert np.abs(g["workload"] - w).max() <= MEAS
    assert np.abs(g["dispatch"] - disp).max() <= MEAS
    assert abs(g["loss"] - loss) <= MEAS
    # the GPU's own residual claim, re-checked by the oracle's independent code
    assert oracle.residual(inst, g["pi"]) <= 1.5 * TOL


@pytest.mark.parametrize("cfg", [1, 2])
def test_configs_full_oracle(hq, cfg):
    inst = hqinst.config_instance(cfg)
    o = oracle.solve(inst, tol=TOL)
    g = gpu_solve(hq, inst)
    check_parity(g, o, inst)


_SMALL = [
    dict(N=6, J=10, clustered=False, L=None),
    dict(N=8, J=20, clustered=False, L=None),   # largest size of the two-pass path
    dict(N=8, J=25, clustered=True, L=3),
    dict(N=9, J=30, clustered=True, L=None),    # smallest size of the tiled path
    dict(N=11, J=40, clustered=False, L=4),
    dict(N=12, J=80, clustered=False, L=None),
    dict(N=13, J=60, clustered=True, L=6),
    dict(N=15, J=100, clustered=False, L=None),
]


@pytest.mark.parametrize("case", range(len(_SMALL)))
@pytest.mark.parametrize("rho", [0.1, 0.5, 0.9])
def test_generator_variants(hq, case, rho):
    c = _SMALL[case]
    inst = hqinst.generate(c["N"], c["J"], seed=100 + case, rho=rho, clustered=c["clustered"], L=c["L"],
                           mu_lo=0.3 if c["clustered"] else 0.5, mu_hi=2.0 if c["clustered"] else 1.5)
    o = oracle.solve(inst, tol=TOL)
    g = gpu_solve(hq, inst)
    check_parity(g, o, inst)


@pytest.mark.parametrize("N,J,L", [(10, 20, None), (14, 50, None), (17, 90, None)])
def test_iterates_match_algorithm1(hq, N, J, L):
    """The staggered red-black schedule performs Algorithm 1's updates: after
    exactly K sweeps (tol <= 0) the GPU iterate equals the oracle's K-th
    iterate up to rounding (full lists: the closed-form mu* equals the inner
    loop's limit, reading R1)."""
    inst = hqinst.generate(N, J, seed=N, rho=0.6, L=L)
    for K in (1, 3, 17):
        o = oracle.solve(inst, tol=0.0, max_iter=K)
        s = hq.Solver.from_instance(inst)
        r = s.solve(tol=0.0, max_iter=K)
        assert r["iters"] == K
        pi = r["pi"].cpu().numpy()
        s.close()
        assert np.abs(pi - o["pi"]).max() <= 1e-14, (K, np.abs(pi - o["pi"]).max())


def test_dense_lu_tiny(hq):
    for N in (1, 2, 3, 4, 5):
        for L in (None, 2):
            if L is not None and L >= N:
                continue
            inst = hqinst.generate(N, 7, seed=N, rho=0.7, L=L)
            if len(set(inst.pref[inst.pref >= 0].tolist())) < N:
                continue   # some unit in no list: reducible, rejected by hq_create
            lu = dense.stationary(inst.lam, inst.mu, inst.pref)
            g = gpu_solve(hq, inst, tol=1e-14)
            assert g["status"] == 0
            assert np.abs(g["pi"] - lu).max() <= 1e-13, (N, L)
            w, d, loss = dense.measures(inst.lam, inst.mu, inst.pref, lu)
            assert np.abs(g["workload"] - w).max() <= 1e-13
            assert np.abs(g["dispatch"] - d).max() <= 1e-13
            assert abs(g["loss"] - loss) <= 1e-13


def test_cfg2_homogeneous_copy_erlang_layer_masses(hq):
    """Homogeneous copy of cfg2 (nu_i = 1, reading C10): the layer masses are the truncated
    Poisson (Erlang loss) distribution, whatever the preference lists."""
    from test_oracle_pins import truncated_poisson, layer_mass

    inst = hqinst.homogeneous_copy(hqinst.config_instance(2))
    g = gpu_solve(hq, inst)
    a = inst.lam.sum()
    np.testing.assert_allclose(layer_mass(g["pi"], inst.N), truncated_poisson(inst.N, a), rtol=0, atol=1e-12)


def test_ordered_hunt_closed_form(hq):
    from test_oracle_pins import erlang_b

    N = 16
    order = np.random.default_rng(3).permutation(N).astype(np.int32)
    inst = hqinst.ordered_hunt(N, 0.6, J=1, order=order)
    g = gpu_solve(hq, inst)
    a = inst.lam.sum()
    B = erlang_b(N, a)
    ref = np.zeros(N)
    for k, u in enumerate(order, start=1):
        ref[u] = a * (B[k - 1] - B[k])
    np.testing.assert_allclose(g["workload"], ref, rtol=0, atol=1e-11)
    assert abs(g["loss"] - B[N]) <= 1e-12


def test_determinism(hq):
    inst = hqinst.config_instance(2)
    a = gpu_solve(hq, inst)
    b = gpu_solve(hq, inst)
    assert np.array_equal(a["pi"], b["pi"])
    assert a["iters"] == b["iters"]


def test_not_converged_status(hq):
    inst = hqinst.config_instance(1)
    s = hq.Solver.from_instance(inst)
    r = s.solve(tol=1e-13, max_iter=5)
    assert r["status"] == hq.HQ_NOT_CONVERGED
    assert r["iters"] == 5
    assert r["residual"] > 1e-13
    s.close()


def test_measures_before_solve_is_order_error(hq):
    inst = hqinst.config_instance(1)
    s = hq.Solver.from_instance(inst)
    pi = torch.zeros(1 << inst.N, dtype=torch.float64, device="cuda")
    with pytest.raises(hq.HQError) as ei:
        s.measures(pi)
    assert ei.value.status == hq.HQ_E_ORDER
    s.close()


def test_rate_program_overflow_falls_back(hq):
    """Thousands of unstructured (random) full lists: the tiled paths' rate programs would hold
    more than V3_MAXPAIRS distinct (unit, pattern) pairs in a tile; hq_solve falls back to the
    general path (per-thread trie walk, stats path 1) instead of failing, and still matches the
    oracle."""
    N, J = 12, 4000
    rng = np.random.default_rng(2026)
    pref = np.array([rng.permutation(N) for _ in range(J)], dtype=np.int32)
    lam = rng.dirichlet(np.ones(J)) * 0.7 * N
    inst = hqinst.from_arrays(lam, np.ones(N) + rng.random(N), pref, name="random-lists")
    g = gpu_solve(hq, inst)
    assert g["stats"]["path"] == 1
    o = oracle.solve(inst, tol=TOL)
    check_parity(g, o, inst)
