"""Pins for the CPU oracle (-m "not gpu").

Every oracle function is checked against something other than itself:
hand-derived N = 1 / N = 2 values, the Erlang-B closed form, the ordered-hunt
closed form, brute force (dense LU of pi Q = 0 built by independent code in
oracle/dense.py), and exact identities of the model.  See DESIGN.md §3 for the
pin map.
"""
import json
import math
import os

import numpy as np
import pytest

import hqinst
import oracle
from oracle import dense

GOLD = os.path.join(os.path.dirname(__file__), "golden", "spec_n2_examples.json")


def _examples():
    with open(GOLD) as f:
        return {e["name"]: e for e in json.load(f)["examples"]}


def _inst(e):
    return hqinst.from_arrays(e["lam"], e["mu"], e["pref"], name=e["name"])


def erlang_b(N, a):
    """Erlang loss recursion B(0)=1, B(k)=aB(k-1)/(k+aB(k-1))."""
    B = [1.0]
    for k in range(1, N + 1):
        B.append(a * B[-1] / (k + a * B[-1]))
    return B


def truncated_poisson(N, a):
    w = np.array([a ** n / math.factorial(n) for n in range(N + 1)])
    return w / w.sum()


def layer_mass(pi, N):
    pc = np.array([bin(m).count("1") for m in range(1 << N)])
    return np.bincount(pc, weights=pi, minlength=N + 1)


# ---------------------------------------------------------------- hand values

@pytest.mark.parametrize("name", ["N2_homogeneous", "N2_heterogeneous", "N1_mm11"])
def test_hand_examples_pi(name):
    e = _examples()[name]
    inst = _inst(e)
    ref = np.array(e["pi"])
    lu = dense.stationary(inst.lam, inst.mu, inst.pref)
    np.testing.assert_allclose(lu, ref, rtol=0, atol=1e-15)
    r = oracle.solve(inst, tol=1e-15)
    np.testing.assert_allclose(r["pi"], ref, rtol=0, atol=1e-15)
    if "layer_mass" in e:
        np.testing.assert_allclose(layer_mass(r["pi"], inst.N), e["layer_mass"], atol=1e-15)
    if "layer1_mu" in e:
        assert abs(r["layer_mu"][1] - e["layer1_mu"]) < 1e-14
    if "layer1_conditional" in e:
        p1 = r["pi"][[1, 2]] / r["pi"][[1, 2]].sum()
        np.testing.assert_allclose(p1, e["layer1_conditional"], atol=1e-15)


@pytest.mark.parametrize("name", ["N2_homogeneous", "N2_heterogeneous", "N1_mm11"])
def test_hand_examples_measures(name):
    e = _examples()[name]
    inst = _inst(e)
    pi = np.array(e["pi"])
    w, d, loss = oracle.measures(inst, pi)
    np.testing.assert_allclose(w, e["workload"], atol=1e-15)
    if "dispatch" in e:
        np.testing.assert_allclose(d, e["dispatch"], atol=1e-15)
        assert abs(loss - e["loss"]) < 1e-15
    w2, d2, loss2 = dense.measures(inst.lam, inst.mu, inst.pref, pi)
    np.testing.assert_allclose(w2, e["workload"], atol=1e-15)


def test_hand_rates_two_atoms():
    e = _examples()["N2_two_atoms_rates"]
    inst = _inst(e)
    for l, ref in e["out_rates"].items():
        out, lost = oracle.out_rates(inst, int(l))
        np.testing.assert_allclose(out, ref, atol=1e-15)
        assert abs(lost - e["lost"][l]) < 1e-15
    # the dispatch form (Algorithm 3) gives the same numbers seen from the destination
    for m in range(4):
        W = oracle.dispatch_rates(inst, m)
        for i in range(2):
            if (m >> i) & 1:
                out, _ = oracle.out_rates(inst, m ^ (1 << i))
                assert abs(W[i] - out[i]) < 1e-15
            else:
                assert W[i] == 0.0


# ---------------------------------------------------------------- rates

@pytest.mark.parametrize("L", [None, 3])
def test_rates_conservation_and_dense_agreement(L):
    inst = hqinst.generate(7, 15, seed=11, rho=0.6, L=L)
    Q = dense.generator_matrix(inst.lam, inst.mu, inst.pref)
    Lam = inst.lam.sum()
    for l in range(1 << inst.N):
        out, lost = oracle.out_rates(inst, l)
        assert abs(out.sum() + lost - Lam) < 1e-12          # every call goes somewhere or is lost
        for i in range(inst.N):
            if not (l >> i) & 1:
                assert abs(Q[l, l | (1 << i)] - out[i]) < 1e-14   # independent construction
        if L is None and l != (1 << inst.N) - 1:
            assert lost == 0.0                                     # full lists: lambda_m = lambda
    for m in range(1 << inst.N):
        W = oracle.dispatch_rates(inst, m)
        for i in range(inst.N):
            if (m >> i) & 1:
                assert abs(W[i] - Q[m ^ (1 << i), m]) < 1e-14


# ---------------------------------------------------------------- brute force

_VARIANTS = [
    dict(N=8, J=20, clustered=False, L=None, mu_lo=0.5, mu_hi=1.5),
    dict(N=9, J=30, clustered=True, L=None, mu_lo=0.3, mu_hi=2.0),
    dict(N=9, J=40, clustered=False, L=4, mu_lo=0.5, mu_hi=1.5),
    dict(N=10, J=20, clustered=False, L=None, mu_lo=0.5, mu_hi=1.5),
]


@pytest.mark.parametrize("var", range(len(_VARIANTS)))
@pytest.mark.parametrize("rho", [0.1, 0.3, 0.6, 0.9])
@pytest.mark.parametrize("seed", [1, 2, 3])
def test_alg1_matches_dense_lu(var, rho, seed):
    v = _VARIANTS[var]
    inst = hqinst.generate(v["N"], v["J"], seed=seed, rho=rho, mu_lo=v["mu_lo"], mu_hi=v["mu_hi"],
                           clustered=v["clustered"], L=v["L"])
    lu = dense.stationary(inst.lam, inst.mu, inst.pref)
    r = oracle.solve(inst, tol=1e-14, max_iter=3000)
    assert r["status"] == 0, r
    assert np.abs(r["pi"] - lu).sum() <= 1e-11
    assert np.abs(r["pi"] - lu).max() <= 1e-13
    assert abs(r["pi"].sum() - 1.0) <= 1e-13
    # measures: C oracle vs the independent enumeration in dense.py
    w, d, loss = oracle.measures(inst, r["pi"])
    w2, d2, loss2 = dense.measures(inst.lam, inst.mu, inst.pref, lu)
    assert np.abs(w - w2).max() < 1e-12 and np.abs(d - d2).max() < 1e-12 and abs(loss - loss2) < 1e-12


def test_residual_matches_dense_definition():
    inst = hqinst.generate(8, 12, seed=5, rho=0.5, L=5)
    rng = np.random.default_rng(0)
    pi = rng.random(1 << inst.N)
    pi /= pi.sum()
    Q = dense.generator_matrix(inst.lam, inst.mu, inst.pref)
    ref = np.abs(pi @ Q).sum() / (pi * -np.diag(Q)).sum()
    assert abs(oracle.residual(inst, pi) - ref) < 1e-14
    # per-state balance gives the same numbers
    states = np.arange(1 << inst.N, dtype=np.uint64)
    nbr = np.stack([pi] + [pi[np.arange(1 << inst.N) ^ (1 << i)] for i in range(inst.N)], axis=1)
    o, i_ = oracle.state_balance(inst, states, nbr)
    assert abs(np.abs(o - i_).sum() / o.sum() - ref) < 1e-14


# ---------------------------------------------------------------- closed forms

@pytest.mark.parametrize("cfg,N", [(1, 10), (2, 14), (3, 16)])
def test_erlang_layer_masses_homogeneous(cfg, N):
    """Homogeneous nu with full lists: the busy count is M/M/N/N, so the layer
    masses are the truncated Poisson (Erlang loss) law, whatever the lists."""
    inst = hqinst.homogeneous_copy(hqinst.config_instance(cfg, N=N, J=40))
    r = oracle.solve(inst, tol=1e-14, max_iter=4000)
    a = inst.lam.sum() / 1.0
    np.testing.assert_allclose(layer_mass(r["pi"], N), truncated_poisson(N, a), rtol=0, atol=1e-13)
    if N <= 10:
        lu = dense.stationary(inst.lam, inst.mu, inst.pref)
        np.testing.assert_allclose(layer_mass(lu, N), truncated_poisson(N, a), rtol=0, atol=1e-14)


@pytest.mark.parametrize("N,rho", [(7, 0.47), (12, 0.6), (15, 0.9)])
def test_ordered_hunt_closed_form(N, rho):
    """Ordered hunt (every atom, same list), nu = 1: the k-th unit of the order
    carries a (B(k-1,a) - B(k,a)) and the loss is B(N,a)."""
    order = np.random.default_rng(N).permutation(N).astype(np.int32)
    inst = hqinst.ordered_hunt(N, rho, J=3, order=order)
    a = inst.lam.sum()
    B = erlang_b(N, a)
    r = oracle.solve(inst, tol=1e-14, max_iter=4000)
    w, d, loss = oracle.measures(inst, r["pi"])
    ref = np.zeros(N)
    for k, u in enumerate(order, start=1):
        ref[u] = a * (B[k - 1] - B[k])
    np.testing.assert_allclose(w, ref, rtol=0, atol=1e-12)
    assert abs(loss - B[N]) < 1e-13
    if N <= 10:
        lu = dense.stationary(inst.lam, inst.mu, inst.pref)
        w2, _, loss2 = dense.measures(inst.lam, inst.mu, inst.pref, lu)
        np.testing.assert_allclose(w2, ref, rtol=0, atol=1e-14)


# ---------------------------------------------------------------- identities

@pytest.mark.parametrize("L", [None, 4])
def test_flow_identities(L):
    inst = hqinst.generate(11, 60, seed=9, rho=0.7, L=L)
    r = oracle.solve(inst, tol=1e-14, max_iter=3000)
    pi = r["pi"]
    N = inst.N
    w, d, loss = oracle.measures(inst, pi)
    Lam = inst.lam.sum()
    assert abs(d.sum() - 1.0) < 1e-12                                   # every served call dispatches one unit
    np.testing.assert_allclose(inst.mu * w, Lam * (1 - loss) * d.sum(axis=0), rtol=0, atol=1e-12)  # unit flow
    # layer cut balance: P(n-1) lambda(n-1) = P(n) mu(n)  (birth-death structure)
    P = layer_mass(pi, N)
    ll, lm = r["layer_lambda"], r["layer_mu"]
    for n in range(1, N + 1):
        assert abs(P[n - 1] * ll[n - 1] - P[n] * lm[n]) < 1e-13
    assert (pi >= 0).all()
    if L is None:
        assert abs(loss - pi[-1]) < 1e-15   # full lists: lost iff all busy


def test_alg1_residual_decreases_geometrically():
    """Theorem 1: the iterates converge geometrically; the
    trace of r(pi) falls by a roughly constant factor per sweep."""
    inst = hqinst.config_instance(1)
    r = oracle.solve(inst, tol=1e-13, trace=True)
    tr = r["trace"]
    ratios = tr[11:] / tr[10:-1]
    assert (ratios < 1.0).all()
    assert 0.3 < np.median(ratios) < 0.95


# ---------------------------------------------------------------- iterate order (Algorithm 1)

def test_first_sweep_hand_worked_n3():
    """Algorithm 1's first sweep on a hand-worked N = 3 instance: one
    atom with the list (0, 1, 2), lambda = 1, nu = (1, 2, 3).  Worked by hand from
    Eq. updateHeter with the initial p_n = 1/C(3, n) and the initial
    layer rates lambda(n) = 1 (n < 3), mu(1) = 2, mu(2) = 4, mu(3) = 6 (Eqs. lambdaHeter,
    muHeter; reading C8):

      layer 1 (k = 1): a = (1/2, 0, 0), b = (5/24, 1/9, 1/16) for m = 001, 010, 100
        (b carries lambda(1)/mu(2) = 1/4); inner limit mu* = (89/144) / (1 - 1/2) = 89/72
        -> p_1 = (119/144, 16/144, 9/144).
      layer 2 (k = 1) reads the NEW p_1 (sequential order): for m = 011, 101, 110
        A = (16/144 + 119/144, 9/144, 0), den = (4, 5, 6) -> a = (15/64, 1/80, 0);
        D = (3, 2, 1), lambda(2)/mu(3) = 1/6 -> b = (1/8, 1/15, 1/36);
        mu* = (281/360) / (1 - 241/320) = 2248/711.
      pi after the sweep: Prop. 1 with Eq. bnd_stationary on lambda = (1, 1, 1, 0),
        mu = (-, 89/72, 2248/711, 6).

    An oracle that read the previous sweep's p_1 for layer 2 (Jacobi) gives
    A(011) = 2/3 instead of 15/16 and fails this pin."""
    from fractions import Fraction as F

    inst = hqinst.from_arrays([1.0], [1.0, 2.0, 3.0], [[0, 1, 2]], name="N3-hand")
    p1 = {0b001: F(119, 144), 0b010: F(16, 144), 0b100: F(9, 144)}
    ms2 = F(2248, 711)
    a2 = {0b011: F(15, 64), 0b101: F(1, 80), 0b110: F(0)}
    b2 = {0b011: F(1, 8), 0b101: F(1, 15), 0b110: F(1, 36)}
    p2 = {m: ms2 * a2[m] + b2[m] for m in a2}
    assert sum(p2.values()) == 1 and sum(p1.values()) == 1
    g = [F(1), F(72, 89)]
    g.append(g[1] * 1 / ms2)
    g.append(g[2] * 1 / 6)
    tot = sum(g)
    ref = np.zeros(8)
    ref[0] = float(g[0] / tot)
    ref[7] = float(g[3] / tot)
    for m, v in p1.items():
        ref[m] = float(g[1] / tot * v)
    for m, v in p2.items():
        ref[m] = float(g[2] / tot * v)
    r = oracle.solve(inst, tol=0.0, max_iter=1)
    assert r["iters"] == 1
    np.testing.assert_allclose(r["pi"], ref, rtol=0, atol=2e-16)
    np.testing.assert_allclose(r["layer_mu"][1:3], [89 / 72, 2248 / 711], rtol=1e-15)


# ---------------------------------------------------------------- memory-lean residual

@pytest.mark.parametrize("cfg,N,J", [(2, 12, 60), (4, 12, 60), (3, 14, 80), (5, 15, 200)])
def test_tree_rates_match_list_scans(cfg, N, J):
    """The prefix-tree rates of oracle_residual_stream equal Algorithm 3 by list scans
    (dispatch_rates) and lambda_m by list scans, state by state (full and truncated lists)."""
    inst = hqinst.config_instance(cfg, N=N, J=J)
    rng = np.random.default_rng(N)
    for m in rng.integers(0, 1 << N, 64):
        W1 = oracle.dispatch_rates(inst, int(m))
        W2, lm = oracle.tree_rates(inst, int(m))
        scale = inst.lam.sum()
        assert np.abs(W1 - W2).max() <= 1e-14 * scale
        assert abs(lm - oracle.lambda_m(inst, int(m))) <= 1e-14 * scale


@pytest.mark.parametrize("cfg,N,J", [(1, 10, 20), (2, 12, 60), (4, 12, 60), (3, 14, 80)])
def test_residual_stream_matches_residual(cfg, N, J):
    """oracle_residual_stream is the residual of Eq. balance_eq_heter (reading C3) evaluated
    with block sums: equal to oracle_residual on arbitrary vectors (not only near a
    solution) and at the solution, for every block size."""
    inst = hqinst.config_instance(cfg, N=N, J=J)
    rng = np.random.default_rng(3)
    x = rng.random(1 << N)
    x /= x.sum()
    r1 = oracle.residual(inst, x)
    for bb in (0, 5, N):
        r2, num, den = oracle.residual_stream(inst, x, bb)
        assert abs(r2 - r1) <= 1e-13 * r1
        assert num > 0 and den > 0
    sol = oracle.solve(inst, tol=1e-13)["pi"]
    r1 = oracle.residual(inst, sol)
    r2, _, _ = oracle.residual_stream(inst, sol, 6)
    assert r2 <= 1e-13 and abs(r2 - r1) <= 1e-15
